// pdlp_b200.hpp — C++20 host API of the B200 restarted-PDHG solver.
//
// Header-only. Mirrors the reference's C++ API (pdhglp, header-only C++20 under
// /root/reference/proj/include/pdhglp) so a caller of `pdhglp::solve` switches by
// changing the namespace and linking libpdlp_b200.so:
//
//   pdlp_b200::CsrMatrix        <- pdhglp::CsrMatrix        sparse_matrix.hpp:35-55
//   pdlp_b200::GeneralFormLp    <- pdhglp::GeneralFormLp    lp_model.hpp:24-72
//   pdlp_b200::SolverParams     <- pdhglp::SolverParams     solver.hpp:59-94
//   pdlp_b200::SolveStatus      <- pdhglp::SolveStatus      solver.hpp:26-45
//   pdlp_b200::ConvergenceInfo  <- pdhglp::ConvergenceInfo  solver.hpp:165-177
//   pdlp_b200::SolveResult      <- pdhglp::SolveResult      solver.hpp:618-630
//   pdlp_b200::solve            <- pdhglp::solve            solver.hpp:935-940
//   pdlp_b200::read_mps_file    <- pdhglp::read_mps_file    mps_io.hpp:582-585
//   pdlp_b200::write_solution   <- pdhglp::write_solution   solution_io.hpp:90-95
//
// Every call goes through the C ABI of include/pdlp_b200.h; the solve runs on
// the GPU (there is no CPU path). Errors follow the reference: invalid input
// throws std::invalid_argument, I/O and device failures std::runtime_error,
// numerical trouble is a status (SolveStatus::kNumericalError).
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pdlp_b200.h"

namespace pdlp_b200 {

using index_t = std::int64_t;  // sparse_matrix.hpp:21
inline constexpr double kInf = std::numeric_limits<double>::infinity();

enum class SolveStatus {
  kOptimal = PDLP_STATUS_OPTIMAL,
  kPrimalInfeasible = PDLP_STATUS_PRIMAL_INFEASIBLE,
  kDualInfeasible = PDLP_STATUS_DUAL_INFEASIBLE,
  kIterationLimit = PDLP_STATUS_ITERATION_LIMIT,
  kTimeLimit = PDLP_STATUS_TIME_LIMIT,
  kNumericalError = PDLP_STATUS_NUMERICAL_ERROR,
};

inline const char* to_string(SolveStatus s) {
  switch (s) {
    case SolveStatus::kOptimal: return "optimal";
    case SolveStatus::kPrimalInfeasible: return "primal_infeasible";
    case SolveStatus::kDualInfeasible: return "dual_infeasible";
    case SolveStatus::kIterationLimit: return "iteration_limit";
    case SolveStatus::kTimeLimit: return "time_limit";
    case SolveStatus::kNumericalError: return "numerical_error";
  }
  return "unknown";
}

enum class RestartCriterion {
  kNone = PDLP_RESTART_NONE,
  kSufficientDecay = PDLP_RESTART_SUFFICIENT_DECAY,
  kNecessaryDecayNoProgress = PDLP_RESTART_NECESSARY_DECAY,
  kLongInnerLoop = PDLP_RESTART_LONG_INNER_LOOP,
};

enum class ScalingMode { kNone = PDLP_SCALING_NONE, kRuiz = PDLP_SCALING_RUIZ,
                         kRuizPockChambolle = PDLP_SCALING_RUIZ_PC };

enum class MpsFormat { kFixed = PDLP_MPS_FIXED, kFree = PDLP_MPS_FREE, kAuto = PDLP_MPS_AUTO };

struct CsrMatrix {
  index_t num_rows = 0;
  index_t num_cols = 0;
  std::vector<index_t> row_offsets{0};
  std::vector<index_t> col_indices;
  std::vector<double> values;

  index_t nnz() const { return static_cast<index_t>(values.size()); }
  /// Array sizes and offsets the C ABI reads through raw pointers (the
  /// reference's vector-backed CsrMatrix cannot be malformed this way).
  void validate_storage(const char* which) const {
    const std::string w(which);
    if (num_rows < 0 || num_cols < 0) throw std::invalid_argument(w + ": negative dimension");
    if (row_offsets.size() != static_cast<std::size_t>(num_rows) + 1)
      throw std::invalid_argument(w + ": row_offsets must have num_rows + 1 entries");
    if (col_indices.size() != values.size())
      throw std::invalid_argument(w + ": col_indices and values differ in length");
    if (row_offsets.front() != 0 || row_offsets.back() != nnz())
      throw std::invalid_argument(w + ": row_offsets must run from 0 to nnz");
    for (std::size_t r = 0; r + 1 < row_offsets.size(); ++r)
      if (row_offsets[r + 1] < row_offsets[r]) throw std::invalid_argument(w + ": row_offsets not monotone");
  }
  static CsrMatrix zero(index_t rows, index_t cols) {
    CsrMatrix m;
    m.num_rows = rows;
    m.num_cols = cols;
    m.row_offsets.assign(static_cast<std::size_t>(rows + 1), 0);
    return m;
  }
};

/// min c'x + objective_constant  s.t.  Gx >= h, Ax = b, l <= x <= u.
struct GeneralFormLp {
  CsrMatrix inequality_matrix;  // G (m1 x n)
  CsrMatrix equality_matrix;    // A (m2 x n)
  std::vector<double> objective;
  std::vector<double> inequality_rhs;
  std::vector<double> equality_rhs;
  std::vector<double> lower;
  std::vector<double> upper;
  double objective_constant = 0.0;

  index_t num_variables() const { return static_cast<index_t>(objective.size()); }
  index_t num_inequalities() const { return inequality_matrix.num_rows; }
  index_t num_equalities() const { return equality_matrix.num_rows; }
  index_t num_constraints() const { return num_inequalities() + num_equalities(); }

  /// GeneralFormLp::validate (lp_model.hpp:45-72), same checks and messages,
  /// plus the CSR storage checks the raw-pointer ABI needs.
  void validate() const {
    inequality_matrix.validate_storage("lp: inequality matrix");
    equality_matrix.validate_storage("lp: equality matrix");
    const index_t n = num_variables();
    if (inequality_matrix.num_cols != n || equality_matrix.num_cols != n)
      throw std::invalid_argument("lp: constraint matrices must have n columns");
    if (static_cast<index_t>(inequality_rhs.size()) != num_inequalities() ||
        static_cast<index_t>(equality_rhs.size()) != num_equalities())
      throw std::invalid_argument("lp: rhs length does not match row count");
    if (static_cast<index_t>(lower.size()) != n || static_cast<index_t>(upper.size()) != n)
      throw std::invalid_argument("lp: bound vectors must have length n");
    const double inf = std::numeric_limits<double>::infinity();
    for (index_t i = 0; i < n; ++i) {
      const double l = lower[static_cast<std::size_t>(i)], u = upper[static_cast<std::size_t>(i)];
      if (std::isnan(l) || std::isnan(u))
        throw std::invalid_argument("lp: NaN bound on variable " + std::to_string(i));
      if (l > u || l == inf || u == -inf)
        throw std::invalid_argument("lp: empty bound interval on variable " + std::to_string(i));
    }
    for (double v : objective)
      if (std::isnan(v)) throw std::invalid_argument("lp: NaN objective entry");
  }
};

struct SolverParams {
  double eps_optimal = 1e-4;
  double eps_infeasible = 1e-8;
  double time_limit_seconds = 3600.0;
  std::int64_t iteration_limit = std::numeric_limits<std::int64_t>::max();
  double beta_sufficient = 0.2;
  double beta_necessary = 0.8;
  double beta_artificial = 0.36;
  double theta_smoothing = 0.5;
  double eps_zero = 1e-10;
  std::int64_t evaluation_frequency = 64;
  ScalingMode scaling = ScalingMode::kRuizPockChambolle;
  int ruiz_iterations = 10;
  double pock_chambolle_alpha = 1.0;
  double step_reduction_exponent = 0.3;
  double step_growth_exponent = 0.6;
  double omega_min = 1e-8;
  double omega_max = 1e8;
  bool record_step_log = false;
  // ---- B200 execution knobs ----
  int device = 0;
  bool parity_mode = false;  // PDLP_MODE_PARITY: bitwise-reference iterates
  bool use_cuda_graph = true;
  int engine = PDLP_ENGINE_AUTO;
  int world_size = 1;  // row sharding: this handle is `rank` of `world_size` (one per GPU)
  int rank = 0;
  int plan_world = 0;

  void validate() const {  // solver.hpp:79-93
    if (!(eps_optimal > 0.0) || !(eps_infeasible > 0.0))
      throw std::invalid_argument("params: tolerances must be positive");
    if (!(beta_sufficient > 0.0 && beta_sufficient < beta_necessary && beta_necessary < 1.0))
      throw std::invalid_argument("params: need 0 < beta_sufficient < beta_necessary < 1");
    if (theta_smoothing < 0.0 || theta_smoothing > 1.0)
      throw std::invalid_argument("params: theta_smoothing must lie in [0, 1]");
    if (evaluation_frequency < 1)
      throw std::invalid_argument("params: evaluation_frequency must be >= 1");
  }
};

struct PrimalDualPoint {
  std::vector<double> primal;
  std::vector<double> dual;
};

struct ReducedCosts {
  std::vector<double> lambda;
  std::vector<double> lambda_pos;
  std::vector<double> lambda_neg;
};

struct ConvergenceInfo {
  double primal_objective = 0.0;
  double dual_objective = 0.0;
  double primal_objective_raw = 0.0;
  double dual_objective_raw = 0.0;
  double gap_abs = 0.0;
  double primal_residual_norm = 0.0;
  double dual_residual_norm = 0.0;
  double relative_gap = 0.0;
  double relative_primal_residual = 0.0;
  double relative_dual_residual = 0.0;
  double kkt_omega = 0.0;
};

struct InfeasibilityCertificate {
  SolveStatus status = SolveStatus::kPrimalInfeasible;
  std::vector<double> primal_ray;  // dual-infeasibility witness
  std::vector<double> dual_ray;    // primal-infeasibility witness
  ReducedCosts dual_ray_reduced_costs;
};

using StepLogEntry = pdlp_step_log_entry;
using RestartEvent = pdlp_restart_event;

struct SolveResult {
  SolveStatus status = SolveStatus::kNumericalError;
  PrimalDualPoint point;
  ReducedCosts reduced;
  ConvergenceInfo info;
  std::int64_t iterations = 0;
  std::int64_t restarts = 0;
  double solve_seconds = 0.0;
  std::optional<InfeasibilityCertificate> certificate;
  std::vector<StepLogEntry> step_log;
  std::vector<RestartEvent> restart_log;
  std::string message;
  // B200 extensions
  double setup_seconds = 0.0;
  double device_seconds = 0.0;
  std::int64_t trials = 0;
};

namespace detail {

[[noreturn]] inline void rethrow(int rc) {
  const char* msg = pdlp_last_error();
  std::string m = msg ? msg : "";
  if (rc == PDLP_EINVAL) throw std::invalid_argument(m);
  throw std::runtime_error("pdlp_b200 error " + std::to_string(rc) + ": " + m);
}

inline void check(int rc) {
  if (rc != PDLP_OK) rethrow(rc);
}

inline pdlp_csr view(const CsrMatrix& m) {
  pdlp_csr c{};
  c.num_rows = m.num_rows;
  c.num_cols = m.num_cols;
  c.nnz = m.nnz();
  c.row_offsets = m.row_offsets.data();
  c.col_indices = m.col_indices.data();
  c.col_indices32 = nullptr;
  c.values = m.values.data();
  return c;
}

inline pdlp_lp view(const GeneralFormLp& lp) {
  pdlp_lp v{};
  v.inequality_matrix = view(lp.inequality_matrix);
  v.equality_matrix = view(lp.equality_matrix);
  v.num_variables = lp.num_variables();
  v.objective = lp.objective.data();
  v.inequality_rhs = lp.inequality_rhs.data();
  v.equality_rhs = lp.equality_rhs.data();
  v.lower = lp.lower.data();
  v.upper = lp.upper.data();
  v.objective_constant = lp.objective_constant;
  return v;
}

inline pdlp_params to_c(const SolverParams& p) {
  pdlp_params c;
  pdlp_default_params(&c);
  c.eps_optimal = p.eps_optimal;
  c.eps_infeasible = p.eps_infeasible;
  c.time_limit_seconds = p.time_limit_seconds;
  c.iteration_limit = p.iteration_limit;
  c.beta_sufficient = p.beta_sufficient;
  c.beta_necessary = p.beta_necessary;
  c.beta_artificial = p.beta_artificial;
  c.theta_smoothing = p.theta_smoothing;
  c.eps_zero = p.eps_zero;
  c.evaluation_frequency = p.evaluation_frequency;
  c.scaling = static_cast<int32_t>(p.scaling);
  c.ruiz_iterations = p.ruiz_iterations;
  c.pock_chambolle_alpha = p.pock_chambolle_alpha;
  c.step_reduction_exponent = p.step_reduction_exponent;
  c.step_growth_exponent = p.step_growth_exponent;
  c.omega_min = p.omega_min;
  c.omega_max = p.omega_max;
  c.record_step_log = p.record_step_log ? 1 : 0;
  c.device = p.device;
  c.mode = p.parity_mode ? PDLP_MODE_PARITY : PDLP_MODE_FAST;
  c.use_cuda_graph = p.use_cuda_graph ? 1 : 0;
  c.engine = p.engine;
  c.world_size = p.world_size;
  c.rank = p.rank;
  c.plan_world = p.plan_world;
  return c;
}

inline std::vector<index_t> widen(const int64_t* p, int64_t n) { return {p, p + n}; }

}  // namespace detail

/// A device-resident instance: the LP is uploaded, K^T built and the
/// preconditioner applied once; solve() may be called repeatedly (each call
/// restarts from z = 0, like pdhglp::solve).
class Solver {
 public:
  Solver(const GeneralFormLp& lp, const SolverParams& params = {}) {
    lp.validate();
    params.validate();
    const pdlp_lp v = detail::view(lp);
    const pdlp_params p = detail::to_c(params);
    detail::check(pdlp_create(&v, &p, &h_));
    n_ = lp.num_variables();
    m_ = lp.num_constraints();
  }
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;
  Solver(Solver&& o) noexcept : h_(std::exchange(o.h_, nullptr)), n_(o.n_), m_(o.m_) {}
  ~Solver() { pdlp_destroy(h_); }

  SolveResult solve() {
    pdlp_result_info info{};
    detail::check(pdlp_solve(h_, &info));
    SolveResult r;
    r.status = static_cast<SolveStatus>(info.status);
    r.iterations = info.iterations;
    r.restarts = info.restarts;
    r.solve_seconds = info.solve_seconds;
    r.setup_seconds = info.setup_seconds;
    r.device_seconds = info.device_seconds;
    r.trials = info.trials;
    r.message = info.message;
    ConvergenceInfo& c = r.info;
    c.primal_objective = info.primal_objective;
    c.dual_objective = info.dual_objective;
    c.primal_objective_raw = info.primal_objective_raw;
    c.dual_objective_raw = info.dual_objective_raw;
    c.gap_abs = info.gap_abs;
    c.primal_residual_norm = info.primal_residual_norm;
    c.dual_residual_norm = info.dual_residual_norm;
    c.relative_gap = info.relative_gap;
    c.relative_primal_residual = info.relative_primal_residual;
    c.relative_dual_residual = info.relative_dual_residual;
    c.kkt_omega = info.kkt_omega;
    const auto n = static_cast<std::size_t>(n_), m = static_cast<std::size_t>(m_);
    r.point.primal.assign(n, 0.0);
    r.point.dual.assign(m, 0.0);
    r.reduced.lambda.assign(n, 0.0);
    r.reduced.lambda_pos.assign(n, 0.0);
    r.reduced.lambda_neg.assign(n, 0.0);
    detail::check(pdlp_get_solution(h_, r.point.primal.data(), r.point.dual.data(),
                                    r.reduced.lambda.data(), r.reduced.lambda_pos.data(),
                                    r.reduced.lambda_neg.data()));
    r.step_log.resize(static_cast<std::size_t>(info.step_log_size));
    r.restart_log.resize(static_cast<std::size_t>(info.restart_log_size));
    if (!r.step_log.empty())
      detail::check(pdlp_get_step_log(h_, r.step_log.data(), info.step_log_size));
    if (!r.restart_log.empty())
      detail::check(pdlp_get_restart_log(h_, r.restart_log.data(), info.restart_log_size));
    if (info.has_certificate) {  // solver.hpp:868-883: the point IS the ray
      InfeasibilityCertificate cert;
      cert.status = r.status;
      if (r.status == SolveStatus::kPrimalInfeasible) {
        cert.dual_ray = r.point.dual;
        cert.dual_ray_reduced_costs = r.reduced;
      } else {
        cert.primal_ray = r.point.primal;
      }
      r.certificate = std::move(cert);
    }
    return r;
  }

  /// spmv / spmv_transpose (sparse_matrix.hpp:117-165) on the device operator.
  std::vector<double> spmv(int op, const std::vector<double>& in) {
    const bool t = op == PDLP_OP_KT_SCALED || op == PDLP_OP_KT_ORIGINAL;
    if (static_cast<index_t>(in.size()) != (t ? m_ : n_))
      throw std::invalid_argument("spmv: dimension mismatch");
    std::vector<double> out(static_cast<std::size_t>(t ? n_ : m_));
    detail::check(pdlp_spmv(h_, op, in.data(), out.data()));
    return out;
  }

  /// pdhg_raw_step (solver.hpp:335-358) on the unscaled saddle problem: one
  /// plain PDHG step from z with explicit extrapolation 2x' - x.
  PrimalDualPoint pdhg_raw_step(const PrimalDualPoint& z, double tau, double sigma) {
    if (static_cast<index_t>(z.primal.size()) != n_ || static_cast<index_t>(z.dual.size()) != m_)
      throw std::invalid_argument("pdhg_raw_step: dimension mismatch");
    PrimalDualPoint next;
    next.primal.resize(z.primal.size());
    next.dual.resize(z.dual.size());
    detail::check(pdlp_pdhg_raw_step(h_, z.primal.data(), z.dual.data(), tau, sigma, next.primal.data(),
                                     next.dual.data()));
    return next;
  }

  /// Row sharding, one process per GPU: export this rank's blob, all-gather
  /// the blobs (MPI, torch.distributed, files), import them in rank order.
  std::vector<unsigned char> shard_export() const {
    std::vector<unsigned char> b(static_cast<std::size_t>(pdlp_shard_blob_size()));
    detail::check(pdlp_shard_export(h_, b.data(), static_cast<int64_t>(b.size())));
    return b;
  }
  void shard_import(const std::vector<std::vector<unsigned char>>& blobs) {
    std::vector<unsigned char> all;
    for (const auto& b : blobs) all.insert(all.end(), b.begin(), b.end());
    detail::check(pdlp_shard_import(h_, all.data(), static_cast<int32_t>(blobs.size())));
  }

  pdlp_handle* handle() const { return h_; }

 private:
  pdlp_handle* h_ = nullptr;
  index_t n_ = 0, m_ = 0;
};

/// pdhglp::solve (solver.hpp:935-940) on the GPU.
inline SolveResult solve(const GeneralFormLp& lp, const SolverParams& params = {}) {
  Solver s(lp, params);
  return s.solve();
}

/// read_mps_file (mps_io.hpp:582-585): fixed / free / auto, gzip by extension.
/// Parse errors throw std::runtime_error naming the line; crossing bounds
/// std::invalid_argument (mps_io.hpp:536-546).
inline GeneralFormLp read_mps_file(const std::string& path, MpsFormat format = MpsFormat::kAuto) {
  pdlp_lp_file* f = nullptr;
  detail::check(pdlp_read_mps(path.c_str(), static_cast<int32_t>(format), &f));
  const pdlp_lp* v = pdlp_lp_file_lp(f);
  GeneralFormLp lp;
  auto copy = [](const pdlp_csr& c) {
    CsrMatrix m;
    m.num_rows = c.num_rows;
    m.num_cols = c.num_cols;
    m.row_offsets = detail::widen(c.row_offsets, c.num_rows + 1);
    m.col_indices = detail::widen(c.col_indices, c.nnz);
    m.values.assign(c.values, c.values + c.nnz);
    return m;
  };
  lp.inequality_matrix = copy(v->inequality_matrix);
  lp.equality_matrix = copy(v->equality_matrix);
  const auto n = v->num_variables, m1 = v->inequality_matrix.num_rows, m2 = v->equality_matrix.num_rows;
  lp.objective.assign(v->objective, v->objective + n);
  lp.inequality_rhs.assign(v->inequality_rhs, v->inequality_rhs + m1);
  lp.equality_rhs.assign(v->equality_rhs, v->equality_rhs + m2);
  lp.lower.assign(v->lower, v->lower + n);
  lp.upper.assign(v->upper, v->upper + n);
  lp.objective_constant = v->objective_constant;
  pdlp_lp_file_free(f);
  return lp;
}

/// write_solution (solution_io.hpp:70-95): the `format_version 1` key-value file.
inline void write_solution(const SolveResult& r, const std::string& path, bool include_vectors = false) {
  pdlp_result_info info{};
  info.status = static_cast<int32_t>(r.status);
  info.primal_objective = r.info.primal_objective;
  info.dual_objective = r.info.dual_objective;
  info.relative_gap = r.info.relative_gap;
  info.primal_residual_norm = r.info.primal_residual_norm;
  info.dual_residual_norm = r.info.dual_residual_norm;
  info.iterations = r.iterations;
  info.solve_seconds = r.solve_seconds;
  const bool v = include_vectors;
  detail::check(pdlp_write_solution(path.c_str(), &info, v ? r.point.primal.data() : nullptr,
                                    static_cast<int64_t>(r.point.primal.size()),
                                    v ? r.point.dual.data() : nullptr,
                                    static_cast<int64_t>(r.point.dual.size())));
}

}  // namespace pdlp_b200
