// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.
//
// Exposes the *unmodified* reference solver (pdhglp, header-only C++20, read
// in place from $(PDHGLP_INCLUDE) = /root/reference/proj/include) behind the
// same C entry points as oracle/pdlp_oracle.c, with prefix ref_ instead of
// oracle_. Built by oracle/Makefile into oracle/_ref/libpdhglp_ref.so, which is
// git-ignored and travels to the GPU box with the snapshot. No reference source
// is copied into this repository; this file only converts between the C-ABI
// structs of include/pdlp_b200.h and pdhglp's types and calls:
//   pdhglp::solve                       solver.hpp:935-940
//   detail::adaptive_step_cached etc.   solver.hpp:130-590 (re-driven loop, as
//                                       SolveLoop::run does, solver.hpp:759-929)
//   make_scaling                        scaling.hpp:117-132
//   spmv / spmv_transpose / explicit_transpose / from_triplets
//                                       sparse_matrix.hpp:57-178
//   read_mps_file                       mps_io.hpp:582-585
//   config_hash / aggregate_records / write_report / run_benchmark
//                                       bench.hpp:29-267
//   restarted_pdhg_standard / kkt_error_standard / spectral_norm /
//   p_s_norm_squared                    standard_form.hpp:36-211
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include <sstream>

#include "pdhglp/bench.hpp"
#include "pdhglp/mps_io.hpp"
#include "pdhglp/standard_form.hpp"
#include "pdhglp/scaling.hpp"
#include "pdhglp/solver.hpp"
#include "pdhglp/sparse_matrix.hpp"

extern "C" {
#include "pdlp_b200.h"
}

using namespace pdhglp;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

CsrMatrix to_csr(const pdlp_csr& c) {
  CsrMatrix m;
  m.num_rows = c.num_rows;
  m.num_cols = c.num_cols;
  m.row_offsets.assign(c.row_offsets, c.row_offsets + c.num_rows + 1);
  m.col_indices.resize(static_cast<size_t>(c.nnz));
  for (int64_t k = 0; k < c.nnz; ++k)
    m.col_indices[k] = c.col_indices ? c.col_indices[k] : c.col_indices32[k];
  m.values.assign(c.values, c.values + c.nnz);
  return m;
}

GeneralFormLp to_lp(const pdlp_lp& in) {
  GeneralFormLp lp;
  lp.inequality_matrix = to_csr(in.inequality_matrix);
  lp.equality_matrix = to_csr(in.equality_matrix);
  const int64_t n = in.num_variables;
  const int64_t m1 = in.inequality_matrix.num_rows, m2 = in.equality_matrix.num_rows;
  lp.objective.assign(in.objective, in.objective + n);
  lp.inequality_rhs.assign(in.inequality_rhs, in.inequality_rhs + m1);
  lp.equality_rhs.assign(in.equality_rhs, in.equality_rhs + m2);
  lp.lower.assign(in.lower, in.lower + n);
  lp.upper.assign(in.upper, in.upper + n);
  lp.objective_constant = in.objective_constant;
  return lp;
}

SolverParams to_params(const pdlp_params& p) {
  SolverParams s;
  s.eps_optimal = p.eps_optimal;
  s.eps_infeasible = p.eps_infeasible;
  s.time_limit_seconds = p.time_limit_seconds;
  s.iteration_limit = p.iteration_limit;
  s.beta_sufficient = p.beta_sufficient;
  s.beta_necessary = p.beta_necessary;
  s.beta_artificial = p.beta_artificial;
  s.theta_smoothing = p.theta_smoothing;
  s.eps_zero = p.eps_zero;
  s.evaluation_frequency = p.evaluation_frequency;
  s.scaling = p.scaling == PDLP_SCALING_NONE ? ScalingMode::kNone
              : p.scaling == PDLP_SCALING_RUIZ ? ScalingMode::kRuiz
                                               : ScalingMode::kRuizPockChambolle;
  s.ruiz_iterations = p.ruiz_iterations;
  s.pock_chambolle_alpha = p.pock_chambolle_alpha;
  s.step_reduction_exponent = p.step_reduction_exponent;
  s.step_growth_exponent = p.step_growth_exponent;
  s.omega_min = p.omega_min;
  s.omega_max = p.omega_max;
  s.record_step_log = p.record_step_log != 0;
  return s;
}

void copy_out(const std::vector<double>& v, double* dst) {
  if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
}

void fill_info(const SolveResult& r, int64_t n, int64_t m, pdlp_result_info* info) {
  std::memset(info, 0, sizeof *info);
  info->status = static_cast<int32_t>(r.status);
  info->has_certificate = r.certificate.has_value() ? 1 : 0;
  info->iterations = r.iterations;
  info->restarts = r.restarts;
  info->solve_seconds = r.solve_seconds;
  info->primal_objective = r.info.primal_objective;
  info->dual_objective = r.info.dual_objective;
  info->primal_objective_raw = r.info.primal_objective_raw;
  info->dual_objective_raw = r.info.dual_objective_raw;
  info->gap_abs = r.info.gap_abs;
  info->primal_residual_norm = r.info.primal_residual_norm;
  info->dual_residual_norm = r.info.dual_residual_norm;
  info->relative_gap = r.info.relative_gap;
  info->relative_primal_residual = r.info.relative_primal_residual;
  info->relative_dual_residual = r.info.relative_dual_residual;
  info->kkt_omega = r.info.kkt_omega;
  info->step_log_size = static_cast<int64_t>(r.step_log.size());
  info->restart_log_size = static_cast<int64_t>(r.restart_log.size());
  info->num_variables = n;
  info->num_constraints = m;
  std::snprintf(info->message, sizeof info->message, "%s", r.message.c_str());
}

void copy_logs(const SolveResult& r, pdlp_step_log_entry* sl, int64_t scap,
               pdlp_restart_event* rl, int64_t rcap) {
  if (sl)
    for (int64_t i = 0; i < static_cast<int64_t>(r.step_log.size()) && i < scap; ++i) {
      const StepLogEntry& e = r.step_log[i];
      sl[i] = {e.step_counter, e.omega, e.eta_accepted, e.eta_bar, e.eta_next, e.movement_sq,
               e.interaction};
    }
  if (rl)
    for (int64_t i = 0; i < static_cast<int64_t>(r.restart_log.size()) && i < rcap; ++i) {
      const RestartEvent& e = r.restart_log[i];
      rl[i].total_iterations = e.total_iterations;
      rl[i].epoch_length = e.epoch_length;
      rl[i].criterion = static_cast<int32_t>(e.criterion);
      rl[i].candidate_is_average = e.candidate_is_average ? 1 : 0;
      rl[i].kkt_candidate = e.kkt_candidate;
      rl[i].kkt_previous_candidate = e.kkt_previous_candidate;
      rl[i].kkt_epoch_start = e.kkt_epoch_start;
      rl[i].omega_before = e.omega_before;
      rl[i].omega_after = e.omega_after;
    }
}

// Re-driven SolveLoop::run (solver.hpp:759-929) using the reference's own
// building blocks, paused every `count` accepted iterations so per-iterate
// state can be read. SolveLoop keeps these members private, hence the mirror.
// The read-only part (the instance, its scaling and saddle form) is shared by
// forked sessions (ref_fork): concurrent independent solves of one instance
// without one copy of the operators per thread.
struct Setup {
  GeneralFormLp lp;
  SolverParams p;
  TerminationNorms norms;
  DiagonalScaling scaling;
  GeneralFormLp scaled;
  SaddleProblem saddle;
};

struct Session {
  explicit Session(std::shared_ptr<Setup> s)
      : su(std::move(s)), lp(su->lp), p(su->p), norms(su->norms), scaling(su->scaling),
        scaled(su->scaled), saddle(su->saddle) {}
  Session(const Session&) = default;
  std::shared_ptr<Setup> su;
  const GeneralFormLp& lp;
  const SolverParams& p;
  const TerminationNorms& norms;
  const DiagonalScaling& scaling;
  const GeneralFormLp& scaled;
  const SaddleProblem& saddle;
  PrimalDualPoint current, epoch_start, last_delta;
  std::vector<double> kx, kty;
  WeightedAverage avg_x{0}, avg_y{0};
  double eta = 0, eta_hat = 0, omega = 1;
  int64_t outer = 0, inner = 0, total = 0, trials = 0;
  double kkt_epoch_start = 0, kkt_last = 0;
  std::chrono::steady_clock::time_point t0;
  bool finished = false;
  SolveResult result;

  double elapsed() const {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }

  struct Eval {
    PrimalDualPoint cand_scaled, cand_unscaled, other_unscaled;
    PointEvaluation cand_eval, other_eval;
    bool cand_is_avg = false, terminated = false, other_terminated = false;
    double kkt_cand = 0;
  };

  Eval evaluate() const {
    Eval ev;
    const PrimalDualPoint avg =
        avg_x.empty() ? current : PrimalDualPoint{avg_x.value(), avg_y.value()};
    const PrimalDualPoint cu = unscale_point(current, scaling);
    const PrimalDualPoint au = unscale_point(avg, scaling);
    const PointEvaluation ec = evaluate_point(lp, cu);
    const PointEvaluation ea = evaluate_point(lp, au);
    const double kc = ec.residuals.weighted(omega), ka = ea.residuals.weighted(omega);
    ev.cand_is_avg = !(kc < ka);
    if (ev.cand_is_avg) {
      ev.cand_scaled = avg; ev.cand_unscaled = au; ev.cand_eval = ea; ev.kkt_cand = ka;
      ev.other_unscaled = cu; ev.other_eval = ec;
    } else {
      ev.cand_scaled = current; ev.cand_unscaled = cu; ev.cand_eval = ec; ev.kkt_cand = kc;
      ev.other_unscaled = au; ev.other_eval = ea;
    }
    ev.terminated = termination_criteria_met(ev.cand_eval.residuals, p.eps_optimal, norms);
    ev.other_terminated = termination_criteria_met(ev.other_eval.residuals, p.eps_optimal, norms);
    return ev;
  }

  void finish(SolveStatus st, const PrimalDualPoint& pt, const PointEvaluation& ev,
              std::string msg = {}) {
    result.status = st;
    result.point = pt;
    result.reduced = ev.reduced;
    result.info = make_convergence_info(lp, ev.residuals, norms, omega);
    result.iterations = total;
    result.restarts = outer;
    result.solve_seconds = elapsed();
    result.message = std::move(msg);
    finished = true;
  }

  static void prepare(Setup& su) {
    su.norms = termination_norms(su.lp);
    su.scaling = make_scaling(vstack(su.lp.inequality_matrix, su.lp.equality_matrix), su.p.scaling,
                              su.p.ruiz_iterations, su.p.pock_chambolle_alpha);
    su.scaled = apply_scaling(su.lp, su.scaling);
    su.saddle = to_saddle(su.scaled);
  }

  void begin() {
    t0 = std::chrono::steady_clock::now();
    const index_t n = saddle.num_variables(), m = saddle.num_constraints();
    current = PrimalDualPoint::zeros(n, m);
    epoch_start = current;
    kx.assign(m, 0.0);
    kty.assign(n, 0.0);
    spmv(saddle.constraint_matrix, current.primal, kx);
    spmv_transpose(saddle.constraint_matrix, current.dual, kty);
    const double max_abs = max_abs_entry(saddle.constraint_matrix);
    eta_hat = max_abs > 0.0 ? 1.0 / max_abs : 1.0;
    eta = eta_hat;
    omega = std::clamp(initialize_primal_weight(saddle.objective, saddle.rhs, p.eps_zero),
                       p.omega_min, p.omega_max);
    avg_x = WeightedAverage(static_cast<size_t>(n));
    avg_y = WeightedAverage(static_cast<size_t>(m));
    last_delta = PrimalDualPoint::zeros(n, m);
    const PrimalDualPoint z0 = unscale_point(current, scaling);
    const PointEvaluation ev0 = evaluate_point(lp, z0);
    kkt_epoch_start = ev0.residuals.weighted(omega);
    kkt_last = kkt_epoch_start;
    if (termination_criteria_met(ev0.residuals, p.eps_optimal, norms))
      finish(SolveStatus::kOptimal, z0, ev0);
  }

  void run(int64_t count) {
    const index_t n = saddle.num_variables(), m = saddle.num_constraints();
    for (int64_t done = 0; !finished && done < count; ++done) {
      if (total >= p.iteration_limit) {
        Eval ev = evaluate();
        finish(SolveStatus::kIterationLimit, ev.cand_unscaled, ev.cand_eval);
        break;
      }
      if (elapsed() >= p.time_limit_seconds) {
        Eval ev = evaluate();
        finish(SolveStatus::kTimeLimit, ev.cand_unscaled, ev.cand_eval);
        break;
      }
      AdaptiveStepResult step = detail::adaptive_step_cached(current, kx, kty, omega, eta_hat,
                                                             total + 1, saddle, p);
      trials += step.trials;
      if (step.numerical_failure) {
        Eval ev = evaluate();
        finish(SolveStatus::kNumericalError, ev.cand_unscaled, ev.cand_eval,
               "non-finite iterate in adaptive step at iteration " + std::to_string(total));
        break;
      }
      if (p.record_step_log)
        result.step_log.push_back({total + 1, omega, step.eta_accepted, step.eta_bar,
                                   step.eta_next, step.movement_sq, step.interaction});
      for (size_t i = 0; i < last_delta.primal.size(); ++i)
        last_delta.primal[i] = step.next.primal[i] - current.primal[i];
      for (size_t i = 0; i < last_delta.dual.size(); ++i)
        last_delta.dual[i] = step.next.dual[i] - current.dual[i];
      current = std::move(step.next);
      kx = std::move(step.k_x_next);
      kty = std::move(step.kt_y_next);
      eta = step.eta_accepted;
      eta_hat = step.eta_next;
      total += 1;
      inner += 1;
      avg_x.add(current.primal, eta);
      avg_y.add(current.dual, eta);
      if (inner % p.evaluation_frequency != 0) continue;

      Eval ev = evaluate();
      if (ev.terminated) { finish(SolveStatus::kOptimal, ev.cand_unscaled, ev.cand_eval); break; }
      if (ev.other_terminated) { finish(SolveStatus::kOptimal, ev.other_unscaled, ev.other_eval); break; }
      {
        PrimalDualPoint normalized = current;
        const double inv_t = 1.0 / static_cast<double>(inner);
        for (size_t i = 0; i < normalized.primal.size(); ++i)
          normalized.primal[i] = inv_t * (normalized.primal[i] - epoch_start.primal[i]);
        for (size_t i = 0; i < normalized.dual.size(); ++i)
          normalized.dual[i] = inv_t * (normalized.dual[i] - epoch_start.dual[i]);
        const auto cert = check_infeasibility(unscale_point(last_delta, scaling),
                                              unscale_point(normalized, scaling), lp,
                                              p.eps_infeasible, p.eps_zero);
        if (cert) {
          PrimalDualPoint ray;
          ReducedCosts red;
          if (cert->status == SolveStatus::kPrimalInfeasible) {
            ray.primal.assign(static_cast<size_t>(n), 0.0);
            ray.dual = cert->dual_ray;
            red = cert->dual_ray_reduced_costs;
          } else {
            ray.primal = cert->primal_ray;
            ray.dual.assign(static_cast<size_t>(m), 0.0);
            red = reduced_costs(lp, ray.dual);
          }
          finish(cert->status, ray, ev.cand_eval);
          result.reduced = red;
          result.certificate = cert;
          break;
        }
      }
      const double prev = kkt_last;
      const RestartCriterion crit =
          should_restart(ev.kkt_cand, prev, kkt_epoch_start, inner, total, p);
      kkt_last = ev.kkt_cand;
      if (crit == RestartCriterion::kNone) continue;
      RestartEvent e;
      e.total_iterations = total;
      e.epoch_length = inner;
      e.criterion = crit;
      e.candidate_is_average = ev.cand_is_avg;
      e.kkt_candidate = ev.kkt_cand;
      e.kkt_previous_candidate = prev;
      e.kkt_epoch_start = kkt_epoch_start;
      e.omega_before = omega;
      const PrimalDualPoint prev_start = epoch_start;
      epoch_start = ev.cand_scaled;
      current = ev.cand_scaled;
      spmv(saddle.constraint_matrix, current.primal, kx);
      spmv_transpose(saddle.constraint_matrix, current.dual, kty);
      outer += 1;
      inner = 0;
      avg_x.reset();
      avg_y.reset();
      omega = std::clamp(update_primal_weight(epoch_start, prev_start, omega, p.theta_smoothing,
                                              p.eps_zero),
                         p.omega_min, p.omega_max);
      e.omega_after = omega;
      result.restart_log.push_back(e);
      kkt_epoch_start = ev.cand_eval.residuals.weighted(omega);
      kkt_last = kkt_epoch_start;
    }
  }
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_solve(const pdlp_lp* lp, const pdlp_params* params, pdlp_result_info* info, double* x,
              double* y, double* lambda, double* lambda_pos, double* lambda_neg,
              pdlp_step_log_entry* step_log, int64_t step_cap, pdlp_restart_event* restart_log,
              int64_t restart_cap) {
  try {
    const GeneralFormLp g = to_lp(*lp);
    const SolveResult r = solve(g, to_params(*params));
    fill_info(r, g.num_variables(), g.num_constraints(), info);
    copy_out(r.point.primal, x);
    copy_out(r.point.dual, y);
    copy_out(r.reduced.lambda, lambda);
    copy_out(r.reduced.lambda_pos, lambda_pos);
    copy_out(r.reduced.lambda_neg, lambda_neg);
    copy_logs(r, step_log, step_cap, restart_log, restart_cap);
    return PDLP_OK;
  } catch (const std::invalid_argument& e) {
    return fail(PDLP_EINVAL, e.what());
  } catch (const std::exception& e) {
    return fail(PDLP_ERUNTIME, e.what());
  }
}

void* ref_begin(const pdlp_lp* lp, const pdlp_params* params, int32_t* status) {
  try {
    auto su = std::make_shared<Setup>();
    su->lp = to_lp(*lp);
    su->lp.validate();
    su->p = to_params(*params);
    su->p.validate();
    Session::prepare(*su);
    auto* s = new Session(std::move(su));
    s->begin();
    if (status) *status = s->finished ? static_cast<int32_t>(s->result.status) : PDLP_STATUS_RUNNING;
    return s;
  } catch (const std::exception& e) {
    fail(PDLP_EINVAL, e.what());
    return nullptr;
  }
}

int ref_run(void* h, int64_t n, int32_t* status) {
  auto* s = static_cast<Session*>(h);
  s->run(n);
  if (status) *status = s->finished ? static_cast<int32_t>(s->result.status) : PDLP_STATUS_RUNNING;
  return PDLP_OK;
}

int ref_get_iterate(void* h, double* x, double* y, double* kx, double* kty, int64_t* counters,
                    double* scalars) {
  auto* s = static_cast<Session*>(h);
  copy_out(s->current.primal, x);
  copy_out(s->current.dual, y);
  copy_out(s->kx, kx);
  copy_out(s->kty, kty);
  if (counters) {
    counters[0] = s->total;
    counters[1] = s->inner;
    counters[2] = s->outer;
    counters[3] = s->trials;
  }
  if (scalars) {
    scalars[0] = s->eta;
    scalars[1] = s->eta_hat;
    scalars[2] = s->omega;
    scalars[3] = s->avg_x.weight_sum();
  }
  return PDLP_OK;
}

int ref_result(void* h, pdlp_result_info* info, double* x, double* y, double* lambda,
               double* lambda_pos, double* lambda_neg, pdlp_step_log_entry* step_log,
               int64_t step_cap, pdlp_restart_event* restart_log, int64_t restart_cap) {
  auto* s = static_cast<Session*>(h);
  if (!s->finished) return fail(PDLP_ESTATE, "ref_result: not finished");
  fill_info(s->result, s->lp.num_variables(), s->lp.num_constraints(), info);
  info->trials = s->trials;
  copy_out(s->result.point.primal, x);
  copy_out(s->result.point.dual, y);
  copy_out(s->result.reduced.lambda, lambda);
  copy_out(s->result.reduced.lambda_pos, lambda_pos);
  copy_out(s->result.reduced.lambda_neg, lambda_neg);
  copy_logs(s->result, step_log, step_cap, restart_log, restart_cap);
  return PDLP_OK;
}

void ref_end(void* h) { delete static_cast<Session*>(h); }

// An independent copy of a session's iterate state sharing its read-only
// setup (bench.py's reference arm: one concurrent solve per host core).
void* ref_fork(void* h) {
  try {
    return new Session(*static_cast<const Session*>(h));
  } catch (const std::exception& e) {
    fail(PDLP_ERUNTIME, e.what());
    return nullptr;
  }
}

int ref_scaling(const pdlp_lp* lp, const pdlp_params* params, double* row_scale, double* col_scale) {
  try {
    const GeneralFormLp g = to_lp(*lp);
    const SolverParams p = to_params(*params);
    const DiagonalScaling s = make_scaling(vstack(g.inequality_matrix, g.equality_matrix), p.scaling,
                                           p.ruiz_iterations, p.pock_chambolle_alpha);
    copy_out(s.row_scale, row_scale);
    copy_out(s.col_scale, col_scale);
    return PDLP_OK;
  } catch (const std::exception& e) {
    return fail(PDLP_EINVAL, e.what());
  }
}

int ref_spmv(const pdlp_csr* a, const double* x, double* out) {
  try {
    const CsrMatrix m = to_csr(*a);
    spmv(m, std::span<const double>(x, m.num_cols), std::span<double>(out, m.num_rows));
    return PDLP_OK;
  } catch (const std::exception& e) {
    return fail(PDLP_EINVAL, e.what());
  }
}

int ref_spmv_transpose(const pdlp_csr* a, const double* y, double* out) {
  try {
    const CsrMatrix m = to_csr(*a);
    spmv_transpose(m, std::span<const double>(y, m.num_rows), std::span<double>(out, m.num_cols));
    return PDLP_OK;
  } catch (const std::exception& e) {
    return fail(PDLP_EINVAL, e.what());
  }
}

int ref_transpose(const pdlp_csr* a, int64_t* off, int64_t* col, double* val) {
  const CsrMatrix t = explicit_transpose(to_csr(*a));
  std::copy(t.row_offsets.begin(), t.row_offsets.end(), off);
  std::copy(t.col_indices.begin(), t.col_indices.end(), col);
  std::copy(t.values.begin(), t.values.end(), val);
  return PDLP_OK;
}

int ref_from_triplets(int64_t rows, int64_t cols, int64_t nt, const int64_t* tr, const int64_t* tc,
                      const double* tv, int64_t* off, int64_t* col, double* val, int64_t* nnz_out) {
  try {
    std::vector<Triplet> t(static_cast<size_t>(nt));
    for (int64_t i = 0; i < nt; ++i) t[i] = {tr[i], tc[i], tv[i]};
    const CsrMatrix m = CsrMatrix::from_triplets(rows, cols, t);
    std::copy(m.row_offsets.begin(), m.row_offsets.end(), off);
    std::copy(m.col_indices.begin(), m.col_indices.end(), col);
    std::copy(m.values.begin(), m.values.end(), val);
    *nnz_out = m.nnz();
    return PDLP_OK;
  } catch (const std::invalid_argument& e) {
    return fail(PDLP_EINVAL, e.what());
  }
}

int ref_check_termination(const pdlp_lp* lp, const double* x, const double* y, double eps,
                          double* out) {
  try {
    const GeneralFormLp g = to_lp(*lp);
    PrimalDualPoint z;
    z.primal.assign(x, x + g.num_variables());
    z.dual.assign(y, y + g.num_constraints());
    const ReducedCosts rc = reduced_costs(g, z.dual);
    const TerminationCheck c = check_termination(g, z, rc, eps, termination_norms(g));
    out[0] = c.terminated ? 1.0 : 0.0;
    out[1] = c.info.primal_residual_norm;
    out[2] = c.info.dual_residual_norm;
    out[3] = c.info.primal_objective_raw;
    out[4] = c.info.dual_objective_raw;
    return PDLP_OK;
  } catch (const std::exception& e) {
    return fail(PDLP_EINVAL, e.what());
  }
}

// pdhg_raw_step (solver.hpp:335-358) on to_saddle(lp), the unscaled saddle
// problem, from (x, y).
int ref_pdhg_raw_step(const pdlp_lp* lp, const double* x, const double* y, double tau, double sigma,
                      double* x_out, double* y_out) {
  try {
    const GeneralFormLp g = to_lp(*lp);
    const SaddleProblem sp = to_saddle(g);
    PrimalDualPoint z;
    z.primal.assign(x, x + g.num_variables());
    z.dual.assign(y, y + g.num_constraints());
    const PrimalDualPoint nx = pdhg_raw_step(z, tau, sigma, sp);
    std::copy(nx.primal.begin(), nx.primal.end(), x_out);
    std::copy(nx.dual.begin(), nx.dual.end(), y_out);
    return PDLP_OK;
  } catch (const std::exception& e) {
    return fail(PDLP_EINVAL, e.what());
  }
}

// MPS loading through the reference parser (fixture generation only).
// Two-phase: ref_mps_load parses and keeps the instance; ref_mps_sizes reports
// {n, m1, m2, nnzG, nnzA}; ref_mps_fill copies into caller buffers.
struct MpsHold {
  GeneralFormLp lp;
};

void* ref_mps_load(const char* path) {
  try {
    auto* h = new MpsHold;
    h->lp = read_mps_file(path);
    return h;
  } catch (const std::exception& e) {
    fail(PDLP_ERUNTIME, e.what());
    return nullptr;
  }
}

void ref_mps_sizes(void* hp, int64_t* sizes) {
  auto* h = static_cast<MpsHold*>(hp);
  sizes[0] = h->lp.num_variables();
  sizes[1] = h->lp.num_inequalities();
  sizes[2] = h->lp.num_equalities();
  sizes[3] = h->lp.inequality_matrix.nnz();
  sizes[4] = h->lp.equality_matrix.nnz();
}

void ref_mps_fill(void* hp, int64_t* g_off, int64_t* g_col, double* g_val, int64_t* a_off,
                  int64_t* a_col, double* a_val, double* c, double* hv, double* b, double* l,
                  double* u, double* c0) {
  auto* h = static_cast<MpsHold*>(hp);
  const GeneralFormLp& lp = h->lp;
  std::copy(lp.inequality_matrix.row_offsets.begin(), lp.inequality_matrix.row_offsets.end(), g_off);
  std::copy(lp.inequality_matrix.col_indices.begin(), lp.inequality_matrix.col_indices.end(), g_col);
  std::copy(lp.inequality_matrix.values.begin(), lp.inequality_matrix.values.end(), g_val);
  std::copy(lp.equality_matrix.row_offsets.begin(), lp.equality_matrix.row_offsets.end(), a_off);
  std::copy(lp.equality_matrix.col_indices.begin(), lp.equality_matrix.col_indices.end(), a_col);
  std::copy(lp.equality_matrix.values.begin(), lp.equality_matrix.values.end(), a_val);
  std::copy(lp.objective.begin(), lp.objective.end(), c);
  std::copy(lp.inequality_rhs.begin(), lp.inequality_rhs.end(), hv);
  std::copy(lp.equality_rhs.begin(), lp.equality_rhs.end(), b);
  std::copy(lp.lower.begin(), lp.lower.end(), l);
  std::copy(lp.upper.begin(), lp.upper.end(), u);
  *c0 = lp.objective_constant;
}

void ref_mps_free(void* hp) { delete static_cast<MpsHold*>(hp); }

// ---- benchmark harness (bench.hpp) ----
int ref_bench_config_hash(const pdlp_params* p, double time_limit, char* out17) {
  const std::string h = config_hash(to_params(*p), time_limit);
  std::snprintf(out17, 17, "%s", h.c_str());
  return 0;
}

int ref_bench_sgm(const double* t, int64_t n, double shift, double* out) {
  try {
    *out = shifted_geometric_mean(std::span<const double>(t, size_t(n)), shift);
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(PDLP_EINVAL, e.what());
  }
}

static int copy_text(const std::string& s, char* buf, int64_t cap, int64_t* len) {
  *len = int64_t(s.size());
  if (buf && cap > 0) std::snprintf(buf, size_t(cap), "%s", s.c_str());
  return int64_t(s.size()) < cap ? 0 : PDLP_EINVAL;
}

// write_report of records given column-wise (names '\n'-separated)
int ref_bench_report(int64_t n, const char* names, const int64_t* nnz, const int32_t* parse_failed,
                     const int32_t* status, const double* solve_s, const double* total_s, const int64_t* iters,
                     const double* obj, const double* gap, const double* rpr, const double* rdr,
                     const pdlp_params* p, double time_limit, char* buf, int64_t cap, int64_t* len) {
  BenchmarkReport rep;
  rep.config_line = config_hash(to_params(*p), time_limit);
  rep.time_limit = time_limit;
  std::istringstream ns(names);
  for (int64_t i = 0; i < n; ++i) {
    BenchmarkRecord r;
    std::getline(ns, r.instance);
    r.nonzeros = nnz[i];
    r.parse_failed = parse_failed[i] != 0;
    r.status = static_cast<SolveStatus>(status[i]);
    r.solve_seconds = solve_s[i];
    r.total_seconds = total_s[i];
    r.iterations = iters[i];
    r.primal_objective = obj[i];
    r.relative_gap = gap[i];
    r.relative_primal_residual = rpr[i];
    r.relative_dual_residual = rdr[i];
    rep.records.push_back(r);
  }
  rep.aggregates = aggregate_records(rep.records, time_limit);
  std::ostringstream out;
  write_report(rep, out);
  return copy_text(out.str(), buf, cap, len);
}

int ref_bench_run(const char* dir, const pdlp_params* p, double time_limit, int32_t jobs, char* buf,
                  int64_t cap, int64_t* len) {
  try {
    const BenchmarkReport rep = run_benchmark(dir, to_params(*p), time_limit, jobs);
    std::ostringstream out;
    write_report(rep, out);
    return copy_text(out.str(), buf, cap, len);
  } catch (const std::exception& e) {
    return fail(PDLP_ERUNTIME, e.what());
  }
}

// ---- standard-form theory harness (standard_form.hpp) ----
static StandardFormLp to_standard(const pdlp_csr* a, const double* b, const double* c) {
  StandardFormLp lp;
  lp.constraint_matrix = to_csr(*a);
  lp.rhs.assign(b, b + a->num_rows);
  lp.objective.assign(c, c + a->num_cols);
  return lp;
}

int ref_kkt_error_standard(const pdlp_csr* a, const double* b, const double* c, const double* x,
                           const double* y, double* out) {
  const StandardFormLp lp = to_standard(a, b, c);
  *out = kkt_error_standard(lp, std::span<const double>(x, size_t(a->num_cols)),
                            std::span<const double>(y, size_t(a->num_rows)));
  return 0;
}

int ref_spectral_norm(const pdlp_csr* a, double tol, int32_t max_iterations, double* out) {
  *out = spectral_norm(to_csr(*a), tol, max_iterations);
  return 0;
}

int ref_p_s_norm_squared(const pdlp_csr* a, const double* b, const double* c, double s, const double* x,
                         const double* y, double* out) {
  const StandardFormLp lp = to_standard(a, b, c);
  *out = p_s_norm_squared(lp, s, std::span<const double>(x, size_t(a->num_cols)),
                          std::span<const double>(y, size_t(a->num_rows)));
  return 0;
}

// restarted_pdhg_standard from z = 0 (or x0/y0 when given). Outputs: per epoch
// start KKT and length (up to `cap` epochs), counters[4] = {epochs,
// total_iterations, converged, numerical_failure}, the last epoch's start
// point (x_last, y_last), and with iter_x/iter_y the recorded iterates.
int ref_standard_pdhg(const pdlp_csr* a, const double* b, const double* c, double step, double decay,
                      double tol, int64_t iteration_limit, const double* x0, const double* y0,
                      double* start_kkt, int64_t* lengths, int64_t cap, int64_t* counters, double* x_last,
                      double* y_last, double* iter_x, double* iter_y, int64_t iter_cap) {
  try {
    const StandardFormLp lp = to_standard(a, b, c);
    StandardPdhgOptions o;
    o.step_size = step;
    o.restart_decay = decay;
    o.convergence_tol = tol;
    o.iteration_limit = iteration_limit;
    o.record_iterates = iter_x && iter_y && iter_cap > 0;
    PrimalDualPoint z0;
    if (x0 && y0) {
      z0.primal.assign(x0, x0 + a->num_cols);
      z0.dual.assign(y0, y0 + a->num_rows);
    }
    const StandardPdhgTrace t = restarted_pdhg_standard(lp, o, z0);
    const int64_t ne = int64_t(t.epochs.size());
    for (int64_t e = 0; e < ne && e < cap; ++e) {
      start_kkt[e] = t.epochs[size_t(e)].start_kkt;
      lengths[e] = t.epochs[size_t(e)].length;
    }
    counters[0] = ne;
    counters[1] = t.total_iterations;
    counters[2] = t.converged ? 1 : 0;
    counters[3] = t.numerical_failure ? 1 : 0;
    if (ne > 0) {
      copy_out(t.epochs.back().start.primal, x_last);
      copy_out(t.epochs.back().start.dual, y_last);
    }
    int64_t k = 0;
    for (const StandardEpoch& e : t.epochs)
      for (const PrimalDualPoint& z : e.iterates) {
        if (k >= iter_cap) break;
        std::copy(z.primal.begin(), z.primal.end(), iter_x + k * a->num_cols);
        std::copy(z.dual.begin(), z.dual.end(), iter_y + k * a->num_rows);
        ++k;
      }
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(PDLP_EINVAL, e.what());
  }
}

}  // extern "C"
