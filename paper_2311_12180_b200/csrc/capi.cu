// capi.cu — extern "C" boundary (include/pdlp_b200.h). Exceptions never cross
// it: std::invalid_argument -> PDLP_EINVAL (the reference's error type for bad
// input, lp_model.hpp:45-72 / solver.hpp:79-93), CUDA failures -> PDLP_ECUDA,
// everything else -> PDLP_ERUNTIME; the message is kept per thread.
#include <algorithm>
#include <cstring>
#include <vector>
#include <limits>
#include <string>

#include "../../include/pdlp_b200.h"
#include "solver.cuh"

struct pdlp_handle {
  pdlp::Solver* solver;
};

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return PDLP_OK;
  } catch (const pdlp::CudaError& e) {
    g_last_error = e.what();
    return PDLP_ECUDA;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return PDLP_EINVAL;
  } catch (const std::logic_error& e) {
    g_last_error = e.what();
    return PDLP_ESTATE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PDLP_ERUNTIME;
  } catch (...) {
    g_last_error = "unknown error";
    return PDLP_ERUNTIME;
  }
}

int null_handle() {
  g_last_error = "null handle";
  return PDLP_EINVAL;
}

}  // namespace

namespace pdlp {
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace pdlp

extern "C" {

int pdlp_abi_version(void) { return PDLP_ABI_VERSION; }

int pdlp_device_count(int32_t* count) {
  if (!count) return PDLP_EINVAL;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *count = n;
  return PDLP_OK;
}

void pdlp_default_params(pdlp_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof *p);
  p->eps_optimal = 1e-4;
  p->eps_infeasible = 1e-8;
  p->time_limit_seconds = 3600.0;
  p->iteration_limit = std::numeric_limits<int64_t>::max();
  p->beta_sufficient = 0.2;
  p->beta_necessary = 0.8;
  p->beta_artificial = 0.36;
  p->theta_smoothing = 0.5;
  p->eps_zero = 1e-10;
  p->evaluation_frequency = 64;
  p->scaling = PDLP_SCALING_RUIZ_PC;
  p->ruiz_iterations = 10;
  p->pock_chambolle_alpha = 1.0;
  p->step_reduction_exponent = 0.3;
  p->step_growth_exponent = 0.6;
  p->omega_min = 1e-8;
  p->omega_max = 1e8;
  p->record_step_log = 0;
  p->device = 0;
  p->mode = PDLP_MODE_FAST;
  p->use_cuda_graph = 1;
  p->l2_persist = 0;  /* opt-in: measured neutral on C2, -2% on C3 */
  p->engine = PDLP_ENGINE_AUTO;
  p->world_size = 1;
  p->rank = 0;
  p->plan_world = 0;
}

int pdlp_create(const pdlp_lp* lp, const pdlp_params* params, pdlp_handle** out) {
  if (!lp || !params || !out) {
    g_last_error = "null argument";
    return PDLP_EINVAL;
  }
  *out = nullptr;
  return guarded([&] {
    auto* h = new pdlp_handle{nullptr};
    try {
      h->solver = new pdlp::Solver(*lp, *params);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void pdlp_destroy(pdlp_handle* h) {
  if (!h) return;
  delete h->solver;
  delete h;
}

int pdlp_solve(pdlp_handle* h, pdlp_result_info* info) {
  if (!h) return null_handle();
  return guarded([&] { h->solver->solve(info); });
}

int pdlp_get_solution(pdlp_handle* h, double* x, double* y, double* lambda, double* lambda_pos,
                      double* lambda_neg) {
  if (!h) return null_handle();
  return guarded([&] { h->solver->get_solution(x, y, lambda, lambda_pos, lambda_neg); });
}

int pdlp_get_step_log(pdlp_handle* h, pdlp_step_log_entry* out, int64_t capacity) {
  if (!h) return null_handle();
  return guarded([&] { h->solver->get_step_log(out, capacity); });
}

int pdlp_get_restart_log(pdlp_handle* h, pdlp_restart_event* out, int64_t capacity) {
  if (!h) return null_handle();
  return guarded([&] { h->solver->get_restart_log(out, capacity); });
}

int pdlp_get_scaling(pdlp_handle* h, double* row_scale, double* col_scale) {
  if (!h) return null_handle();
  return guarded([&] { h->solver->get_scaling(row_scale, col_scale); });
}

int pdlp_spmv(pdlp_handle* h, int32_t op, const double* in, double* out) {
  if (!h) return null_handle();
  return guarded([&] { h->solver->spmv(op, in, out); });
}

int pdlp_iterate_begin(pdlp_handle* h, int32_t* status) {
  if (!h) return null_handle();
  return guarded([&] { h->solver->iterate_begin(status); });
}

int pdlp_iterate_run(pdlp_handle* h, int64_t n, int32_t* status) {
  if (!h) return null_handle();
  return guarded([&] { h->solver->iterate_run(n, status); });
}

int pdlp_get_iterate(pdlp_handle* h, double* x, double* y, double* kx, double* kty,
                     int64_t* counters, double* scalars) {
  if (!h) return null_handle();
  return guarded([&] { h->solver->get_iterate(x, y, kx, kty, counters, scalars); });
}

int pdlp_time_kernel(pdlp_handle* h, int32_t which, int32_t reps, double* avg_ms,
                     double* bytes_per_launch) {
  if (!h) return null_handle();
  return guarded([&] { h->solver->time_kernel(which, reps, avg_ms, bytes_per_launch); });
}

int pdlp_kernel_bytes(pdlp_handle* h, int32_t which, double* out) {
  if (!h) return null_handle();
  return guarded([&] {
    if (!out || which < 0 || which > 3) throw std::invalid_argument("pdlp_kernel_bytes: which must be 0..3");
    h->solver->kernel_bytes(which, out, out + 1);
    out[2] = double(h->solver->panels(which == 0 || which == 2 ? 0 : 1));
  });
}

int pdlp_get_sizes(pdlp_handle* h, int64_t* sizes) {
  if (!h) return null_handle();
  return guarded([&] { h->solver->sizes(sizes); });
}

const char* pdlp_last_error(void) { return g_last_error.c_str(); }

// ---- row sharding ------------------------------------------------------

int64_t pdlp_shard_blob_size(void) { return int64_t(sizeof(pdlp::ShardBlob)); }

int pdlp_shard_link_local(pdlp_handle** handles, int32_t world) {
  if (!handles || world < 1) {
    g_last_error = "null handles";
    return PDLP_EINVAL;
  }
  return guarded([&] {
    std::vector<pdlp::Solver*> ranks;
    for (int q = 0; q < world; ++q) {
      if (!handles[q]) throw std::invalid_argument("shard link: null handle");
      ranks.push_back(handles[q]->solver);
    }
    pdlp::Solver::link_local(ranks);
  });
}

int pdlp_shard_export(pdlp_handle* h, void* blob, int64_t capacity) {
  if (!h) return null_handle();
  if (!blob || capacity < int64_t(sizeof(pdlp::ShardBlob))) {
    g_last_error = "shard export: blob buffer too small";
    return PDLP_EINVAL;
  }
  return guarded([&] { h->solver->export_shard(static_cast<pdlp::ShardBlob*>(blob)); });
}

int pdlp_shard_import(pdlp_handle* h, const void* blobs, int32_t world) {
  if (!h) return null_handle();
  if (!blobs) {
    g_last_error = "null blobs";
    return PDLP_EINVAL;
  }
  return guarded([&] {
    if (world < 1 || world > pdlp::kMaxShards)
      throw std::invalid_argument("shards: world must lie in [1, " + std::to_string(pdlp::kMaxShards) + "]");
    std::vector<pdlp::ShardBlob> v(static_cast<size_t>(world));
    std::memcpy(v.data(), blobs, sizeof(pdlp::ShardBlob) * size_t(world));
    h->solver->import_shards(v.data(), world);
  });
}

int pdlp_shard_info(pdlp_handle* h, int64_t* out) {
  if (!h) return null_handle();
  if (!out) {
    g_last_error = "null output";
    return PDLP_EINVAL;
  }
  return guarded([&] { h->solver->shard_info(out); });
}

int pdlp_pdhg_raw_step(pdlp_handle* h, const double* x, const double* y, double tau, double sigma,
                       double* x_out, double* y_out) {
  if (!h) return null_handle();
  return guarded([&] {
    int64_t sz[4];
    h->solver->sizes(sz);
    if ((sz[0] && (!x || !x_out)) || (sz[1] && (!y || !y_out)))
      throw std::invalid_argument("pdhg_raw_step: null vector");
    h->solver->pdhg_raw_step(x, y, tau, sigma, x_out, y_out);
  });
}

int pdlp_shard_exchange(pdlp_handle* h, int64_t* out) {
  if (!h) return null_handle();
  if (!out) {
    g_last_error = "null output";
    return PDLP_EINVAL;
  }
  return guarded([&] { h->solver->shard_exchange(out); });
}

// Host-only twin of the device gather masks (kernels.cu shard_mask_kernel):
// bit q of xmask[c] = a row of K owned by rank q holds column c; bit q of
// ymask[r] = row r holds a column owned by rank q. Per rank, the x' / y'
// values it pushes per trial with the masks and with an all-to-all push.
int pdlp_plan_exchange(const pdlp_lp* lp, int32_t world, int64_t* pushed, int64_t* all_to_all, uint32_t* xmask,
                       uint32_t* ymask) {
  if (!lp || !pushed || !all_to_all) {
    g_last_error = "null argument";
    return PDLP_EINVAL;
  }
  return guarded([&] {
    std::vector<int64_t> kc(size_t(world) + 1), ktc(size_t(world) + 1);
    if (int rc = pdlp_plan_shards(lp, world, kc.data(), ktc.data()); rc != PDLP_OK)
      throw std::invalid_argument(g_last_error);
    const pdlp_csr& G = lp->inequality_matrix;
    const pdlp_csr& A = lp->equality_matrix;
    const int64_t m1 = G.num_rows, m2 = A.num_rows, n = lp->num_variables, m = m1 + m2;
    std::vector<uint32_t> xm(size_t(n), 0u), ym(size_t(m), 0u);
    auto owner = [](const std::vector<int64_t>& cuts, int64_t i) {
      return int(std::upper_bound(cuts.begin() + 1, cuts.end(), i) - cuts.begin() - 1);
    };
    int64_t r = 0;
    for (const pdlp_csr* c : {&G, &A})
      for (int64_t i = 0; i < c->num_rows; ++i, ++r) {
        const int pr = owner(kc, r);
        for (int64_t k = c->row_offsets[i]; k < c->row_offsets[i + 1]; ++k) {
          const int64_t j = c->col_indices ? c->col_indices[k] : c->col_indices32[k];
          xm[size_t(j)] |= 1u << pr;
          ym[size_t(r)] |= 1u << owner(ktc, j);
        }
      }
    for (int q = 0; q < world; ++q) {
      const uint32_t others = ((world >= 32 ? 0xffffffffu : ((1u << world) - 1u)) & ~(1u << q));
      int64_t a = 0;
      for (int64_t j = ktc[size_t(q)]; j < ktc[size_t(q) + 1]; ++j) a += __builtin_popcount(xm[size_t(j)] & others);
      for (int64_t i = kc[size_t(q)]; i < kc[size_t(q) + 1]; ++i) a += __builtin_popcount(ym[size_t(i)] & others);
      pushed[q] = a;
      all_to_all[q] = ((ktc[size_t(q) + 1] - ktc[size_t(q)]) + (kc[size_t(q) + 1] - kc[size_t(q)])) * (world - 1);
    }
    if (xmask) std::copy(xm.begin(), xm.end(), xmask);
    if (ymask) std::copy(ym.begin(), ym.end(), ymask);
  });
}

int pdlp_plan_shards(const pdlp_lp* lp, int32_t world, int64_t* k_cuts, int64_t* kt_cuts) {
  if (!lp || !k_cuts || !kt_cuts) {
    g_last_error = "null argument";
    return PDLP_EINVAL;
  }
  return guarded([&] {
    if (world < 1 || world > pdlp::kMaxShards)
      throw std::invalid_argument("shards: world must lie in [1, " + std::to_string(pdlp::kMaxShards) + "]");
    pdlp::validate_lp(*lp);
    // row offsets of K = vstack(G, A) and of K^T (column counts), on the host
    const pdlp_csr& G = lp->inequality_matrix;
    const pdlp_csr& A = lp->equality_matrix;
    const int64_t m1 = G.num_rows, m2 = A.num_rows, n = lp->num_variables;
    std::vector<int64_t> rp(size_t(m1 + m2 + 1), 0), rpt(size_t(n + 1), 0);
    for (int64_t i = 0; i <= m1; ++i) rp[size_t(i)] = G.row_offsets ? G.row_offsets[i] : 0;
    for (int64_t i = 1; i <= m2; ++i) rp[size_t(m1 + i)] = G.nnz + A.row_offsets[i];
    for (const pdlp_csr* c : {&G, &A})
      for (int64_t k = 0; k < c->nnz; ++k) {
        const int64_t j = c->col_indices ? c->col_indices[k] : c->col_indices32[k];
        if (j < 0 || j >= n) throw std::invalid_argument("csr: column index out of range");
        ++rpt[size_t(j) + 1];
      }
    for (int64_t j = 0; j < n; ++j) rpt[size_t(j) + 1] += rpt[size_t(j)];
    const auto kc = pdlp::shard_cuts<int64_t>(m1 + m2, rp.data(), world);
    const auto ktc = pdlp::shard_cuts<int64_t>(n, rpt.data(), world);
    std::copy(kc.begin(), kc.end(), k_cuts);
    std::copy(ktc.begin(), ktc.end(), kt_cuts);
  });
}

}  // extern "C"
