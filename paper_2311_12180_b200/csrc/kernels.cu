// kernels.cu — sm_100a kernels of the restarted-PDHG hot path.
//
// Reference routine each kernel replaces (paths relative to
// /root/reference/proj/include/pdhglp/):
//   dual_kernel     adaptive_step_cached trial: spmv(K, x') solver.hpp:409, the
//                   dual update :410-415, all_finite :417-420, dy^2/interaction
//                   :428-435, eta_bar / eta' / accept :436-466 (last CTA), plus the
//                   WeightedAverage weight bookkeeping (vector_ops.hpp:95-107).
//   primal_kernel   accept: spmv_transpose(K, y') :456 as a gather over the stored
//                   K^T, fused with avg_x/avg_y .add (solver.hpp:838-839) and the
//                   NEXT trial's primal update :404-408 and dx^2 :422-427;
//                   reject: the primal update alone for the shrunk step.
//   eval_*          evaluate_candidates (solver.hpp:705-739) for current + average
//                   and check_infeasibility's two rays (:581-590) in one pass over
//                   K and one over K^T, four points side by side.
//   setup kernels   from_triplets/explicit_transpose/vstack (sparse_matrix.hpp:57-200),
//                   ruiz/pock-chambolle/apply_scaling (scaling.hpp:32-170).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <utility>

#include "../../include/pdlp_b200.h"
#include "kernels.cuh"
#include "epilogues.cuh"
#include "spmv_engine.cuh"

namespace pdlp {

namespace {
int ceil_div(int64_t a, int64_t b) { return int((a + b - 1) / b); }
}  // namespace

// ===========================================================================
// Iteration: dual kernel
// ===========================================================================


// Sequential (reference-order) sums used by the parity mode's reductions.
__device__ double seq_sum(const double* v, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += __ldcg(v + i);
  return s;
}
__device__ double seq_sum_sq(const double* v, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) {
    const double a = __ldcg(v + i);
    s += a * a;
  }
  return s;
}

// Outcome of the step decision (adaptive_step_cached, solver.hpp:436-466).
constexpr int kHeadTab = 128;  // step factors staged at the primal head

struct Decision {
  int mode;  // kPAccept / kPRetry / kPNone
  int cont;  // run another trial in this window
  double eta;  // step size of the next trial
  double omega;
  double ratio;
  int first;
  int ix_cur, ix_trial, iy_cur, ikty_cur;
  int64_t trials;  // trials_total after this decision
};

// The decision from the reduced trial terms, on the pre-decision state `s`.
// `st` (may be null) receives the new state; `log` the accepted step.
__device__ Decision step_decision(const DevState& s, const DevIter& it, double dy2, double inter,
                                  double dx2, bool finite, double red_k, double gro_k,
                                  DevState* st) {
  Decision d;
  const double omega = s.omega, eta = s.eta;
  d.cont = 0;
  d.mode = kPNone;
  d.eta = eta;
  d.omega = omega;
  d.ratio = s.avg_ratio;
  d.first = s.avg_first;
  d.ix_cur = s.ix_cur, d.ix_trial = s.ix_trial, d.iy_cur = s.iy_cur, d.ikty_cur = s.ikty_cur;
  d.trials = s.trials_total + 1;
  int trials_in_step = s.trials_in_step + 1;
  if (st) {
    st->trials_total = d.trials;
    st->trials_in_step = trials_in_step;
  }
  if (!finite) {
    if (st) {
      st->failure = 1;
      st->p_mode = kPNone;
    }
    return d;
  }
  const double movement = omega * dx2 + dy2 / omega;  // solver.hpp:436
  const double ia = fabs(inter);
  const double eta_bar = ia > 0.0 ? movement / (2.0 * ia) : INFINITY;
  const double eta_next = smin(red_k * eta_bar, gro_k * eta);
  d.eta = eta_next;
  if (eta <= eta_bar) {  // accept
    const double w = s.wsum + eta;  // WeightedAverage::add
    d.first = (w == eta) ? 1 : 0;
    d.ratio = eta / w;
    d.mode = kPAccept;
    // rotate: prev <- cur <- trial <- old prev
    d.ix_cur = s.ix_trial, d.ix_trial = s.ix_prev;
    d.iy_cur = s.iy_trial;
    d.ikty_cur = 1 - s.ikty_cur;
    d.cont = s.window_accepts + 1 < s.window_target;
    if (st) {
      if (s.record_log) {
        pdlp_step_log_entry* log = reinterpret_cast<pdlp_step_log_entry*>(it.step_log);
        pdlp_step_log_entry e;
        e.step_counter = s.total + 1;
        e.omega = omega;
        e.eta_accepted = eta;
        e.eta_bar = eta_bar;
        e.eta_next = eta_next;
        e.movement_sq = movement;
        e.interaction = inter;
        log[s.window_accepts] = e;
      }
      st->eta_acc = eta;
      st->eta_bar = eta_bar;
      st->eta_next = eta_next;
      st->mov = movement;
      st->inter = inter;
      st->total = s.total + 1;
      st->inner = s.inner + 1;
      st->window_accepts = s.window_accepts + 1;
      st->wsum = w;
      st->avg_first = d.first;
      st->avg_ratio = d.ratio;
      st->ix_prev = s.ix_cur;
      st->ix_cur = d.ix_cur;
      st->ix_trial = d.ix_trial;
      st->iy_prev = s.iy_cur;
      st->iy_cur = d.iy_cur;
      st->iy_trial = s.iy_prev;
      st->ikx_cur = 1 - s.ikx_cur;
      st->ikty_cur = d.ikty_cur;
      st->eta = eta_next;
      st->trials_in_step = 0;
      st->accepted = 1;
      st->p_mode = kPAccept;
    }
  } else {  // reject: shrink the step
    const bool bad = !(eta_next > 0.0) || !isfinite(eta_next) || trials_in_step >= 80;
    d.mode = bad ? kPNone : kPRetry;
    d.cont = bad ? 0 : 1;
    if (st) {
      st->eta = eta_next;
      st->accepted = 0;
      st->failure = bad ? 1 : 0;
      st->p_mode = d.mode;
    }
  }
  return d;
}

// decide_sep == 2: the last dual CTA to finish sums the dual partials once and
// commits the step decision (same sums and order as every other placement).
__device__ __forceinline__ void dual_tail_decision(const DevIter& it, DevState* st,
                                                   cudaGraphConditionalHandle cond, int use_cond) {
  if (!grid_last_block(&st->ctr_dual, gridDim.x)) return;
  double dp[3];
  sum_partials<3, 0>(it.d_part, it.d_tiles, dp);
  if (threadIdx.x != 0) return;
  const DevState pre = *st;
  const int64_t ti = pre.total - pre.table_base;
  const double px0 = __ldcg(it.px_total), px1 = __ldcg(it.px_total + 1);
  const Decision d = step_decision(pre, it, dp[0], dp[1], px0, dp[2] == 0.0 && px1 == 0.0,
                                   it.red_tab[2 * ti], it.red_tab[2 * ti + 1], st);
  __threadfence();
  if (use_cond) cudaGraphSetConditional(cond, d.cont ? 1u : 0u);
}

// Dual side of a trial: K x' fused with the projected dual update and the dy^2 /
// interaction partials. In fast mode the step decision is taken at the head of
// the primal kernel (every primal CTA recomputes it from the same partials in
// the same order), so this kernel has no serial tail; CTA 0 snapshots the state
// the decision will start from. Parity mode keeps the decision here (last CTA),
// where the reference-order sequential sums run.
template <bool kSeq, bool kShard>
#ifndef PDLP_ITER_CTAS
#define PDLP_ITER_CTAS 4
#endif
__global__ void __launch_bounds__(kThreads, PDLP_ITER_CTAS) dual_kernel(DevCsr K, DevIter it,
                                                           cudaGraphConditionalHandle cond,
                                                           int use_cond) {
  extern __shared__ __align__(16) unsigned char smem[];
  // fast mode: CTA 0 is a helper (state snapshot, dx^2 of x') running beside
  // the tile CTAs 1..ntiles instead of delaying one of them
  const bool helper = !kSeq && blockIdx.x == 0;
  const int tile = K.tile0 + int(blockIdx.x) - (kSeq ? 0 : 1);  // global tile index
  const Tile t = K.tiles[helper ? K.tile0 : tile];
  if (!helper && it.prefetch) prefetch_tile(t, K.rp, K.col, K.val);
  griddep_wait();  // x' and the state come from the previous primal kernel
  DevState* st = it.st;
  // A failed or completed window parks the remaining (stream-engine) launches;
  // parking is decided from state that is identical on every rank.
  bool parked = st->failure || st->window_accepts >= st->window_target;
  if (kShard && !parked && !shard_wait(it.sync, it.world, kSyncPrimal)) {
    // a peer never published its x' slice: end the solve with a numerical error
    if (blockIdx.x == 0 && threadIdx.x == 0) st->failure = 1;
    parked = true;
  }
  if (helper) {
    if (threadIdx.x == 0) *it.snap = *st;
    // the primal partials of x' (the decision's dx^2) are reduced here, off the
    // critical path, so the decision at the primal head has one round trip
    double pp[2];
    sum_partials<2, 0>(it.p_part + size_t(st->trials_total & 1) * it.p_tiles * 2, it.p_tiles, pp);
    if (threadIdx.x == 0) {
      it.px_total[0] = pp[0];
      it.px_total[1] = pp[1];
    }
  }
  if (parked) {
    if (kSeq && blockIdx.x == 0 && threadIdx.x == 0) st->p_mode = kPNone;
    return;
  }
  if (helper) {
    if (kShard) {
      shard_signal(it.shv, it.sync, it.world, it.rank, kSyncDual);
      return;
    }
    if (it.decide_sep == 2) dual_tail_decision(it, st, cond, use_cond);
    return;
  }
  DualEpi<kSeq, false, kShard> epi;
  epi.xg = it.x[st->ix_trial];
  epi.y = it.y[st->iy_cur];
  epi.kx = it.kx[st->ikx_cur];
  epi.q = it.q;
  epi.yt = it.y[st->iy_trial];
  epi.kxt = it.kx[1 - st->ikx_cur];
  epi.seq_dy2 = it.seq_dy2;
  epi.seq_inter = it.seq_inter;
  epi.sigma = st->eta * st->omega;  // sigma = eta * omega, solver.hpp:402
  epi.m1 = it.m1;
  if (kShard) epi.push = PeerPush{it.shv->y_all, size_t(st->iy_trial) * it.m, it.world, it.rank, it.ymask};
  double red[3] = {0.0, 0.0, 0.0};
  const int role = run_tile<DualEpi<kSeq, false, kShard>, kSeq>(t, K.rp, K.col, K.val, epi, red,
                                                                K.chunk_part, K.chunk_ctr, smem);
  // the primal kernel's CTAs may start their prologue once every dual CTA is
  // past its tile (triggering earlier would let them take slots from our waves)
  griddep_launch_dependents();
  const PartialSlots ps = store_tile_partial<3, 0>(red, it.d_part, t, role, tile, it.d_tiles);
  if (kShard) {
    push_tile_partial<3, 0>(it.shv->d_part, it.world, it.rank, 0, ps, size_t(it.d_tiles), red);
    shard_signal(it.shv, it.sync, it.world, it.rank, kSyncDual);
    return;
  }
  if (!kSeq) {
    if (it.decide_sep == 2) dual_tail_decision(it, st, cond, use_cond);
    return;
  }

  // ---- parity mode: the decision in the last CTA, sums in reference order ----
  if (!grid_last_block(&st->ctr_dual, gridDim.x)) return;
  double dpart[3], ppart[2];
  sum_partials<3, 0>(it.d_part, it.d_tiles, dpart);
  sum_partials<2, 0>(it.p_part + size_t(st->trials_total & 1) * it.p_tiles * 2, it.p_tiles, ppart);
  if (threadIdx.x != 0) return;
  const double dx2 = seq_sum(it.seq_dx2, it.n);  // solver.hpp:422-435
  double dy2 = 0.0, inter = 0.0;
  for (int i = 0; i < it.m; ++i) {
    dy2 += __ldcg(it.seq_dy2 + i);
    inter += __ldcg(it.seq_inter + i);
  }
  const DevState pre = *st;
  const int64_t ti = pre.total - pre.table_base;
  const Decision d = step_decision(pre, it, dy2, inter, dx2, dpart[2] == 0.0 && ppart[1] == 0.0,
                                   it.red_tab[2 * ti], it.red_tab[2 * ti + 1], st);
  __threadfence();
  if (use_cond) cudaGraphSetConditional(cond, d.cont ? 1u : 0u);
}

// ---------------------------------------------------------------------------
// Chained windows: the evaluation block's decision (solver.cu evaluation_block,
// solver.hpp:843-892) with the host's exact arithmetic (IEEE sqrt and the same
// operation order, --fmad=false), so the device continues exactly when the
// host would have found nothing to do.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double chain_weighted(double prn, double drn, double pobj, double dobj, double omega) {
  const double pr = omega * prn, dr = drn / omega, g = dobj - pobj;  // KktHost::gap
  return sqrt(pr * pr + dr * dr + g * g);
}

__device__ __forceinline__ bool chain_terminated(double prn, double drn, double pobj, double dobj,
                                                 const ChainConsts& k) {
  if (!isfinite(prn) || !isfinite(drn) || !isfinite(pobj) || !isfinite(dobj)) return false;
  const double eps = k.eps_optimal;
  const bool gap_ok = fabs(dobj - pobj) <= eps * (1.0 + fabs(dobj) + fabs(pobj));
  const bool p_ok = prn <= eps * (1.0 + k.rhs_norm);
  const bool d_ok = drn <= eps * (1.0 + k.obj_norm);
  return gap_ok && p_ok && d_ok;
}

__global__ void chain_decide_kernel(DevState* st, const EvalOut* e, ChainConsts k,
                                    cudaGraphConditionalHandle outer, cudaGraphConditionalHandle inner) {
  if (threadIdx.x != 0) return;
  bool stop = st->failure != 0;
  double kkt_cand = 0.0;
  if (!stop) {
    const double w = st->omega;
    const double kc = chain_weighted(e->prn[0], e->drn[0], e->pobj[0], e->dobj[0], w);
    const double ka = chain_weighted(e->prn[1], e->drn[1], e->pobj[1], e->dobj[1], w);
    const int cand = !(kc < ka) ? 1 : 0;
    kkt_cand = cand ? ka : kc;
    stop = chain_terminated(e->prn[cand], e->drn[cand], e->pobj[cand], e->dobj[cand], k) ||
           chain_terminated(e->prn[1 - cand], e->drn[1 - cand], e->pobj[1 - cand], e->dobj[1 - cand], k);
    for (int r = 0; r < 2 && !stop; ++r) {
      const double yn = e->y_norm[r];
      if (yn > k.eps_zero && e->kty_resid[r] <= k.eps_infeasible * yn && e->ray_dobj[r] > k.eps_infeasible * yn)
        stop = true;
      const double xn = e->x_norm[r];
      if (!stop && xn > k.eps_zero) {
        const double tol = k.eps_infeasible * xn;
        if (e->ax_norm[r] <= tol && !(e->gx_negmax[r] > tol) && !(e->xl_negmax[r] > tol) &&
            !(e->xu_max[r] > tol) && e->cx[r] < -tol)
          stop = true;
      }
    }
    if (!stop) {  // should_restart: any criterion sends the evaluation to the host
      if (kkt_cand <= k.beta_sufficient * st->kkt_epoch_start)
        stop = true;
      else if (kkt_cand <= k.beta_necessary * st->kkt_epoch_start && kkt_cand > st->kkt_last)
        stop = true;
      else if (double(st->inner) >= k.beta_artificial * double(st->total))
        stop = true;
    }
  }
  if (stop) {
    st->chain_stop = 1;
    cudaGraphSetConditional(outer, 0u);
    return;
  }
  st->kkt_last = kkt_cand;
  st->chain_evals += 1;
  if (st->chain_left > 0 && st->total + k.freq <= k.iteration_limit) {
    st->chain_left -= 1;
    st->window_accepts = 0;
    st->window_target = k.freq;
    cudaGraphSetConditional(inner, 1u);
    cudaGraphSetConditional(outer, 1u);
  } else {
    st->chain_stop = 2;
    cudaGraphSetConditional(outer, 0u);
  }
}

// ===========================================================================
// Iteration: primal kernel
// ===========================================================================

// Primal side of a trial. mode_override >= 0 forces a branch (first trial of a
// solve: retry; after a restart: restart). Otherwise the fast mode takes the
// step decision first (all CTAs, CTA 0 commits it), parity mode reads it.
template <bool kSeq, bool kNonneg, bool kShard>
__global__ void __launch_bounds__(kThreads, PDLP_ITER_CTAS) primal_kernel(DevCsr KT, DevIter it, int mode_override,
                                                             cudaGraphConditionalHandle cond,
                                                             int use_cond) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Decision sd;
  const int bid = blockIdx.x;
  const int tile = KT.tile0 + bid;  // global tile index (CTAs >= ntiles: avg_y slices)
  if (bid < KT.ntiles && it.prefetch) {
    const Tile tp = KT.tiles[tile];
    prefetch_tile(tp, KT.rp, KT.col, KT.val);
  }
  griddep_wait();  // y' and the dual partials come from the dual kernel
  DevState* st = it.st;
  Decision d;
  if (mode_override >= 0 || kSeq || it.decide_sep) {
    // forced branch, or the decision was committed to the state already
    // (parity mode: the dual's last CTA; many tiles: decide_kernel)
    const DevState& s = *st;
    d.mode = mode_override >= 0 ? mode_override : s.p_mode;
    d.eta = s.eta;
    d.omega = s.omega;
    d.ratio = s.avg_ratio;
    d.first = s.avg_first;
    d.ix_cur = s.ix_cur, d.ix_trial = s.ix_trial, d.iy_cur = s.iy_cur, d.ikty_cur = s.ikty_cur;
    d.trials = s.trials_total;
  } else {
    // decision inputs, all issued as independent loads (one round trip): the
    // state snapshot the dual kernel ran on, the window's step-factor table,
    // the pre-reduced dx^2, and the dual partials (sharded: after every rank
    // published its partials)
    __shared__ DevState s_snap;
    __shared__ double s_tab[2][kHeadTab];
    __shared__ double s_px[2];
    __shared__ double s_dp[3];
    constexpr int kWords = int(sizeof(DevState) / sizeof(unsigned long long));
    const int tid = threadIdx.x;
    unsigned long long w = 0;
    if (tid < kWords) w = __ldcg(reinterpret_cast<const unsigned long long*>(it.snap) + tid);
    double tr = 0.0, tg = 0.0, px = 0.0;
    if (tid < kHeadTab) {
      tr = __ldcg(it.red_tab + 2 * tid);
      tg = __ldcg(it.red_tab + 2 * tid + 1);
    }
    if (tid < 2) px = __ldcg(it.px_total + tid);
    double dp[3];
    if (!kShard) sum_partials<3, 0>(it.d_part, it.d_tiles, dp);
    if (tid < kWords) reinterpret_cast<unsigned long long*>(&s_snap)[tid] = w;
    if (tid < kHeadTab) {
      s_tab[0][tid] = tr;
      s_tab[1][tid] = tg;
    }
    if (tid < 2) s_px[tid] = px;
    __syncthreads();
    bool parked = s_snap.failure || s_snap.window_accepts >= s_snap.window_target;
    if (kShard && !parked) {
      if (!shard_wait(it.sync, it.world, kSyncDual)) {
        if (bid == 0 && tid == 0) st->failure = 1;
        parked = true;
      } else {
        sum_partials<3, 0>(it.d_part, it.d_tiles, dp);
        if (tid == 0) s_dp[0] = dp[0], s_dp[1] = dp[1], s_dp[2] = dp[2];
        __syncthreads();
        dp[0] = s_dp[0], dp[1] = s_dp[1], dp[2] = s_dp[2];
      }
    }
    if (tid == 0) {
      const DevState& s = s_snap;
      if (parked) {
        sd.mode = kPNone;  // parked launch of a completed window (stream engine)
      } else {
        const bool commit = bid == 0;
        const int64_t ti = s.total - s.table_base;
        const double rk = ti < kHeadTab ? s_tab[0][ti] : it.red_tab[2 * ti];
        const double gk = ti < kHeadTab ? s_tab[1][ti] : it.red_tab[2 * ti + 1];
        sd = step_decision(s, it, dp[0], dp[1], s_px[0], dp[2] == 0.0 && s_px[1] == 0.0, rk, gk,
                           commit ? st : nullptr);
        if (commit) {
          __threadfence();
          if (use_cond) cudaGraphSetConditional(cond, sd.cont ? 1u : 0u);
        }
      }
    }
    __syncthreads();
    d = sd;
    if (d.mode == kPNone) return;
  }
  if (d.mode == kPNone) return;  // keep the partials of the last real trial
  double red[2] = {0.0, 0.0};
  int role = kRoleOwn;
  const double tau = d.eta / d.omega;  // tau = eta / omega, solver.hpp:401
  const PeerPush push{kShard ? it.shv->x_all : nullptr, size_t(d.ix_trial) * it.n, it.world, it.rank, it.xmask};
  if (bid >= KT.ntiles) {
    // avg_y .add (solver.hpp:839) on this CTA's slice of the own dual rows; no partial
    if (d.mode == kPAccept) {
      const int nb = it.avg_blocks, b = bid - KT.ntiles;
      const int rows = it.row1 - it.row0;
      const int per = (rows + nb - 1) / nb;
      const int i0 = it.row0 + b * per, i1 = min(it.row1, i0 + per);
      const double* yc = it.y[d.iy_cur];
      for (int i = i0 + threadIdx.x; i < i1; i += kThreads)
        it.avg_y[i] = d.first ? yc[i] : it.avg_y[i] + d.ratio * (yc[i] - it.avg_y[i]);
    }
    if (kShard) shard_signal(it.shv, it.sync, it.world, it.rank, kSyncPrimal);
    return;
  }
  const Tile t = KT.tiles[tile];
  // kty_lazy: an accepted step keeps no K'y'; a later rejected trial recomputes
  // it (the SpMV branch below, without the averages) before its x'
  const bool lazy_retry = !kSeq && it.kty_lazy && d.mode == kPRetry && mode_override < 0;
  if (d.mode == kPAccept || d.mode == kPRestart || lazy_retry) {
    const bool acc = d.mode == kPAccept;
    if (it.prefetch) {
      // the epilogue's contiguous operands of this tile's columns -> L2 while
      // the matrix and the gathers are in flight
      const int j0 = t.row0;
      const int j1 = t.kind == kTileChunk ? t.row0 + 1 : t.row1;
      for (int j = (j0 & ~15) + 16 * int(threadIdx.x); j < j1; j += 16 * kThreads) {
        prefetch_l2(it.x[d.ix_cur] + j);
        prefetch_l2(it.c + j);
        if (acc) prefetch_l2(it.avg_x + j);
        if (!kNonneg) {
          prefetch_l2(it.l + j);
          prefetch_l2(it.u + j);
        }
      }
    }
    PrimalEpi<kSeq, kNonneg, false, kShard> epi;
    epi.yg = it.y[d.iy_cur];
    epi.xc = it.x[d.ix_cur];
    epi.c = it.c;
    epi.l = it.l;
    epi.u = it.u;
    epi.kty_out = it.kty[d.ikty_cur];
    epi.xt = it.x[d.ix_trial];
    epi.avg_x = it.avg_x;
    epi.seq_dx2 = it.seq_dx2;
    epi.tau = tau;
    epi.ratio = d.ratio;
    epi.do_avg = acc;
    epi.avg_first = d.first;
    epi.store_kty = (acc && !kSeq && it.kty_lazy) ? 0 : 1;
    epi.push = push;
    role = run_tile<PrimalEpi<kSeq, kNonneg, false, kShard>, kSeq>(t, KT.rp, KT.col, KT.val, epi, red,
                                                                   KT.chunk_part, KT.chunk_ctr, smem);
  } else if (d.mode == kPRetry) {
    // x' for the shrunk step over this tile's columns (a split column is
    // handled by its first slice), so the partials keep the tile layout
    const int j0 = t.row0;
    const int j1 = t.kind == kTileChunk ? (t.part == 0 ? t.row0 + 1 : t.row0) : t.row1;
    const double* xc = it.x[d.ix_cur];
    const double* kty = it.kty[d.ikty_cur];
    double* xt = it.x[d.ix_trial];
    for (int j = j0 + threadIdx.x; j < j1; j += kThreads) {
      const double xa = xc[j];
      const double v = xa - tau * (it.c[j] - kty[j]);
      const double xn = kNonneg ? smax(v, 0.0) : clamp_box(v, it.l[j], it.u[j]);
      xt[j] = xn;
      if (kShard) push(j, xn);
      const double dd = (xn - xa) * (xn - xa);
      if (kSeq) it.seq_dx2[j] = dd;
      red[0] += dd;
      red[1] += isfinite(xn) ? 0.0 : 1.0;
    }
  }
  griddep_launch_dependents();
  // ping-pong by trial parity: the next decision reads these while this launch's
  // late CTAs may still be reading the previous ones
  const size_t half = size_t(d.trials & 1) * it.p_tiles * 2;
  const PartialSlots ps = store_tile_partial<2, 0>(red, it.p_part + half, t, role, tile, it.p_tiles);
  if (kShard) {
    push_tile_partial<2, 0>(it.shv->p_part, it.world, it.rank, half, ps, size_t(it.p_tiles), red);
    shard_signal(it.shv, it.sync, it.world, it.rank, kSyncPrimal);
  }
}

// Step decision as its own one-CTA kernel between the dual and the primal
// kernel, used when the operator has so many tiles that recomputing it in every
// primal CTA would cost more than a launch (sum_partials over all dual
// partials per CTA). Same sums in the same order as the primal-head variant,
// so both give bitwise identical decisions.
template <bool kShard>
__global__ void __launch_bounds__(kThreads) decide_kernel(DevIter it, cudaGraphConditionalHandle cond,
                                                          int use_cond) {
  griddep_wait();
  DevState* st = it.st;
  if (st->failure || st->window_accepts >= st->window_target) {
    if (threadIdx.x == 0) st->p_mode = kPNone;
    return;
  }
  if (kShard && !shard_wait(it.sync, it.world, kSyncDual)) {
    if (threadIdx.x == 0) {
      st->failure = 1;
      st->p_mode = kPNone;
      if (use_cond) cudaGraphSetConditional(cond, 0u);
    }
    return;
  }
  double dp[3];
  sum_partials<3, 0>(it.d_part, it.d_tiles, dp);
  griddep_launch_dependents();
  if (threadIdx.x != 0) return;
  const DevState pre = *st;
  const int64_t ti = pre.total - pre.table_base;
  const double px0 = __ldcg(it.px_total), px1 = __ldcg(it.px_total + 1);
  const Decision d = step_decision(pre, it, dp[0], dp[1], px0, dp[2] == 0.0 && px1 == 0.0,
                                   it.red_tab[2 * ti], it.red_tab[2 * ti + 1], st);
  __threadfence();
  if (use_cond) cudaGraphSetConditional(cond, d.cont ? 1u : 0u);
}

// ===========================================================================
// Plain SpMV (kernel parity API and restart products)
// ===========================================================================

struct MatvecEpi : EpiBase<MatvecEpi> {
  static constexpr int NP = 1, NA = 1, NR = 1;
  static constexpr bool kUniform = true;
  static constexpr TileGeom kGeom = kIterGeom;
  static constexpr bool kNeedCol = false;
  const double* __restrict__ x;
  double* __restrict__ out;
  __device__ __forceinline__ void gather(int c, double (&g)[1]) const { g[0] = __ldg(x + c); }
  __device__ __forceinline__ void add(double (&a)[1], const double (&p)[1], int) const { a[0] += p[0]; }
  __device__ __forceinline__ void row_done(int r, const double (&a)[1], double (&)[1]) const {
    out[r] = a[0];
  }
};

template <bool kSeq>
__global__ void __launch_bounds__(kThreads) spmv_kernel(DevCsr A, const double* val,
                                                        const double* x, double* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  MatvecEpi epi;
  epi.x = x;
  epi.out = out;
  double red[1] = {0.0};
  const Tile t = A.tiles[A.tile0 + blockIdx.x];
  run_tile<MatvecEpi, kSeq>(t, A.rp, A.col, val, epi, red, A.chunk_part, A.chunk_ctr, smem);
}

__global__ void zero_iterate_kernel(DevIter it) {
  const DevState* st = it.st;
  double* x = it.x[st->ix_cur];
  double* y = it.y[st->iy_cur];
  double* kx = it.kx[st->ikx_cur];
  double* kty = it.kty[st->ikty_cur];
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < it.n; j += stride) {
    x[j] = 0.0;
    kty[j] = 0.0;
    it.x_start[j] = 0.0;
    it.avg_x[j] = 0.0;
    it.x[st->ix_prev][j] = 0.0;
  }
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < it.m; i += stride) {
    y[i] = 0.0;
    kx[i] = 0.0;
    it.y_start[i] = 0.0;
    it.avg_y[i] = 0.0;
    it.y[st->iy_prev][i] = 0.0;
  }
}

// Restart block (solver.hpp:907-909): z_start = z = candidate (current or average).
__global__ void restart_copy_kernel(DevIter it, int from_avg) {
  const DevState* st = it.st;
  double* x = it.x[st->ix_cur];
  double* y = it.y[st->iy_cur];
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < it.n; j += stride) {
    const double v = from_avg ? it.avg_x[j] : x[j];
    x[j] = v;
    it.x_start[j] = v;
  }
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < it.m; i += stride) {
    const double v = from_avg ? it.avg_y[i] : y[i];
    y[i] = v;
    it.y_start[i] = v;
  }
}

// ===========================================================================
// Evaluation block
// ===========================================================================

// EV0: unscaled copies of the four points (unscale_point, scaling.hpp:174-184),
// and the restart displacement ||cand - z_start||^2 of both candidates.
constexpr int kEv0Items = 4;  // elements per thread per block pass

__global__ void __launch_bounds__(kThreads) eval_prep_kernel(DevIter it, DevEval ev, int xblocks) {
  // sharded: every rank evaluates the four points redundantly on full vectors,
  // once the peers' average slices arrived (push_avg_kernel)
  if (it.world > 1) shard_wait(it.sync, it.world, kSyncAvg);
  const DevState* st = it.st;
  const bool empty = st->wsum == 0.0;
  const double inv_t = st->inner > 0 ? 1.0 / double(st->inner) : 0.0;
  double red[4] = {0.0, 0.0, 0.0, 0.0};
  const int span = kThreads * kEv0Items;
  if (int(blockIdx.x) < xblocks) {
    const double* xc = it.x[st->ix_cur];
    const double* xp = it.x[st->ix_prev];
    const double* xa = empty ? xc : it.avg_x;
    const int j0 = blockIdx.x * span, j1 = min(it.n, j0 + span);
    for (int j = j0 + threadIdx.x; j < j1; j += kThreads) {
      const double d2 = ev.d2[j], c = xc[j], a = xa[j], s = it.x_start[j];
      double2* dst = reinterpret_cast<double2*>(ev.X4 + size_t(j) * 4);
      dst[0] = make_double2(c * d2, a * d2);
      dst[1] = make_double2((c - xp[j]) * d2, (inv_t * (c - s)) * d2);
      const double dc = c - s, da = a - s;
      red[0] += dc * dc;
      red[1] += da * da;
    }
  } else {
    const double* yc = it.y[st->iy_cur];
    const double* yp = it.y[st->iy_prev];
    const double* ya = empty ? yc : it.avg_y;
    const int b = blockIdx.x - xblocks;
    const int i0 = b * span, i1 = min(it.m, i0 + span);
    for (int i = i0 + threadIdx.x; i < i1; i += kThreads) {
      const double d1 = ev.d1[i], c = yc[i], a = ya[i], s = it.y_start[i];
      double r2 = (c - yp[i]) * d1;
      double r3 = (inv_t * (c - s)) * d1;
      if (i < it.m1) {  // certificate_from_ray projects the ray (solver.hpp:509-510)
        if (r2 < 0.0) r2 = 0.0;
        if (r3 < 0.0) r3 = 0.0;
      }
      double2* dst = reinterpret_cast<double2*>(ev.Y4 + size_t(i) * 4);
      dst[0] = make_double2(c * d1, a * d1);
      dst[1] = make_double2(r2, r3);
      const double dc = c - s, da = a - s;
      red[2] += dc * dc;
      red[3] += da * da;
    }
  }
  store_partial<4, 0>(red, ev.part0, blockIdx.x, ev.grid0);
}

// Sharded evaluation: this rank's slices of the averages to every peer (the
// iteration keeps averages rank-local; they are gathered once per window),
// and, when trials push only to the peers that gather a value (masks), its
// slices of the current and previous iterates, which the evaluation reads in
// full.
__global__ void push_avg_kernel(DevIter it) {
  const ShardView* v = it.shv;
  const DevState* st = it.st;
  const int stride = gridDim.x * blockDim.x;
  for (int j = it.col0 + blockIdx.x * blockDim.x + threadIdx.x; j < it.col1; j += stride) {
    push_peers(v->avg_x, it.world, it.rank, size_t(j), it.avg_x[j]);
    if (it.xmask) {
      push_peers(v->x_all, it.world, it.rank, size_t(st->ix_cur) * it.n + j, it.x[st->ix_cur][j]);
      push_peers(v->x_all, it.world, it.rank, size_t(st->ix_prev) * it.n + j, it.x[st->ix_prev][j]);
    }
  }
  for (int i = it.row0 + blockIdx.x * blockDim.x + threadIdx.x; i < it.row1; i += stride) {
    push_peers(v->avg_y, it.world, it.rank, size_t(i), it.avg_y[i]);
    if (it.ymask) {
      push_peers(v->y_all, it.world, it.rank, size_t(st->iy_cur) * it.m + i, it.y[st->iy_cur][i]);
      push_peers(v->y_all, it.world, it.rank, size_t(st->iy_prev) * it.m + i, it.y[st->iy_prev][i]);
    }
  }
  shard_signal(v, it.sync, it.world, it.rank, kSyncAvg);
}

// Gather masks: for every nonzero (r, c) of K, rank owner(r) reads x'[c] and
// rank owner_t(c) reads y'[r] (owners by the row cuts of K and of K^T).
__global__ void shard_mask_kernel(const int* rp, const int* col, int rows, const int64_t* kc, const int64_t* ktc,
                                  int world, unsigned* xmask, unsigned* ymask) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    int pr = 0;
    while (pr + 1 < world && r >= kc[pr + 1]) ++pr;
    unsigned ym = 0;
    for (int k = rp[r]; k < rp[r + 1]; ++k) {
      const int c = col[k];
      int pc = 0;
      while (pc + 1 < world && c >= ktc[pc + 1]) ++pc;
      atomicOr(xmask + c, 1u << pr);  // integer: order-free
      ym |= 1u << pc;
    }
    ymask[r] = ym;
  }
}

// Values this rank pushes per trial with the masks (out[0]) and without (out[1]).
__global__ void shard_volume_kernel(const unsigned* xmask, const unsigned* ymask, int col0, int col1, int row0,
                                    int row1, int world, int rank, unsigned long long* out) {
  unsigned long long a = 0, b = 0;
  const unsigned others = ((world >= 32 ? 0xffffffffu : ((1u << world) - 1u)) & ~(1u << rank));
  for (int j = col0 + blockIdx.x * blockDim.x + threadIdx.x; j < col1; j += gridDim.x * blockDim.x)
    a += __popc(xmask[j] & others), b += world - 1;
  for (int i = row0 + blockIdx.x * blockDim.x + threadIdx.x; i < row1; i += gridDim.x * blockDim.x)
    a += __popc(ymask[i] & others), b += world - 1;
  atomicAdd(out, a);
  atomicAdd(out + 1, b);
}


// Waits (on the device) until every rank published `kind`.
__global__ void shard_barrier_kernel(ShardSync* sync, int world, int kind) {
  shard_wait(sync, world, kind);
}

int eval_grid0(int n, int m) {
  const int span = kThreads * kEv0Items;
  return ceil_div(n, span) + ceil_div(m, span);
}

__device__ __forceinline__ void load4(const double* p, double (&g)[4]) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  g[0] = a.x;
  g[1] = a.y;
  g[2] = b.x;
  g[3] = b.y;
}

// EV1 over rows of the ORIGINAL (G; A): primal residuals (lp_model.hpp:202-218),
// q'y (lp_model.hpp:240-247), ray tests on Ax/Gx and ||y|| (solver.hpp:509-566).
// Reductions: [0..5] KKT slots (viol^2, eq^2, q'y) x2, [6..11] ray slots
// (|Ax|^2, |y|^2, q'y) x2; maxima [12..13]: max_i(-Gx_i) per ray.
template <bool kSeq>
struct Ev1Epi : EpiBase<Ev1Epi<kSeq>> {
  static constexpr int NP = 4, NA = 4, NR = 14;
  static constexpr TileGeom kGeom = kEvalGeom;
  static constexpr bool kNeedCol = false;
  const double* __restrict__ X4;
  const double* __restrict__ Y4;
  const double* __restrict__ q;
  double* __restrict__ seq_r;
  int m, m1;
  __device__ __forceinline__ void gather(int c, double (&g)[4]) const { load4(X4 + size_t(c) * 4, g); }
  __device__ __forceinline__ void add(double (&a)[4], const double (&p)[4], int) const {
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] += p[i];
  }
  __device__ __forceinline__ void row_done(int r, const double (&a)[4], double (&red)[14]) const {
    const double qr = q[r];
    if (r < m1) {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const double v = smax(qr - a[s], 0.0);  // [h - Gx]+
        red[s * 3 + 0] += v * v;
        if (kSeq) seq_r[size_t(s) * m + r] = v;
      }
#pragma unroll
      for (int s = 2; s < 4; ++s) {
        const double ng = -a[s];
        if (ng > red[12 + s - 2]) red[12 + s - 2] = ng;
      }
    } else {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const double v = a[s] + -1.0 * qr;  // Ax + (-1) b, axpy order
        red[s * 3 + 1] += v * v;
        if (kSeq) seq_r[size_t(s) * m + r] = v;
      }
#pragma unroll
      for (int s = 2; s < 4; ++s) {
        red[6 + (s - 2) * 3 + 0] += a[s] * a[s];
        if (kSeq) seq_r[size_t(s) * m + r] = a[s];
      }
    }
    double y[4];
    load4(Y4 + size_t(r) * 4, y);
    red[2] += qr * y[0];
    red[5] += qr * y[1];
    red[7] += y[2] * y[2];
    red[8] += qr * y[2];
    red[10] += y[3] * y[3];
    red[11] += qr * y[3];
  }
};

// EV2 over rows of the ORIGINAL K^T, G- and A-parts summed separately as
// dual_slack does (lp_model.hpp:179-190). Reductions: KKT slots (|c-K'y-lam|^2,
// c'x, lambda terms) x2 = [0..5]; ray slots (|K'y+lam|^2, lambda terms, |x|^2,
// c'x) x2 = [6..13]; maxima [14..17]: (max -x over finite l, max x over finite u)
// per ray.
template <bool kSeq>
struct Ev2Epi : EpiBase<Ev2Epi<kSeq>> {
  static constexpr int NP = 4, NA = 8, NR = 18;
  static constexpr bool kUniform = true;  // K^T rows are often uniform (C1, C2, C4)
  static constexpr TileGeom kGeom = kEvalGeom;
  static constexpr bool kNeedCol = true;
  const double* __restrict__ Y4;
  const double* __restrict__ X4;
  const double* __restrict__ c;
  const double* __restrict__ l;
  const double* __restrict__ u;
  double* __restrict__ lam;
  double* __restrict__ seq_d;
  int n, m1;
  int lam_slot;  // slot whose reduced costs are stored (-1: none; parity mode: all)
  PeerPush lam_push;  // sharded finish: the stored slot's reduced costs to every peer
  __device__ __forceinline__ void gather(int r, double (&g)[4]) const { load4(Y4 + size_t(r) * 4, g); }
  __device__ __forceinline__ void add(double (&a)[8], const double (&p)[4], int col) const {
    if (col < m1) {
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] += p[i];
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) a[4 + i] += p[i];
    }
  }
  __device__ __forceinline__ void row_done(int j, const double (&a)[8], double (&red)[18]) const {
    const double cj = c[j], lj = l[j], uj = u[j];
    double x[4];
    load4(X4 + size_t(j) * 4, x);
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const double slack = (cj + -1.0 * a[s]) + -1.0 * a[4 + s];
      const double lm = reduced_cost(slack, lj, uj);
      if (kSeq || s == lam_slot) {
        lam[size_t(s) * n + j] = lm;
        if (s == lam_slot && lam_push.world > 1) lam_push(s * n + j, lm);
      }
      const double dres = slack + -1.0 * lm;
      if (kSeq) seq_d[size_t(s) * n + j] = dres;
      red[s * 3 + 0] += dres * dres;
      red[s * 3 + 1] += cj * x[s];
      red[s * 3 + 2] += lambda_term(lm, lj, uj);
    }
#pragma unroll
    for (int s = 2; s < 4; ++s) {
      const double kty = a[s] + 1.0 * a[4 + s];
      const double lm = reduced_cost(-kty, lj, uj);
      if (kSeq || s == lam_slot) {
        lam[size_t(s) * n + j] = lm;
        if (s == lam_slot && lam_push.world > 1) lam_push(s * n + j, lm);
      }
      const double viol = kty + 1.0 * lm;
      if (kSeq) seq_d[size_t(s) * n + j] = viol;
      const int o = 6 + (s - 2) * 4;
      red[o + 0] += viol * viol;
      red[o + 1] += lambda_term(lm, lj, uj);
      red[o + 2] += x[s] * x[s];
      red[o + 3] += cj * x[s];
      const int mo = 14 + (s - 2) * 2;
      if (lj > -INFINITY && -x[s] > red[mo]) red[mo] = -x[s];
      if (uj < INFINITY && x[s] > red[mo + 1]) red[mo + 1] = x[s];
    }
  }
};

template <bool kSeq>
__global__ void __launch_bounds__(kThreads, 3) eval_rows_kernel(DevCsr K, DevEval ev, int m, int m1) {
  extern __shared__ __align__(16) unsigned char smem[];
  Ev1Epi<kSeq> epi;
  epi.X4 = ev.X4, epi.Y4 = ev.Y4, epi.q = ev.q, epi.seq_r = ev.seq_r, epi.m = m, epi.m1 = m1;
  double red[14];
#pragma unroll
  for (int i = 0; i < 14; ++i) red[i] = i < 12 ? 0.0 : -INFINITY;
  // one tile per CTA, one partial per (global) tile
  const int ti = K.tile0 + int(blockIdx.x);
  const Tile t = K.tiles[ti];
  const int role = run_tile<Ev1Epi<kSeq>, kSeq>(t, K.rp, K.col, K.val_orig, epi, red, K.chunk_part,
                                                K.chunk_ctr, smem);
  const PartialSlots ps = store_tile_partial<12, 2>(red, ev.part1, t, role, ti, ev.ev1_tiles);
  if (ev.world > 1) {
    push_tile_partial<12, 2>(ev.shv->part1, ev.world, ev.rank, 0, ps, size_t(ev.ev1_tiles), red);
    shard_signal(ev.shv, ev.sync, ev.world, ev.rank, kSyncEvRows);
  }
}

template <bool kSeq>
__global__ void __launch_bounds__(kThreads) eval_cols_kernel(DevCsr KT, DevEval ev, int n, int m1,
                                                             int lam_slot) {
  extern __shared__ __align__(16) unsigned char smem[];
  Ev2Epi<kSeq> epi;
  epi.Y4 = ev.Y4, epi.X4 = ev.X4, epi.c = ev.c, epi.l = ev.l, epi.u = ev.u, epi.lam = ev.lam;
  epi.seq_d = ev.seq_d, epi.n = n, epi.m1 = m1, epi.lam_slot = lam_slot;
  double red[18];
#pragma unroll
  for (int i = 0; i < 18; ++i) red[i] = i < 14 ? 0.0 : -INFINITY;
  epi.lam_push = PeerPush{ev.shv ? ev.shv->lam : nullptr, 0, ev.world, ev.rank};
  const int ti = KT.tile0 + int(blockIdx.x);
  const Tile t = KT.tiles[ti];
  const int role = run_tile<Ev2Epi<kSeq>, kSeq>(t, KT.rp, KT.col, KT.val_orig, epi, red, KT.chunk_part,
                                                KT.chunk_ctr, smem);
  const PartialSlots ps = store_tile_partial<14, 4>(red, ev.part2, t, role, ti, ev.ev2_tiles);
  if (ev.world > 1) {
    push_tile_partial<14, 4>(ev.shv->part2, ev.world, ev.rank, 0, ps, size_t(ev.ev2_tiles), red);
    shard_signal(ev.shv, ev.sync, ev.world, ev.rank, kSyncEvCols);
  }
}

// Parity-mode dual objective: the single sequential accumulator of
// dual_objective (lp_model.hpp:236-253) minus the constant.
__device__ double seq_dual_objective(const DevEval& ev, int slot, int n, int m) {
  double obj = ev.objective_constant;
  for (int i = 0; i < m; ++i) obj += ev.q[i] * ev.Y4[size_t(i) * 4 + slot];
  const double* lam = ev.lam + size_t(slot) * n;
  for (int j = 0; j < n; ++j) {
    const double v = lam[j];
    if (v > 0.0) obj += ev.l[j] * v;
    if (v < 0.0) obj -= ev.u[j] * -v;
  }
  return obj - ev.objective_constant;
}

// First level of the evaluation reductions: CTA g sums chunk g of each
// partial array (fixed chunks, so the order is fixed) into ev.stage
// ([36][kEvalReduceCtas], component-major).
__global__ void __launch_bounds__(kThreads) eval_reduce_kernel(DevEval ev) {
  if (ev.world > 1) {
    shard_wait(ev.sync, ev.world, kSyncEvRows);
    shard_wait(ev.sync, ev.world, kSyncEvCols);
  }
  const int g = blockIdx.x, G = gridDim.x;
  auto chunk = [&](int count, int& j0, int& j1) {
    const int per = (count + G - 1) / G;
    j0 = min(count, g * per);
    j1 = min(count, j0 + per);
  };
  int a, b;
  double p0[4], p1[14], p2[18];
  chunk(ev.grid0, a, b);
  sum_partials_range<4, 0>(ev.part0, ev.grid0, a, b, p0);
  chunk(ev.ev1_tiles, a, b);
  sum_partials_range<12, 2>(ev.part1, ev.ev1_tiles, a, b, p1);
  chunk(ev.ev2_tiles, a, b);
  sum_partials_range<14, 4>(ev.part2, ev.ev2_tiles, a, b, p2);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) ev.stage[i * G + g] = p0[i];
    for (int i = 0; i < 14; ++i) ev.stage[(4 + i) * G + g] = p1[i];
    for (int i = 0; i < 18; ++i) ev.stage[(18 + i) * G + g] = p2[i];
  }
}

template <bool kSeq>
__global__ void __launch_bounds__(kThreads) eval_final_kernel(DevEval ev, int grid1, int grid2,
                                                              int n, int m, int m1) {
  // the partial arrays were pre-reduced by kEvalReduceCtas CTAs of
  // eval_reduce_kernel (fixed chunks); sum their chunk results in order
  double p0[4], p1[14], p2[18];
  sum_partials<4, 0>(ev.stage, kEvalReduceCtas, p0);
  sum_partials<12, 2>(ev.stage + 4 * kEvalReduceCtas, kEvalReduceCtas, p1);
  sum_partials<14, 4>(ev.stage + 18 * kEvalReduceCtas, kEvalReduceCtas, p2);
  (void)grid1;
  (void)grid2;
  EvalOut* o = ev.out;
  const double c0 = ev.objective_constant;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      o->prn[s] = sqrt(p1[s * 3 + 1] + p1[s * 3 + 0]);  // sqrt(|eq|^2 + |viol|^2)
      o->drn[s] = sqrt(p2[s * 3 + 0]);
      o->pobj[s] = p2[s * 3 + 1];
      o->dobj[s] = ((c0 + p1[s * 3 + 2]) + p2[s * 3 + 2]) - c0;
    }
    for (int r = 0; r < 2; ++r) {
      o->ax_norm[r] = sqrt(p1[6 + r * 3 + 0]);
      o->y_norm[r] = sqrt(p1[6 + r * 3 + 1]);
      o->kty_resid[r] = sqrt(p2[6 + r * 4 + 0]);
      o->ray_dobj[r] = ((c0 + p1[6 + r * 3 + 2]) + p2[6 + r * 4 + 1]) - c0;
      o->x_norm[r] = sqrt(p2[6 + r * 4 + 2]);
      o->cx[r] = p2[6 + r * 4 + 3];
      o->gx_negmax[r] = p1[12 + r];
      o->xl_negmax[r] = p2[14 + r * 2];
      o->xu_max[r] = p2[14 + r * 2 + 1];
    }
    o->dx2[0] = p0[0];
    o->dx2[1] = p0[1];
    o->dy2[0] = p0[2];
    o->dy2[1] = p0[3];
  }
  if (!kSeq) return;
  __syncthreads();
  // Parity mode: every sum in the reference's sequential order, one thread per sum.
  const int t = threadIdx.x;
  if (t < 2) {  // primal residual of the KKT points
    const double* r = ev.seq_r + size_t(t) * m;
    double eq = 0.0, vi = 0.0;
    for (int i = m1; i < m; ++i) eq += r[i] * r[i];
    for (int i = 0; i < m1; ++i) vi += r[i] * r[i];
    o->prn[t] = sqrt(eq + vi);
  } else if (t < 4) {
    const int s = t - 2;
    o->drn[s] = sqrt(seq_sum_sq(ev.seq_d + size_t(s) * n, n));
  } else if (t < 6) {
    const int s = t - 4;
    double a = 0.0;
    for (int j = 0; j < n; ++j) a += ev.c[j] * ev.X4[size_t(j) * 4 + s];
    o->pobj[s] = a;
  } else if (t < 8) {
    o->dobj[t - 6] = seq_dual_objective(ev, t - 6, n, m);
  } else if (t < 10) {
    const int s = t - 8 + 2;
    double a = 0.0;
    for (int i = 0; i < m; ++i) a += ev.Y4[size_t(i) * 4 + s] * ev.Y4[size_t(i) * 4 + s];
    o->y_norm[s - 2] = sqrt(a);
  } else if (t < 12) {
    const int s = t - 10 + 2;
    o->kty_resid[s - 2] = sqrt(seq_sum_sq(ev.seq_d + size_t(s) * n, n));
  } else if (t < 14) {
    const int s = t - 12 + 2;
    o->ray_dobj[s - 2] = seq_dual_objective(ev, s, n, m);
  } else if (t < 16) {
    const int s = t - 14 + 2;
    double a = 0.0;
    for (int j = 0; j < n; ++j) a += ev.X4[size_t(j) * 4 + s] * ev.X4[size_t(j) * 4 + s];
    o->x_norm[s - 2] = sqrt(a);
  } else if (t < 18) {
    const int s = t - 16 + 2;
    const double* r = ev.seq_r + size_t(s) * m;
    double a = 0.0;
    for (int i = m1; i < m; ++i) a += r[i] * r[i];
    o->ax_norm[s - 2] = sqrt(a);
  } else if (t < 20) {
    const int s = t - 18 + 2;
    double a = 0.0;
    for (int j = 0; j < n; ++j) a += ev.c[j] * ev.X4[size_t(j) * 4 + s];
    o->cx[s - 2] = a;
  }
}

// Parity-mode restart displacement (update_primal_weight, solver.hpp:309-317).
__global__ void eval_seq_displacement_kernel(DevIter it, EvalOut* o) {
  const DevState* st = it.st;
  const bool empty = st->wsum == 0.0;
  const int t = threadIdx.x;
  if (t < 2) {
    const double* xc = it.x[st->ix_cur];
    const double* v = (t == 1 && !empty) ? it.avg_x : xc;
    double a = 0.0;
    for (int j = 0; j < it.n; ++j) {
      const double d = v[j] - it.x_start[j];
      a += d * d;
    }
    o->dx2[t] = a;
  } else if (t < 4) {
    const double* yc = it.y[st->iy_cur];
    const double* v = (t == 3 && !empty) ? it.avg_y : yc;
    double a = 0.0;
    for (int i = 0; i < it.m; ++i) {
      const double d = v[i] - it.y_start[i];
      a += d * d;
    }
    o->dy2[t - 2] = a;
  }
}

// reduced_costs(lp, 0) for a dual-infeasibility exit (solver.hpp:877): slack = c.
__global__ void reduced_of_objective_kernel(const double* c, const double* l, const double* u,
                                            int n, double* lam) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    lam[j] = reduced_cost((c[j] + -1.0 * 0.0) + -1.0 * 0.0, l[j], u[j]);
}

// ===========================================================================
// Setup kernels
// ===========================================================================

__global__ void build_rowptr_kernel(const int64_t* g_off, const int64_t* a_off, int64_t m1,
                                    int64_t m2, int64_t nnz_g, int* rp) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i <= m1 + m2; i += stride) {
    rp[i] = i <= m1 ? int(g_off[i]) : int(a_off[i - m1] + nnz_g);
  }
}

__global__ void narrow_cols_kernel(const int64_t* c64, int* c32, int64_t nnz, int n, int* err) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nnz; k += stride) {
    const int64_t v = c64[k];
    if (v < 0 || v >= n) atomicOr(err, 1);
    c32[k] = int(v);
  }
}

__global__ void check_cols_kernel(const int* c32, int64_t nnz, int n, int* err) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nnz; k += stride) {
    const int v = c32[k];
    if (v < 0 || v >= n) atomicOr(err, 1);
  }
}

// CSR invariants (sparse_matrix.hpp:29-34): nondecreasing offsets, strictly
// increasing columns within a row.
__global__ void check_rows_kernel(const int* rp, const int* col, int rows, int* err) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    const int a = rp[r], b = rp[r + 1];
    if (b < a) {
      atomicOr(err, 2);
      continue;
    }
    for (int k = a + 1; k < b; ++k)
      if (col[k] <= col[k - 1]) {
        atomicOr(err, 4);
        break;
      }
  }
}

__global__ void expand_rows_kernel(const int* rp, int rows, int* row_of) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
    for (int k = rp[r]; k < rp[r + 1]; ++k) row_of[k] = r;
}

__global__ void iota_kernel(int* p, int64_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += stride) p[k] = int(k);
}

__global__ void count_cols_kernel(const int* col, int64_t nnz, int* counts) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nnz; k += stride)
    atomicAdd(counts + col[k], 1);
}

__global__ void gather_transpose_kernel(const int* perm, const int* row_of, const double* val,
                                        int64_t nnz, int* col_t, double* val_t) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < nnz; k += stride) {
    const int p = perm[k];
    col_t[k] = row_of[p];
    val_t[k] = val[p];
  }
}

// Planner input: does row r have mostly consecutive columns (and more than
// min_len entries)? One warp per row.
__global__ void row_contig_kernel(const int* rp, const int* col, int rows, int min_len,
                                  int want_contig, unsigned char* out) {
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= rows) return;
  const int k0 = rp[w], k1 = rp[w + 1];
  int cnt = 0;
  if (k1 - k0 > min_len)
    for (int k = k0 + lane; k + 1 < k1; k += 32) cnt += (col[k + 1] == col[k] + 1) ? 1 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  int flag = (k1 - k0 > min_len && 2 * cnt >= k1 - k0 - 1) ? 1 : 0;
  if (!want_contig) flag = 0;
  // 2: first row of four column-shifted rows (row w + i = row w's columns + i)
  // (only for rows long enough to give each of the group's 64 lanes per row
  // several elements; short shifted rows stay in ordinary WARP tiles)
  if ((w & 3) == 0 && w + 3 < rows && k1 - k0 >= 256) {
    const int L = k1 - k0;
    bool ok = rp[w + 4] - rp[w + 3] == L && rp[w + 3] - rp[w + 2] == L && rp[w + 2] - rp[w + 1] == L;
    if (ok) {
      int bad = 0;
      for (int i = 1; i < 4; ++i)
        for (int k = lane; k < L; k += 32) bad |= col[k0 + i * L + k] != col[k0 + k] + i;
      ok = __any_sync(0xffffffffu, bad) == 0;
    }
    if (ok) flag = 2;
  }
  if (lane == 0) out[w] = (unsigned char)flag;
}

__global__ void extract_slot_kernel(const double* v4, int slot, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = v4[i * 4 + slot];
}

__global__ void fill_kernel(double* p, int64_t n, double v) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += stride) p[k] = v;
}

__global__ void fill_int_kernel(int* p, int64_t n, int v) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += stride) p[k] = v;
}

// One warp per row: max |v * (d_self[r] * d_other[col])| (order-free, exact).
// Short rows: one thread per row (max is order-free, so any assignment gives
// the same bits).
__global__ void row_absmax_thread_kernel(const int* rp, const int* col, const double* val, int rows,
                                         const double* d_self, const double* d_other, double* out) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    const double dr = d_self[r];
    double mx = 0.0;
    for (int k = rp[r]; k < rp[r + 1]; ++k) mx = smax(mx, fabs(val[k] * (dr * d_other[col[k]])));
    out[r] = mx;
  }
}

__global__ void row_absmax_kernel(const int* rp, const int* col, const double* val, int rows,
                                  const double* d_self, const double* d_other, double* out) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int r = warp; r < rows; r += nwarps) {
    const double dr = d_self[r];
    double mx = 0.0;
    for (int k = rp[r] + lane; k < rp[r + 1]; k += 32) {
      // scaled_copy multiplies v *= dr * dc (scaling.hpp:38-40)
      const double a = fabs(val[k] * (dr * d_other[col[k]]));
      mx = smax(mx, a);
    }
    mx = warp_max(mx);
    if (lane == 0) out[r] = mx;
  }
}

// Thread per row, sequential in index order (row_norms / col_norms accumulate
// in that order, sparse_matrix.hpp:214-248), then the p-norm root.
__global__ void row_pnorm_kernel(const int* rp, const int* col, const double* val, int rows,
                                 const double* d_self, const double* d_other, double p,
                                 double* out) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    const double dr = d_self[r];
    double acc = 0.0;
    for (int k = rp[r]; k < rp[r + 1]; ++k) {
      const double a = fabs(val[k] * (dr * d_other[col[k]]));
      if (p == 0.0)
        acc += 1.0;
      else if (p == 1.0)
        acc += a;  // pow(a, 1.0) == a exactly
      else
        acc += pow(a, p);
    }
    if (p != 0.0 && p != 1.0 && acc > 0.0) acc = pow(acc, 1.0 / p);
    out[r] = acc;
  }
}

__global__ void ruiz_update_kernel(double* d, const double* norm, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double v = norm[i];
    if (v > 0.0) d[i] /= sqrt(v);
  }
}

// pock_chambolle_scale + compose (scaling.hpp:83-111): d *= 1/sqrt(sum^p).
__global__ void pc_update_kernel(double* d, const double* sum, int n, double p) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = sum[i];
    if (p != 0.0 && p != 1.0 && s > 0.0) s = pow(s, p);
    const double pc = s > 0.0 ? 1.0 / sqrt(s) : 1.0;
    d[i] *= pc;
  }
}

__global__ void scale_values_kernel(const int* rp, const int* col, const double* val, int rows,
                                    const double* d_self, const double* d_other, double* out) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int r = warp; r < rows; r += nwarps) {
    const double dr = d_self[r];
    for (int k = rp[r] + lane; k < rp[r + 1]; k += 32) out[k] = val[k] * (dr * d_other[col[k]]);
  }
}

// apply_scaling on the vectors (scaling.hpp:158-168).
__global__ void scale_vectors_kernel(const double* c, const double* l, const double* u,
                                     const double* q, const double* d1, const double* d2, int n,
                                     int m, double* cs, double* ls, double* us, double* qs) {
  const int stride = gridDim.x * blockDim.x;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    const double s = d2[j];
    cs[j] = c[j] * s;
    ls[j] = isfinite(l[j]) ? l[j] / s : l[j];
    us[j] = isfinite(u[j]) ? u[j] / s : u[j];
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) qs[i] = q[i] * d1[i];
}

__global__ void block_absmax_kernel(const double* v, int64_t n, double* partials) {
  __shared__ double sred[kWarps];
  double mx = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += stride)
    mx = smax(mx, fabs(v[k]));
  double a[1] = {mx};
  block_reduce<0, 1>(a, sred);
  if (threadIdx.x == 0) partials[blockIdx.x] = a[0];
}

// ===========================================================================
// Launchers
// ===========================================================================

namespace {
int grid_for(int64_t n, int per = kThreads) {
  int64_t g = (n + per - 1) / per;
  if (g < 1) g = 1;
  if (g > 148 * 16) g = 148 * 16;
  return int(g);
}
}  // namespace

void set_kernel_attributes() {
  // once per device (function attributes are per device), from any thread
  static std::mutex mu;
  static unsigned long long done = 0;
  int dev = 0;
  PDLP_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> g(mu);
    if (dev < 64 && (done >> dev) & 1ull) return;
    if (dev < 64) done |= 1ull << dev;
  }
  auto big = [](const void* f, size_t bytes) {
    PDLP_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
  };
  big((const void*)eval_rows_kernel<false>, stream_smem_bytes<Ev1Epi<false>>());
  big((const void*)eval_rows_kernel<true>, stream_smem_bytes<Ev1Epi<true>>());
  big((const void*)eval_cols_kernel<false>, stream_smem_bytes<Ev2Epi<false>>());
  big((const void*)eval_cols_kernel<true>, stream_smem_bytes<Ev2Epi<true>>());
  panel_kernel_attributes();
}

void launch_build_rowptr(const int64_t* g_off, const int64_t* a_off, int64_t m1, int64_t m2,
                         int64_t nnz_g, int* rp, cudaStream_t s) {
  build_rowptr_kernel<<<grid_for(m1 + m2 + 1), kThreads, 0, s>>>(g_off, a_off, m1, m2, nnz_g, rp);
  PDLP_CUDA(cudaGetLastError());
}
void launch_narrow_cols(const int64_t* col64, int* col32, int64_t nnz, int n, int* err,
                        cudaStream_t s) {
  narrow_cols_kernel<<<grid_for(nnz), kThreads, 0, s>>>(col64, col32, nnz, n, err);
  PDLP_CUDA(cudaGetLastError());
}
void launch_check_cols(const int* col32, int64_t nnz, int n, int* err, cudaStream_t s) {
  check_cols_kernel<<<grid_for(nnz), kThreads, 0, s>>>(col32, nnz, n, err);
  PDLP_CUDA(cudaGetLastError());
}
void launch_check_rows(const int* rp, const int* col, int rows, int* err, cudaStream_t s) {
  check_rows_kernel<<<grid_for(rows), kThreads, 0, s>>>(rp, col, rows, err);
  PDLP_CUDA(cudaGetLastError());
}
void launch_expand_rows(const int* rp, int rows, int* row_of, cudaStream_t s) {
  expand_rows_kernel<<<grid_for(rows), kThreads, 0, s>>>(rp, rows, row_of);
  PDLP_CUDA(cudaGetLastError());
}
void launch_iota(int* p, int64_t n, cudaStream_t s) {
  iota_kernel<<<grid_for(n), kThreads, 0, s>>>(p, n);
  PDLP_CUDA(cudaGetLastError());
}
void launch_count_cols(const int* col, int64_t nnz, int* counts, cudaStream_t s) {
  count_cols_kernel<<<grid_for(nnz), kThreads, 0, s>>>(col, nnz, counts);
  PDLP_CUDA(cudaGetLastError());
}
void launch_gather_transpose(const int* perm, const int* row_of, const double* val, int64_t nnz,
                             int* col_t, double* val_t, cudaStream_t s) {
  gather_transpose_kernel<<<grid_for(nnz), kThreads, 0, s>>>(perm, row_of, val, nnz, col_t, val_t);
  PDLP_CUDA(cudaGetLastError());
}
void launch_row_contig(const int* rp, const int* col, int rows, int min_len, int want_contig,
                       unsigned char* out, cudaStream_t s) {
  const int64_t threads = int64_t(rows) * 32;
  const int64_t grid = (threads + kThreads - 1) / kThreads;
  if (grid > 0)
    row_contig_kernel<<<unsigned(grid), kThreads, 0, s>>>(rp, col, rows, min_len, want_contig, out);
  PDLP_CUDA(cudaGetLastError());
}
void launch_extract_slot(const double* v4, int slot, int64_t n, double* out, cudaStream_t s) {
  extract_slot_kernel<<<grid_for(n), kThreads, 0, s>>>(v4, slot, n, out);
  PDLP_CUDA(cudaGetLastError());
}
void launch_fill(double* p, int64_t n, double v, cudaStream_t s) {
  fill_kernel<<<grid_for(n), kThreads, 0, s>>>(p, n, v);
  PDLP_CUDA(cudaGetLastError());
}
void launch_fill_int(int* p, int64_t n, int v, cudaStream_t s) {
  fill_int_kernel<<<grid_for(n), kThreads, 0, s>>>(p, n, v);
  PDLP_CUDA(cudaGetLastError());
}
void launch_row_absmax(const int* rp, const int* col, const double* val, int rows,
                       const double* d_self, const double* d_other, double* out, cudaStream_t s,
                       double avg_len) {
  if (avg_len <= 8.0)
    row_absmax_thread_kernel<<<grid_for(rows), kThreads, 0, s>>>(rp, col, val, rows, d_self, d_other, out);
  else
    row_absmax_kernel<<<grid_for(int64_t(rows) * 32), kThreads, 0, s>>>(rp, col, val, rows, d_self,
                                                                       d_other, out);
  PDLP_CUDA(cudaGetLastError());
}
void launch_row_pnorm(const int* rp, const int* col, const double* val, int rows,
                      const double* d_self, const double* d_other, double p, double* out,
                      cudaStream_t s) {
  row_pnorm_kernel<<<grid_for(rows, 128), 128, 0, s>>>(rp, col, val, rows, d_self, d_other, p, out);
  PDLP_CUDA(cudaGetLastError());
}
void launch_ruiz_update(double* d, const double* norm, int n, cudaStream_t s) {
  ruiz_update_kernel<<<grid_for(n), kThreads, 0, s>>>(d, norm, n);
  PDLP_CUDA(cudaGetLastError());
}
void launch_pc_update(double* d, const double* sum, int n, double p, cudaStream_t s) {
  pc_update_kernel<<<grid_for(n), kThreads, 0, s>>>(d, sum, n, p);
  PDLP_CUDA(cudaGetLastError());
}
void launch_scale_values(const int* rp, const int* col, const double* val_orig, int rows,
                         const double* d_self, const double* d_other, double* val_out,
                         cudaStream_t s) {
  scale_values_kernel<<<grid_for(int64_t(rows) * 32), kThreads, 0, s>>>(rp, col, val_orig, rows,
                                                                       d_self, d_other, val_out);
  PDLP_CUDA(cudaGetLastError());
}
void launch_scale_vectors(const double* c, const double* l, const double* u, const double* q,
                          const double* d1, const double* d2, int n, int m, double* cs,
                          double* ls, double* us, double* qs, cudaStream_t s) {
  scale_vectors_kernel<<<grid_for(n > m ? n : m), kThreads, 0, s>>>(c, l, u, q, d1, d2, n, m, cs, ls,
                                                                   us, qs);
  PDLP_CUDA(cudaGetLastError());
}
void launch_block_absmax(const double* v, int64_t n, double* partials, int nblocks,
                         cudaStream_t s) {
  block_absmax_kernel<<<nblocks, kThreads, 0, s>>>(v, n, partials);
  PDLP_CUDA(cudaGetLastError());
}

void launch_spmv(const DevCsr& a, bool orig_vals, const double* x, double* out, bool seq,
                 cudaStream_t s) {
  if (a.ntiles == 0) return;
  const size_t sm = stream_smem_bytes<MatvecEpi>();
  const double* val = orig_vals ? a.val_orig : a.val;
  if (seq)
    spmv_kernel<true><<<a.ntiles, kThreads, sm, s>>>(a, val, x, out);
  else
    spmv_kernel<false><<<a.ntiles, kThreads, sm, s>>>(a, val, x, out);
  PDLP_CUDA(cudaGetLastError());
}

namespace {
// Launch with programmatic stream serialization (PDL): the kernel may begin
// its static-data prologue while the previous kernel in the stream drains.
template <class... P, class... A>
void launch_pdl(void (*kern)(P...), int grid, size_t smem, cudaStream_t s, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  static const bool no_pdl = std::getenv("PDLP_NO_PDL") != nullptr;  // diagnostics
  cfg.attrs = attr;
  cfg.numAttrs = no_pdl ? 0 : 1;
  PDLP_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...));
}
}  // namespace

void launch_dual(const DevCsr& k, const DevIter& it, bool seq, unsigned long long cond,
                 int use_cond, cudaStream_t s) {
  const size_t sm = stream_smem_bytes<DualEpi<false>>();
  cudaGraphConditionalHandle h = static_cast<cudaGraphConditionalHandle>(cond);
  if (seq)
    launch_pdl(dual_kernel<true, false>, k.ntiles, sm, s, k, it, h, use_cond);
  else if (it.world > 1)
    launch_pdl(dual_kernel<false, true>, k.ntiles + 1, sm, s, k, it, h, use_cond);
  else
    launch_pdl(dual_kernel<false, false>, k.ntiles + 1, sm, s, k, it, h, use_cond);
}

void launch_decide(const DevIter& it, cudaStream_t s, unsigned long long cond, int use_cond) {
  cudaGraphConditionalHandle h = static_cast<cudaGraphConditionalHandle>(cond);
  if (it.world > 1)
    launch_pdl(decide_kernel<true>, 1, 0, s, it, h, use_cond);
  else
    launch_pdl(decide_kernel<false>, 1, 0, s, it, h, use_cond);
}

void launch_primal(const DevCsr& kt, const DevIter& it, bool seq, int mode_override,
                   cudaStream_t s, unsigned long long cond, int use_cond) {
  cudaGraphConditionalHandle h = static_cast<cudaGraphConditionalHandle>(cond);
  const size_t sm = stream_smem_bytes<PrimalEpi<false, false>>();
  if (seq) {
    if (it.nonneg)
      launch_pdl(primal_kernel<true, true, false>, it.p_grid, sm, s, kt, it, mode_override, h, use_cond);
    else
      launch_pdl(primal_kernel<true, false, false>, it.p_grid, sm, s, kt, it, mode_override, h, use_cond);
  } else if (it.world > 1) {
    if (it.nonneg)
      launch_pdl(primal_kernel<false, true, true>, it.p_grid, sm, s, kt, it, mode_override, h, use_cond);
    else
      launch_pdl(primal_kernel<false, false, true>, it.p_grid, sm, s, kt, it, mode_override, h, use_cond);
  } else {
    if (it.nonneg)
      launch_pdl(primal_kernel<false, true, false>, it.p_grid, sm, s, kt, it, mode_override, h, use_cond);
    else
      launch_pdl(primal_kernel<false, false, false>, it.p_grid, sm, s, kt, it, mode_override, h, use_cond);
  }
}

void launch_zero_iterate(const DevIter& it, cudaStream_t s) {
  zero_iterate_kernel<<<grid_for(it.n > it.m ? it.n : it.m), kThreads, 0, s>>>(it);
  PDLP_CUDA(cudaGetLastError());
}

void launch_restart_copy(const DevIter& it, int from_avg, cudaStream_t s) {
  restart_copy_kernel<<<grid_for(it.n > it.m ? it.n : it.m), kThreads, 0, s>>>(it, from_avg);
  PDLP_CUDA(cudaGetLastError());
}

int eval_grid(int ntiles) { return ntiles; }  // one tile per CTA: short latency chains

void launch_eval(const DevCsr& k, const DevCsr& kt, const DevIter& it, const DevEval& ev, bool seq,
                 cudaStream_t s, const PhaseFn& phase, const EvalFork* fork) {
  const int span = kThreads * kEv0Items;
  const int xblocks = ceil_div(it.n, span);
  if (it.world > 1) {  // the average slices to every rank, then the redundant EV0
    push_avg_kernel<<<grid_for(std::max(it.col1 - it.col0, it.row1 - it.row0)), kThreads, 0, s>>>(it);
    PDLP_CUDA(cudaGetLastError());
    if (phase) phase();
  }
  eval_prep_kernel<<<ev.grid0, kThreads, 0, s>>>(it, ev, xblocks);
  PDLP_CUDA(cudaGetLastError());
  const size_t sm1 = stream_smem_bytes<Ev1Epi<false>>();
  const size_t sm2 = stream_smem_bytes<Ev2Epi<false>>();
  const int g1 = eval_grid(k.ntiles), g2 = eval_grid(kt.ntiles);
  if (seq) {
    eval_rows_kernel<true><<<g1, kThreads, sm1, s>>>(k, ev, it.m, it.m1);
    eval_cols_kernel<true><<<g2, kThreads, sm2, s>>>(kt, ev, it.n, it.m1, -1);
    eval_reduce_kernel<<<kEvalReduceCtas, kThreads, 0, s>>>(ev);
    eval_final_kernel<true><<<1, kThreads, 0, s>>>(ev, ev.ev1_tiles, ev.ev2_tiles, it.n, it.m, it.m1);
    eval_seq_displacement_kernel<<<1, 32, 0, s>>>(it, ev.out);
  } else {
    if (fork && it.world == 1) {
      // EV1 (rows of K) and EV2 (rows of K^T) are independent latency-bound
      // passes over the same unscaled points: run them side by side
      PDLP_CUDA(cudaEventRecord(fork->e_fork, s));
      PDLP_CUDA(cudaStreamWaitEvent(fork->s2, fork->e_fork, 0));
      eval_cols_kernel<false><<<g2, kThreads, sm2, fork->s2>>>(kt, ev, it.n, it.m1, -1);
      PDLP_CUDA(cudaGetLastError());
      PDLP_CUDA(cudaEventRecord(fork->e_join, fork->s2));
      eval_rows_kernel<false><<<g1, kThreads, sm1, s>>>(k, ev, it.m, it.m1);
      PDLP_CUDA(cudaStreamWaitEvent(s, fork->e_join, 0));
    } else {
      eval_rows_kernel<false><<<g1, kThreads, sm1, s>>>(k, ev, it.m, it.m1);
      eval_cols_kernel<false><<<g2, kThreads, sm2, s>>>(kt, ev, it.n, it.m1, -1);
    }
    PDLP_CUDA(cudaGetLastError());
    if (it.world > 1 && phase) phase();
    eval_reduce_kernel<<<kEvalReduceCtas, kThreads, 0, s>>>(ev);
    eval_final_kernel<false><<<1, kThreads, 0, s>>>(ev, ev.ev1_tiles, ev.ev2_tiles, it.n, it.m, it.m1);
  }
  PDLP_CUDA(cudaGetLastError());
}

void launch_chain_decide(DevState* st, const EvalOut* e, const ChainConsts& k, unsigned long long outer,
                         unsigned long long inner, cudaStream_t s) {
  chain_decide_kernel<<<1, 32, 0, s>>>(st, e, k, static_cast<cudaGraphConditionalHandle>(outer),
                                       static_cast<cudaGraphConditionalHandle>(inner));
  PDLP_CUDA(cudaGetLastError());
}

void launch_eval_lambda(const DevCsr& kt, const DevIter& it, const DevEval& ev, bool seq, int slot,
                        cudaStream_t s, const PhaseFn& phase) {
  if (seq) return;  // parity mode stores every slot's reduced costs on each evaluation
  const size_t sm2 = stream_smem_bytes<Ev2Epi<false>>();
  eval_cols_kernel<false><<<eval_grid(kt.ntiles), kThreads, sm2, s>>>(kt, ev, it.n, it.m1, slot);
  PDLP_CUDA(cudaGetLastError());
  if (it.world > 1) {  // wait for every rank's slice of the reduced costs
    if (phase) phase();
    shard_barrier_kernel<<<1, 32, 0, s>>>(ev.sync, ev.world, int(kSyncEvCols));
    PDLP_CUDA(cudaGetLastError());
  }
}

void launch_reduced_of_objective(const double* c, const double* l, const double* u, int n,
                                 double* lam, cudaStream_t s) {
  reduced_of_objective_kernel<<<grid_for(n), kThreads, 0, s>>>(c, l, u, n, lam);
  PDLP_CUDA(cudaGetLastError());
}

void launch_shard_masks(const int* rp, const int* col, int rows, const int64_t* kc, const int64_t* ktc, int world,
                        unsigned* xmask, unsigned* ymask, cudaStream_t s) {
  shard_mask_kernel<<<grid_for(rows), kThreads, 0, s>>>(rp, col, rows, kc, ktc, world, xmask, ymask);
  PDLP_CUDA(cudaGetLastError());
}
void launch_shard_volume(const unsigned* xmask, const unsigned* ymask, int col0, int col1, int row0, int row1,
                         int world, int rank, unsigned long long* out, cudaStream_t s) {
  shard_volume_kernel<<<grid_for(int64_t(col1 - col0) + (row1 - row0)), kThreads, 0, s>>>(
      xmask, ymask, col0, col1, row0, row1, world, rank, out);
  PDLP_CUDA(cudaGetLastError());
}

// pdhg_raw_step (solver.hpp:335-358), its elementwise halves on the unscaled
// saddle problem: x' = clamp(x - tau (c - K'y)) and the extrapolation 2x' - x;
// then y' = proj(y + sigma (q - K ext)) on the first m1 rows.
__global__ void raw_primal_kernel(const double* x, const double* kty, const double* c, const double* l,
                                  const double* u, double tau, int64_t n, double* xo, double* ext) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double xn = clamp_box(x[i] - tau * (c[i] - kty[i]), l[i], u[i]);
    xo[i] = xn;
    ext[i] = 2.0 * xn - x[i];
  }
}
__global__ void raw_dual_kernel(const double* y, const double* kext, const double* q, double sigma, int64_t m,
                                int64_t m1, double* yo) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    double yn = y[i] + sigma * (q[i] - kext[i]);
    if (i < m1 && yn < 0.0) yn = 0.0;  // project_dual_in_place, lp_model.hpp:124-129
    yo[i] = yn;
  }
}
void launch_raw_primal(const double* x, const double* kty, const double* c, const double* l, const double* u,
                       double tau, int64_t n, double* xo, double* ext, cudaStream_t s) {
  raw_primal_kernel<<<grid_for(n), kThreads, 0, s>>>(x, kty, c, l, u, tau, n, xo, ext);
  PDLP_CUDA(cudaGetLastError());
}
void launch_raw_dual(const double* y, const double* kext, const double* q, double sigma, int64_t m, int64_t m1,
                     double* yo, cudaStream_t s) {
  raw_dual_kernel<<<grid_for(m), kThreads, 0, s>>>(y, kext, q, sigma, m, m1, yo);
  PDLP_CUDA(cudaGetLastError());
}

}  // namespace pdlp
