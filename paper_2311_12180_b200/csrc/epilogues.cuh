// epilogues.cuh — the fused projected updates of the two iteration SpMVs,
// shared by the per-trial kernels (kernels.cu) and the column-panel sweeps
// (panels.cu).
#pragma once

#include "common.cuh"
#include "shard.cuh"
#include "spmv_engine.cuh"

namespace pdlp {


__device__ __forceinline__ double clamp_box(double v, double l, double u) {
  return smin(smax(v, l), u);  // std::min(std::max(x, l), u), vector_ops.hpp:56
}

// reduced_costs_from_slack (lp_model.hpp:155-174), one component.
__device__ __forceinline__ double reduced_cost(double v, double l, double u) {
  const bool lf = l > -INFINITY, uf = u < INFINITY;
  if (lf && uf) return v;
  if (lf) return smax(v, 0.0);
  if (uf) return smin(v, 0.0);
  return 0.0;
}

// l'lambda+ - u'lambda- contribution of one component (lp_model.hpp:248-251).
__device__ __forceinline__ double lambda_term(double lam, double l, double u) {
  if (lam > 0.0) return l * lam;
  if (lam < 0.0) return -(u * -lam);
  return 0.0;
}



// Loads of iteration vectors: the per-trial kernels may use the read-only
// (.nc) path; kCoh selects coherent L1-cached loads for data other CTAs wrote
// earlier in the same launch.
template <bool kCoh>
__device__ __forceinline__ double ldv(const double* p) {
  if (kCoh) return __ldca(p);
  return __ldg(p);
}
template <bool kCoh>
__device__ __forceinline__ double2 ldv2(const double* p) {
  if (kCoh) return __ldca(reinterpret_cast<const double2*>(p));
  return __ldg(reinterpret_cast<const double2*>(p));
}

// Dense operand streams of rows_strided: default caching, or kStreamIO =
// L2 evict-first style streaming (ld/st .cs) so a column-panel sweep's final
// pass does not push its L2-resident panel slice out with the update streams.
template <bool kCoh, bool kStreamIO>
__device__ __forceinline__ double ld_io(const double* p) {
  if (kStreamIO) return __ldcs(p);
  return ldv<kCoh>(p);
}
template <bool kStreamIO>
__device__ __forceinline__ double ld_io_plain(const double* p) {
  if (kStreamIO) return __ldcs(p);
  return *p;
}
template <bool kStreamIO>
__device__ __forceinline__ void st_io(double* p, double v) {
  if (kStreamIO)
    __stcs(p, v);
  else
    *p = v;
}

// Peer copies of the values an epilogue owns (row sharding, shard.cuh): to
// every peer, or only to the peers that gather value i (mask[i], bit q = rank q).
struct PeerPush {
  double* const* field;  // ShardView pointer array of the exchanged buffer
  size_t off;            // element offset of the active rotation buffer
  int world, rank;
  const unsigned* mask = nullptr;
  __device__ __forceinline__ void operator()(int i, double v) const {
    if (mask)
      push_peers_mask(field, world, rank, off + size_t(i), v, __ldg(mask + i));
    else
      push_peers(field, world, rank, off + size_t(i), v);
  }
};

template <bool kSeq, bool kCoh = false, bool kShard = false>
struct DualEpi : EpiBase<DualEpi<kSeq, kCoh, kShard>> {
  static constexpr int NP = 1, NA = 1, NR = 3;
  static constexpr TileGeom kGeom = kIterGeom;
  static constexpr bool kNeedCol = false;
  const double* __restrict__ xg;
  const double* __restrict__ y;
  const double* __restrict__ kx;
  const double* __restrict__ q;
  double* __restrict__ yt;
  double* __restrict__ kxt;
  double* __restrict__ seq_dy2;
  double* __restrict__ seq_inter;
  double sigma;
  int m1;
  PeerPush push;  // y' to every peer (kShard)
  __device__ __forceinline__ void gather(int c, double (&g)[1]) const { g[0] = ldv<kCoh>(xg + c); }
  __device__ __forceinline__ void add(double (&a)[1], const double (&p)[1], int) const { a[0] += p[0]; }
  __device__ __forceinline__ void row_done(int r, const double (&a)[1], double (&red)[3]) const {
    const double kxn = a[0];
    const double kxo = ldv<kCoh>(kx + r), yo = ldv<kCoh>(y + r);
    double yn = yo + sigma * (q[r] - 2.0 * kxn + kxo);  // solver.hpp:412-413
    if (r < m1 && yn < 0.0) yn = 0.0;                    // project_dual_in_place
    yt[r] = yn;
    if (kShard) push(r, yn);
    kxt[r] = kxn;
    const double d = yn - yo;
    const double dd = d * d, di = d * (kxn - kxo);
    if (kSeq) {
      seq_dy2[r] = dd;
      seq_inter[r] = di;
    }
    red[0] += dd;
    red[1] += di;
    red[2] += isfinite(yn) ? 0.0 : 1.0;
  }
  // all operand loads of the thread's rows first, then the updates (ILP)
  template <int RPT, int NA, int NR, bool kStreamIO = false>
  __device__ __forceinline__ void rows_strided(int r0, int stride, int nvalid,
                                               const double (&acc)[RPT][NA],
                                               double (&red)[NR]) const {
    double kxo[RPT], yo[RPT], qq[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      if (i < nvalid) {
        const int r = r0 + i * stride;
        kxo[i] = ld_io<kCoh, kStreamIO>(kx + r);
        yo[i] = ld_io<kCoh, kStreamIO>(y + r);
        qq[i] = ld_io_plain<kStreamIO>(q + r);
      }
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      if (i < nvalid) {
        const int r = r0 + i * stride;
        const double kxn = acc[i][0];
        double yn = yo[i] + sigma * (qq[i] - 2.0 * kxn + kxo[i]);  // solver.hpp:412-413
        if (r < m1 && yn < 0.0) yn = 0.0;
        st_io<kStreamIO>(yt + r, yn);
        if (kShard) push(r, yn);
        st_io<kStreamIO>(kxt + r, kxn);
        const double d = yn - yo[i];
        const double dd = d * d, di = d * (kxn - kxo[i]);
        if (kSeq) {
          seq_dy2[r] = dd;
          seq_inter[r] = di;
        }
        red[0] += dd;
        red[1] += di;
        red[2] += isfinite(yn) ? 0.0 : 1.0;
      }
  }
};

template <bool kSeq, bool kNonneg, bool kCoh = false, bool kShard = false>
struct PrimalEpi : EpiBase<PrimalEpi<kSeq, kNonneg, kCoh, kShard>> {
  static constexpr int NP = 1, NA = 1, NR = 2;
  static constexpr bool kUniform = !kCoh;  // K^T rows are often uniform (2 per column in C2, 5 in C1/C4)
  static constexpr TileGeom kGeom = kIterGeom;
  static constexpr bool kNeedCol = false;
  const double* __restrict__ yg;
  const double* __restrict__ xc;
  const double* __restrict__ c;
  const double* __restrict__ l;
  const double* __restrict__ u;
  double* __restrict__ kty_out;
  double* __restrict__ xt;
  double* __restrict__ avg_x;
  double* __restrict__ seq_dx2;
  double tau;
  double ratio;
  int do_avg;
  int avg_first;
  int store_kty;  // 0: K'y' of an accepted step is not kept (kty_lazy)
  PeerPush push;  // x' to every peer (kShard)
  __device__ __forceinline__ void gather(int r, double (&g)[1]) const { g[0] = ldv<kCoh>(yg + r); }
  __device__ __forceinline__ void add(double (&a)[1], const double (&p)[1], int) const { a[0] += p[0]; }
  __device__ __forceinline__ void row_done(int j, const double (&a)[1], double (&red)[2]) const {
    const double s = a[0];
    if (store_kty) kty_out[j] = s;
    const double xa = ldv<kCoh>(xc + j);
    if (do_avg) avg_x[j] = avg_first ? xa : avg_x[j] + ratio * (xa - avg_x[j]);
    const double v = xa - tau * (c[j] - s);  // solver.hpp:404-408
    const double xn = kNonneg ? smax(v, 0.0) : clamp_box(v, l[j], u[j]);
    xt[j] = xn;
    if (kShard) push(j, xn);
    const double d = xn - xa;
    const double dd = d * d;
    if (kSeq) seq_dx2[j] = dd;
    red[0] += dd;
    red[1] += isfinite(xn) ? 0.0 : 1.0;
  }
  // Four consecutive columns with 128-bit loads/stores when 16-byte aligned.
  __device__ __forceinline__ void rows_done(int j0, int nr, const double (&a)[4][1],
                                            double (&red)[2]) const {
    if (nr != 4 || (j0 & 1)) {
      for (int i = 0; i < nr; ++i) row_done(j0 + i, a[i], red);
      return;
    }
    double xa[4], cc[4], ll[4], uu[4], av[4];
    auto ld2 = [](const double* p, double* o) {
      const double2 v0 = ldv2<kCoh>(p);
      const double2 v1 = ldv2<kCoh>(p + 2);
      o[0] = v0.x, o[1] = v0.y, o[2] = v1.x, o[3] = v1.y;
    };
    auto st2 = [](double* p, const double* o) {
      reinterpret_cast<double2*>(p)[0] = make_double2(o[0], o[1]);
      reinterpret_cast<double2*>(p)[1] = make_double2(o[2], o[3]);
    };
    ld2(xc + j0, xa);
    ld2(c + j0, cc);
    if (!kNonneg) {
      ld2(l + j0, ll);
      ld2(u + j0, uu);
    }
    if (do_avg && !avg_first) ld2(avg_x + j0, av);
    double s4[4], xn4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      s4[i] = a[i][0];
      if (do_avg) av[i] = avg_first ? xa[i] : av[i] + ratio * (xa[i] - av[i]);
      const double v = xa[i] - tau * (cc[i] - s4[i]);
      xn4[i] = kNonneg ? smax(v, 0.0) : clamp_box(v, ll[i], uu[i]);
      const double d = xn4[i] - xa[i];
      const double dd = d * d;
      if (kSeq) seq_dx2[j0 + i] = dd;
      red[0] += dd;
      red[1] += isfinite(xn4[i]) ? 0.0 : 1.0;
    }
    if (store_kty) st2(kty_out + j0, s4);
    st2(xt + j0, xn4);
    if (kShard)
      for (int i = 0; i < 4; ++i) push(j0 + i, xn4[i]);
    if (do_avg) st2(avg_x + j0, av);
  }
  // all operand loads of the thread's columns first, then the updates (ILP)
  template <int RPT, int NA, int NR, bool kStreamIO = false>
  __device__ __forceinline__ void rows_strided(int j0, int stride, int nvalid,
                                               const double (&acc)[RPT][NA],
                                               double (&red)[NR]) const {
    double xa[RPT], cc[RPT], av[RPT], ll[RPT], uu[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      if (i < nvalid) {
        const int j = j0 + i * stride;
        xa[i] = ld_io<kCoh, kStreamIO>(xc + j);
        cc[i] = ld_io_plain<kStreamIO>(c + j);
        if (do_avg && !avg_first) av[i] = ld_io_plain<kStreamIO>(avg_x + j);
        if (!kNonneg) {
          ll[i] = ld_io_plain<kStreamIO>(l + j);
          uu[i] = ld_io_plain<kStreamIO>(u + j);
        }
      }
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      if (i < nvalid) {
        const int j = j0 + i * stride;
        const double s = acc[i][0];
        if (store_kty) st_io<kStreamIO>(kty_out + j, s);
        if (do_avg) st_io<kStreamIO>(avg_x + j, avg_first ? xa[i] : av[i] + ratio * (xa[i] - av[i]));
        const double v = xa[i] - tau * (cc[i] - s);  // solver.hpp:404-408
        const double xn = kNonneg ? smax(v, 0.0) : clamp_box(v, ll[i], uu[i]);
        st_io<kStreamIO>(xt + j, xn);
        if (kShard) push(j, xn);
        const double d = xn - xa[i];
        const double dd = d * d;
        if (kSeq) seq_dx2[j] = dd;
        red[0] += dd;
        red[1] += isfinite(xn) ? 0.0 : 1.0;
      }
  }
};

}  // namespace pdlp
