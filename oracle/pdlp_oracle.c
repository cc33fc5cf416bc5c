/* pdlp_oracle.c — TEST INFRASTRUCTURE ONLY (see pdlp_oracle.h).
 *
 * Plain-C restatement of the reference CPU solver. Every function cites the
 * reference routine it restates (paths relative to
 * /root/reference/proj/include/pdhglp/). Floating-point expressions keep the
 * reference's evaluation order; build with -O2 -ffp-contract=off (the
 * reference's default x86-64 build never contracts to FMA), so results are
 * bitwise identical to the reference (pinned by tests/test_oracle_pin.py).
 */
#define _POSIX_C_SOURCE 199309L
#include "pdlp_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* oracle_last_error(void) { return g_err; }

/* Summation-order probe (tests only, default 0 = the reference's sequential
 * loops). 1: the step-size sums dx^2, dy^2 and the interaction of
 * adaptive_step_cached (solver.hpp:422-435) as pairwise trees over blocks of 8
 * terms, i.e. another legal summation order of the same terms. It measures how
 * far a reordering alone moves the reference's own iterates. */
static int g_sum_order = 0;
void oracle_set_sum_order(int order) { g_sum_order = order; }

static double pairwise(const double* t, int64_t n) {
  if (n <= 8) {
    double a = 0.0;
    for (int64_t i = 0; i < n; ++i) a += t[i];
    return a;
  }
  const int64_t h = n / 2;
  return pairwise(t, h) + pairwise(t + h, n - h);
}

/* std::min / std::max / std::clamp exactly as libstdc++ defines them. */
static inline double smin(double a, double b) { return (b < a) ? b : a; }
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double sclamp(double v, double lo, double hi) {
  return (v < lo) ? lo : ((hi < v) ? hi : v);
}

/* ------------------------------------------------------------------------ */
/* CSR (sparse_matrix.hpp:35-55)                                            */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t rows, cols, nnz;
  int64_t* off;
  int64_t* col;
  double* val;
} csr_t;

static void csr_free(csr_t* a) {
  free(a->off);
  free(a->col);
  free(a->val);
  memset(a, 0, sizeof *a);
}

static void* xmalloc(size_t n) {
  void* p = malloc(n ? n : 1);
  if (!p) {
    fprintf(stderr, "oracle: out of memory (%zu bytes)\n", n);
    abort();
  }
  return p;
}

static double* dvec(int64_t n) { return (double*)xmalloc((size_t)n * sizeof(double)); }
static double* dzeros(int64_t n) {
  double* p = dvec(n);
  for (int64_t i = 0; i < n; ++i) p[i] = 0.0;
  return p;
}
static double* dcopy(const double* s, int64_t n) {
  double* p = dvec(n);
  if (n) memcpy(p, s, (size_t)n * sizeof(double));
  return p;
}

static csr_t csr_copy(const csr_t* a) {
  csr_t o = *a;
  o.off = (int64_t*)xmalloc((size_t)(a->rows + 1) * sizeof(int64_t));
  memcpy(o.off, a->off, (size_t)(a->rows + 1) * sizeof(int64_t));
  o.col = (int64_t*)xmalloc((size_t)a->nnz * sizeof(int64_t));
  if (a->nnz) memcpy(o.col, a->col, (size_t)a->nnz * sizeof(int64_t));
  o.val = dcopy(a->val, a->nnz);
  return o;
}

static int csr_from_abi(const pdlp_csr* in, csr_t* out) {
  memset(out, 0, sizeof *out);
  if (in->num_rows < 0 || in->num_cols < 0 || in->nnz < 0)
    return fail(PDLP_EINVAL, "csr: negative dimension");
  out->rows = in->num_rows;
  out->cols = in->num_cols;
  out->nnz = in->nnz;
  out->off = (int64_t*)xmalloc((size_t)(out->rows + 1) * sizeof(int64_t));
  out->col = (int64_t*)xmalloc((size_t)out->nnz * sizeof(int64_t));
  out->val = dvec(out->nnz);
  if (in->row_offsets) {
    memcpy(out->off, in->row_offsets, (size_t)(out->rows + 1) * sizeof(int64_t));
  } else {
    if (out->rows != 0 || out->nnz != 0) return fail(PDLP_EINVAL, "csr: missing row_offsets");
    out->off[0] = 0;
  }
  for (int64_t k = 0; k < out->nnz; ++k) {
    out->col[k] = in->col_indices ? in->col_indices[k] : (int64_t)in->col_indices32[k];
    out->val[k] = in->values[k];
  }
  if (out->off[0] != 0 || out->off[out->rows] != out->nnz)
    return fail(PDLP_EINVAL, "csr: row_offsets must start at 0 and end at nnz");
  return PDLP_OK;
}

/* Insertion/merge sort of a row slice by column (stable). The reference uses
 * std::sort (unstable); the order only matters for >= 3 duplicates of one
 * (row, col), which none of our instances contain. */
typedef struct {
  int64_t col;
  double val;
} slot_t;

static void sort_slots(slot_t* a, int64_t n, slot_t* tmp) {
  if (n < 16) {
    for (int64_t i = 1; i < n; ++i) {
      slot_t x = a[i];
      int64_t j = i - 1;
      while (j >= 0 && a[j].col > x.col) {
        a[j + 1] = a[j];
        --j;
      }
      a[j + 1] = x;
    }
    return;
  }
  int64_t h = n / 2;
  sort_slots(a, h, tmp);
  sort_slots(a + h, n - h, tmp);
  int64_t i = 0, j = h, k = 0;
  while (i < h && j < n) tmp[k++] = (a[j].col < a[i].col) ? a[j++] : a[i++];
  while (i < h) tmp[k++] = a[i++];
  while (j < n) tmp[k++] = a[j++];
  memcpy(a, tmp, (size_t)n * sizeof(slot_t));
}

/* CsrMatrix::from_triplets (sparse_matrix.hpp:57-108) */
static int csr_from_triplets(int64_t rows, int64_t cols, int64_t nt, const int64_t* tr,
                             const int64_t* tc, const double* tv, csr_t* out) {
  memset(out, 0, sizeof *out);
  for (int64_t i = 0; i < nt; ++i) {
    if (tr[i] < 0 || tr[i] >= rows || tc[i] < 0 || tc[i] >= cols)
      return fail(PDLP_EINVAL, "triplet %lld at (%lld, %lld) is outside a %lldx%lld matrix",
                  (long long)i, (long long)tr[i], (long long)tc[i], (long long)rows,
                  (long long)cols);
  }
  int64_t* count = (int64_t*)calloc((size_t)rows + 1, sizeof(int64_t));
  for (int64_t i = 0; i < nt; ++i) ++count[tr[i] + 1];
  for (int64_t r = 0; r < rows; ++r) count[r + 1] += count[r];
  slot_t* slot = (slot_t*)xmalloc((size_t)nt * sizeof(slot_t));
  slot_t* tmp = (slot_t*)xmalloc((size_t)nt * sizeof(slot_t));
  int64_t* next = (int64_t*)xmalloc((size_t)(rows + 1) * sizeof(int64_t));
  memcpy(next, count, (size_t)(rows + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < nt; ++i) {
    slot_t s = {tc[i], tv[i]};
    slot[next[tr[i]]++] = s;
  }
  out->rows = rows;
  out->cols = cols;
  out->off = (int64_t*)calloc((size_t)rows + 1, sizeof(int64_t));
  out->col = (int64_t*)xmalloc((size_t)nt * sizeof(int64_t));
  out->val = dvec(nt);
  int64_t nnz = 0;
  for (int64_t r = 0; r < rows; ++r) {
    slot_t* b = slot + count[r];
    int64_t len = count[r + 1] - count[r];
    sort_slots(b, len, tmp);
    for (int64_t i = 0; i < len;) {
      int64_t c = b[i].col;
      double sum = 0.0;
      for (; i < len && b[i].col == c; ++i) sum += b[i].val;
      if (sum != 0.0) {
        out->col[nnz] = c;
        out->val[nnz] = sum;
        ++nnz;
      }
    }
    out->off[r + 1] = nnz;
  }
  out->nnz = nnz;
  free(count);
  free(slot);
  free(tmp);
  free(next);
  return PDLP_OK;
}

/* spmv (sparse_matrix.hpp:117-132): row-sequential sums starting at 0.0 */
static void spmv(const csr_t* a, const double* x, double* out) {
  for (int64_t r = 0; r < a->rows; ++r) {
    double sum = 0.0;
    for (int64_t k = a->off[r]; k < a->off[r + 1]; ++k) sum += a->val[k] * x[a->col[k]];
    out[r] = sum;
  }
}

/* spmv_transpose (sparse_matrix.hpp:142-158): scatter in row order, zero y skipped */
static void spmv_t(const csr_t* a, const double* y, double* out) {
  for (int64_t c = 0; c < a->cols; ++c) out[c] = 0.0;
  for (int64_t r = 0; r < a->rows; ++r) {
    const double yr = y[r];
    if (yr == 0.0) continue;
    for (int64_t k = a->off[r]; k < a->off[r + 1]; ++k) out[a->col[k]] += a->val[k] * yr;
  }
}

/* explicit_transpose (sparse_matrix.hpp:167-178) */
static int csr_transpose(const csr_t* a, csr_t* out) {
  int64_t* tr = (int64_t*)xmalloc((size_t)a->nnz * sizeof(int64_t));
  int64_t* tc = (int64_t*)xmalloc((size_t)a->nnz * sizeof(int64_t));
  for (int64_t r = 0; r < a->rows; ++r)
    for (int64_t k = a->off[r]; k < a->off[r + 1]; ++k) {
      tr[k] = a->col[k];
      tc[k] = r;
    }
  int rc = csr_from_triplets(a->cols, a->rows, a->nnz, tr, tc, a->val, out);
  free(tr);
  free(tc);
  return rc;
}

/* vstack (sparse_matrix.hpp:181-200) */
static csr_t csr_vstack(const csr_t* top, const csr_t* bot) {
  csr_t m;
  m.rows = top->rows + bot->rows;
  m.cols = top->cols;
  m.nnz = top->nnz + bot->nnz;
  m.off = (int64_t*)xmalloc((size_t)(m.rows + 1) * sizeof(int64_t));
  m.col = (int64_t*)xmalloc((size_t)m.nnz * sizeof(int64_t));
  m.val = dvec(m.nnz);
  memcpy(m.off, top->off, (size_t)(top->rows + 1) * sizeof(int64_t));
  for (int64_t i = 1; i <= bot->rows; ++i) m.off[top->rows + i] = bot->off[i] + top->nnz;
  if (top->nnz) {
    memcpy(m.col, top->col, (size_t)top->nnz * sizeof(int64_t));
    memcpy(m.val, top->val, (size_t)top->nnz * sizeof(double));
  }
  if (bot->nnz) {
    memcpy(m.col + top->nnz, bot->col, (size_t)bot->nnz * sizeof(int64_t));
    memcpy(m.val + top->nnz, bot->val, (size_t)bot->nnz * sizeof(double));
  }
  return m;
}

/* max_abs_entry (sparse_matrix.hpp:203-207) */
static double max_abs_entry(const csr_t* a) {
  double m = 0.0;
  for (int64_t k = 0; k < a->nnz; ++k) m = smax(m, fabs(a->val[k]));
  return m;
}

/* row_norms / col_norms (sparse_matrix.hpp:212-255) */
static void row_norms(const csr_t* a, double p, double* out) {
  for (int64_t r = 0; r < a->rows; ++r) {
    double acc = 0.0;
    for (int64_t k = a->off[r]; k < a->off[r + 1]; ++k) {
      const double v = fabs(a->val[k]);
      if (isinf(p))
        acc = smax(acc, v);
      else if (p == 0.0)
        acc += 1.0;
      else
        acc += pow(v, p);
    }
    if (!isinf(p) && p != 0.0 && acc > 0.0) acc = pow(acc, 1.0 / p);
    out[r] = acc;
  }
}

static void col_norms(const csr_t* a, double p, double* out) {
  for (int64_t c = 0; c < a->cols; ++c) out[c] = 0.0;
  for (int64_t r = 0; r < a->rows; ++r)
    for (int64_t k = a->off[r]; k < a->off[r + 1]; ++k) {
      const double v = fabs(a->val[k]);
      double* acc = &out[a->col[k]];
      if (isinf(p))
        *acc = smax(*acc, v);
      else if (p == 0.0)
        *acc += 1.0;
      else
        *acc += pow(v, p);
    }
  if (!isinf(p) && p != 0.0)
    for (int64_t c = 0; c < a->cols; ++c)
      if (out[c] > 0.0) out[c] = pow(out[c], 1.0 / p);
}

/* ------------------------------------------------------------------------ */
/* Scaling (scaling.hpp)                                                    */
/* ------------------------------------------------------------------------ */
typedef struct {
  double* row; /* D1, m */
  double* col; /* D2, n */
} scaling_t;

static scaling_t scaling_identity(int64_t m, int64_t n) {
  scaling_t s = {dvec(m), dvec(n)};
  for (int64_t i = 0; i < m; ++i) s.row[i] = 1.0;
  for (int64_t i = 0; i < n; ++i) s.col[i] = 1.0;
  return s;
}

/* detail::scaled_copy (scaling.hpp:32-44): v * (dr * dc) */
static csr_t scaled_copy(const csr_t* k, const scaling_t* s) {
  csr_t o = csr_copy(k);
  for (int64_t r = 0; r < k->rows; ++r) {
    const double dr = s->row[r];
    for (int64_t i = k->off[r]; i < k->off[r + 1]; ++i) o.val[i] *= dr * s->col[k->col[i]];
  }
  return o;
}

/* ruiz_equilibrate (scaling.hpp:52-66) */
static scaling_t ruiz(const csr_t* k, int iterations) {
  scaling_t s = scaling_identity(k->rows, k->cols);
  double* rn = dvec(k->rows);
  double* cn = dvec(k->cols);
  for (int it = 0; it < iterations; ++it) {
    csr_t sc = scaled_copy(k, &s);
    row_norms(&sc, INFINITY, rn);
    col_norms(&sc, INFINITY, cn);
    for (int64_t r = 0; r < k->rows; ++r)
      if (rn[r] > 0.0) s.row[r] /= sqrt(rn[r]);
    for (int64_t c = 0; c < k->cols; ++c)
      if (cn[c] > 0.0) s.col[c] /= sqrt(cn[c]);
    csr_free(&sc);
  }
  free(rn);
  free(cn);
  return s;
}

/* pock_chambolle_scale (scaling.hpp:72-94) */
static scaling_t pock_chambolle(const csr_t* k, double alpha) {
  scaling_t s = scaling_identity(k->rows, k->cols);
  double* rs = dvec(k->rows);
  double* cs = dvec(k->cols);
  row_norms(k, 2.0 - alpha, rs);
  col_norms(k, alpha, cs);
  const double row_p = 2.0 - alpha, col_p = alpha;
  for (int64_t r = 0; r < k->rows; ++r) {
    double sum = rs[r];
    if (row_p != 0.0 && sum > 0.0) sum = pow(sum, row_p);
    if (sum > 0.0) s.row[r] = 1.0 / sqrt(sum);
  }
  for (int64_t c = 0; c < k->cols; ++c) {
    double sum = cs[c];
    if (col_p != 0.0 && sum > 0.0) sum = pow(sum, col_p);
    if (sum > 0.0) s.col[c] = 1.0 / sqrt(sum);
  }
  free(rs);
  free(cs);
  return s;
}

/* make_scaling (scaling.hpp:117-132) + compose (:98-112) */
static scaling_t make_scaling(const csr_t* k, int mode, int ruiz_it, double alpha) {
  if (mode == PDLP_SCALING_NONE) return scaling_identity(k->rows, k->cols);
  scaling_t r = ruiz(k, ruiz_it);
  if (mode == PDLP_SCALING_RUIZ) return r;
  csr_t after = scaled_copy(k, &r);
  scaling_t pc = pock_chambolle(&after, alpha);
  for (int64_t i = 0; i < k->rows; ++i) r.row[i] *= pc.row[i];
  for (int64_t i = 0; i < k->cols; ++i) r.col[i] *= pc.col[i];
  csr_free(&after);
  free(pc.row);
  free(pc.col);
  return r;
}

/* ------------------------------------------------------------------------ */
/* LP model (lp_model.hpp)                                                  */
/* ------------------------------------------------------------------------ */
typedef struct {
  csr_t G, A;
  int64_t n, m1, m2;
  double *c, *h, *b, *l, *u;
  double c0;
} lp_t;

static void lp_free(lp_t* lp) {
  csr_free(&lp->G);
  csr_free(&lp->A);
  free(lp->c);
  free(lp->h);
  free(lp->b);
  free(lp->l);
  free(lp->u);
}

/* GeneralFormLp::validate (lp_model.hpp:45-72) */
static int lp_from_abi(const pdlp_lp* in, lp_t* lp) {
  memset(lp, 0, sizeof *lp);
  int rc = csr_from_abi(&in->inequality_matrix, &lp->G);
  if (rc) return rc;
  rc = csr_from_abi(&in->equality_matrix, &lp->A);
  if (rc) return rc;
  const int64_t n = in->num_variables;
  lp->n = n;
  lp->m1 = lp->G.rows;
  lp->m2 = lp->A.rows;
  if (lp->G.cols != n || lp->A.cols != n)
    return fail(PDLP_EINVAL, "lp: constraint matrices must have n columns");
  lp->c = dcopy(in->objective, n);
  lp->h = dcopy(in->inequality_rhs, lp->m1);
  lp->b = dcopy(in->equality_rhs, lp->m2);
  lp->l = dcopy(in->lower, n);
  lp->u = dcopy(in->upper, n);
  lp->c0 = in->objective_constant;
  for (int64_t i = 0; i < n; ++i) {
    const double l = lp->l[i], u = lp->u[i];
    if (isnan(l) || isnan(u)) return fail(PDLP_EINVAL, "lp: NaN bound on variable %lld", (long long)i);
    if (l > u || l == INFINITY || u == -INFINITY)
      return fail(PDLP_EINVAL, "lp: empty bound interval on variable %lld", (long long)i);
  }
  for (int64_t i = 0; i < n; ++i)
    if (isnan(lp->c[i])) return fail(PDLP_EINVAL, "lp: NaN objective entry");
  return PDLP_OK;
}

/* apply_scaling (scaling.hpp:137-170) */
static lp_t apply_scaling(const lp_t* lp, const scaling_t* s) {
  lp_t o = *lp;
  o.G = csr_copy(&lp->G);
  o.A = csr_copy(&lp->A);
  for (int64_t r = 0; r < o.G.rows; ++r) {
    const double dr = s->row[r];
    for (int64_t i = o.G.off[r]; i < o.G.off[r + 1]; ++i) o.G.val[i] *= dr * s->col[o.G.col[i]];
  }
  for (int64_t r = 0; r < o.A.rows; ++r) {
    const double dr = s->row[lp->m1 + r];
    for (int64_t i = o.A.off[r]; i < o.A.off[r + 1]; ++i) o.A.val[i] *= dr * s->col[o.A.col[i]];
  }
  o.h = dcopy(lp->h, lp->m1);
  o.b = dcopy(lp->b, lp->m2);
  o.c = dcopy(lp->c, lp->n);
  o.l = dcopy(lp->l, lp->n);
  o.u = dcopy(lp->u, lp->n);
  for (int64_t i = 0; i < lp->m1; ++i) o.h[i] *= s->row[i];
  for (int64_t i = 0; i < lp->m2; ++i) o.b[i] *= s->row[lp->m1 + i];
  for (int64_t i = 0; i < lp->n; ++i) {
    o.c[i] *= s->col[i];
    if (isfinite(o.l[i])) o.l[i] /= s->col[i];
    if (isfinite(o.u[i])) o.u[i] /= s->col[i];
  }
  return o;
}

static double sqnorm(const double* x, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += x[i] * x[i];
  return s;
}
static double norm2(const double* x, int64_t n) { return sqrt(sqnorm(x, n)); }
static double dot(const double* x, const double* y, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}

typedef struct {
  double* lambda;
  double* pos;
  double* neg;
} reduced_t;

static void reduced_free(reduced_t* r) {
  free(r->lambda);
  free(r->pos);
  free(r->neg);
  memset(r, 0, sizeof *r);
}

/* reduced_costs_from_slack (lp_model.hpp:147-176) */
static reduced_t reduced_from_slack(const double* slack, const double* l, const double* u, int64_t n) {
  reduced_t rc = {dzeros(n), dzeros(n), dzeros(n)};
  for (int64_t i = 0; i < n; ++i) {
    const int lf = l[i] > -INFINITY, uf = u[i] < INFINITY;
    double v = slack[i];
    if (lf && uf) {
    } else if (lf) {
      v = smax(v, 0.0);
    } else if (uf) {
      v = smin(v, 0.0);
    } else {
      v = 0.0;
    }
    rc.lambda[i] = v;
    if (v > 0.0)
      rc.pos[i] = v;
    else if (v < 0.0)
      rc.neg[i] = -v;
  }
  return rc;
}

/* dual_slack (lp_model.hpp:179-190): r = c - G'y1 - A'y2 via two scatters */
static double* dual_slack(const lp_t* lp, const double* y) {
  double* r = dcopy(lp->c, lp->n);
  double* tmp = dvec(lp->n);
  spmv_t(&lp->G, y, tmp);
  for (int64_t i = 0; i < lp->n; ++i) r[i] += -1.0 * tmp[i];
  spmv_t(&lp->A, y + lp->m1, tmp);
  for (int64_t i = 0; i < lp->n; ++i) r[i] += -1.0 * tmp[i];
  free(tmp);
  return r;
}

/* dual_objective (lp_model.hpp:236-253) */
static double dual_objective(const lp_t* lp, const double* y, const reduced_t* rc) {
  double obj = lp->c0;
  for (int64_t i = 0; i < lp->m1; ++i) obj += lp->h[i] * y[i];
  for (int64_t i = 0; i < lp->m2; ++i) obj += lp->b[i] * y[lp->m1 + i];
  for (int64_t i = 0; i < lp->n; ++i) {
    if (rc->pos[i] != 0.0) obj += lp->l[i] * rc->pos[i];
    if (rc->neg[i] != 0.0) obj -= lp->u[i] * rc->neg[i];
  }
  return obj;
}

/* ------------------------------------------------------------------------ */
/* KKT / termination (solver.hpp:106-249)                                   */
/* ------------------------------------------------------------------------ */
typedef struct {
  double prn, drn, pobj, dobj;
} kkt_t;

static double kkt_gap(const kkt_t* r) { return r->dobj - r->pobj; }
/* KktResiduals::weighted (solver.hpp:117-122) */
static double kkt_weighted(const kkt_t* r, double omega) {
  const double pr = omega * r->prn, dr = r->drn / omega, g = kkt_gap(r);
  return sqrt(pr * pr + dr * dr + g * g);
}

typedef struct {
  kkt_t res;
  reduced_t red;
} point_eval_t;

/* evaluate_point (solver.hpp:130-144) with primal_residual (lp_model.hpp:202-218) */
static point_eval_t evaluate_point(const lp_t* lp, const double* x, const double* y) {
  point_eval_t ev;
  double* eq = dvec(lp->m2);
  spmv(&lp->A, x, eq);
  for (int64_t i = 0; i < lp->m2; ++i) eq[i] += -1.0 * lp->b[i];
  double* gx = dvec(lp->m1);
  spmv(&lp->G, x, gx);
  for (int64_t i = 0; i < lp->m1; ++i) gx[i] = smax(lp->h[i] - gx[i], 0.0);
  ev.res.prn = sqrt(sqnorm(eq, lp->m2) + sqnorm(gx, lp->m1));
  free(eq);
  free(gx);
  double* slack = dual_slack(lp, y);
  ev.red = reduced_from_slack(slack, lp->l, lp->u, lp->n);
  for (int64_t i = 0; i < lp->n; ++i) slack[i] += -1.0 * ev.red.lambda[i];
  ev.res.drn = norm2(slack, lp->n);
  free(slack);
  ev.res.pobj = dot(lp->c, x, lp->n);
  ev.res.dobj = dual_objective(lp, y, &ev.red) - lp->c0;
  return ev;
}

typedef struct {
  double rhs_norm, obj_norm;
} term_norms_t;

/* termination_criteria_met (solver.hpp:204-222) */
static int termination_met(const kkt_t* r, double eps, const term_norms_t* nn) {
  if (!isfinite(r->prn) || !isfinite(r->drn) || !isfinite(r->pobj) || !isfinite(r->dobj)) return 0;
  const int gap_ok = fabs(kkt_gap(r)) <= eps * (1.0 + fabs(r->dobj) + fabs(r->pobj));
  const int p_ok = r->prn <= eps * (1.0 + nn->rhs_norm);
  const int d_ok = r->drn <= eps * (1.0 + nn->obj_norm);
  return gap_ok && p_ok && d_ok;
}

/* should_restart (solver.hpp:270-286) */
static int should_restart(double now, double prev, double start, int64_t t, int64_t k,
                          const pdlp_params* p) {
  if (now <= p->beta_sufficient * start) return PDLP_RESTART_SUFFICIENT_DECAY;
  if (now <= p->beta_necessary * start && now > prev) return PDLP_RESTART_NECESSARY_DECAY;
  if ((double)t >= p->beta_artificial * (double)k) return PDLP_RESTART_LONG_INNER_LOOP;
  return PDLP_RESTART_NONE;
}

/* ------------------------------------------------------------------------ */
/* Infeasibility (solver.hpp:503-590)                                       */
/* ------------------------------------------------------------------------ */
typedef struct {
  int status; /* 0 none, else PDLP_STATUS_* */
  double* ray_x;
  double* ray_y;
  reduced_t red;
} cert_t;

static void project_dual(double* y, int64_t m1) {
  for (int64_t i = 0; i < m1; ++i)
    if (y[i] < 0.0) y[i] = 0.0;
}

/* detail::certificate_from_ray (solver.hpp:503-574) */
static cert_t certificate_from_ray(const lp_t* lp, const double* rx, const double* ry,
                                   double eps_inf, double eps_zero) {
  cert_t cert;
  memset(&cert, 0, sizeof cert);
  const int64_t n = lp->n, m = lp->m1 + lp->m2;
  double* y = dcopy(ry, m);
  project_dual(y, lp->m1);
  const double y_norm = norm2(y, m);
  if (y_norm > eps_zero) {
    double* kty = dvec(n);
    double* tmp = dvec(n);
    spmv_t(&lp->G, y, kty);
    spmv_t(&lp->A, y + lp->m1, tmp);
    for (int64_t i = 0; i < n; ++i) kty[i] += 1.0 * tmp[i];
    for (int64_t i = 0; i < n; ++i) tmp[i] = -kty[i];
    reduced_t lam = reduced_from_slack(tmp, lp->l, lp->u, n);
    for (int64_t i = 0; i < n; ++i) kty[i] += 1.0 * lam.lambda[i];
    const double residual = norm2(kty, n);
    const double objective = dual_objective(lp, y, &lam) - lp->c0;
    free(kty);
    free(tmp);
    if (residual <= eps_inf * y_norm && objective > eps_inf * y_norm) {
      cert.status = PDLP_STATUS_PRIMAL_INFEASIBLE;
      cert.ray_y = y;
      cert.red = lam;
      return cert;
    }
    reduced_free(&lam);
  }
  free(y);
  const double x_norm = norm2(rx, n);
  if (x_norm > eps_zero) {
    const double tol = eps_inf * x_norm;
    double* ax = dvec(lp->m2);
    spmv(&lp->A, rx, ax);
    int ok = norm2(ax, lp->m2) <= tol;
    free(ax);
    if (ok) {
      double* gx = dvec(lp->m1);
      spmv(&lp->G, rx, gx);
      for (int64_t i = 0; i < lp->m1; ++i)
        if (gx[i] < -tol) {
          ok = 0;
          break;
        }
      free(gx);
    }
    if (ok)
      for (int64_t i = 0; i < n && ok; ++i) {
        if (lp->l[i] > -INFINITY && rx[i] < -tol) ok = 0;
        if (lp->u[i] < INFINITY && rx[i] > tol) ok = 0;
      }
    if (ok && dot(lp->c, rx, n) < -tol) {
      cert.status = PDLP_STATUS_DUAL_INFEASIBLE;
      cert.ray_x = dcopy(rx, n);
      return cert;
    }
  }
  return cert;
}

/* ------------------------------------------------------------------------ */
/* Solve loop (solver.hpp:634-929)                                          */
/* ------------------------------------------------------------------------ */
struct oracle_session {
  pdlp_params p;
  lp_t orig;
  term_norms_t norms;
  scaling_t s;
  lp_t scaled;
  csr_t K; /* saddle matrix (solver.hpp:644, lp_model.hpp:88-98) */
  double *q;
  int64_t n, m, m1;
  /* iterate state */
  double *x, *y, *kx, *kty;
  double *xs, *ys; /* epoch start */
  double *ax, *ay, wsum; /* WeightedAverage (vector_ops.hpp:86-116) */
  double *dx_last, *dy_last;
  double eta, eta_hat, omega;
  int64_t outer, inner, total, trials;
  double kkt_epoch_start, kkt_last_candidate;
  struct timespec t0;
  /* scratch for the adaptive step */
  double *xn, *yn, *kxn;
  /* logs */
  pdlp_step_log_entry* slog;
  int64_t slog_n, slog_cap;
  pdlp_restart_event* rlog;
  int64_t rlog_n, rlog_cap;
  /* result */
  int finished;
  pdlp_result_info info;
  double *rx, *ry;
  reduced_t rred;
};

static double elapsed(const oracle_session* s) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (double)(t.tv_sec - s->t0.tv_sec) + 1e-9 * (double)(t.tv_nsec - s->t0.tv_nsec);
}

/* params.validate (solver.hpp:79-93) */
static int params_validate(const pdlp_params* p) {
  if (!(p->eps_optimal > 0.0) || !(p->eps_infeasible > 0.0))
    return fail(PDLP_EINVAL, "params: tolerances must be positive");
  if (!(p->beta_sufficient > 0.0 && p->beta_sufficient < p->beta_necessary && p->beta_necessary < 1.0))
    return fail(PDLP_EINVAL, "params: need 0 < beta_sufficient < beta_necessary < 1");
  if (p->theta_smoothing < 0.0 || p->theta_smoothing > 1.0)
    return fail(PDLP_EINVAL, "params: theta_smoothing must lie in [0, 1]");
  if (p->evaluation_frequency < 1) return fail(PDLP_EINVAL, "params: evaluation_frequency must be >= 1");
  if (p->ruiz_iterations < 0) return fail(PDLP_EINVAL, "ruiz: negative iteration count");
  if (p->pock_chambolle_alpha < 0.0 || p->pock_chambolle_alpha > 2.0)
    return fail(PDLP_EINVAL, "pock-chambolle: alpha must lie in [0, 2]");
  return PDLP_OK;
}

static void push_step(oracle_session* s, pdlp_step_log_entry e) {
  if (s->slog_n == s->slog_cap) {
    s->slog_cap = s->slog_cap ? 2 * s->slog_cap : 1024;
    s->slog = (pdlp_step_log_entry*)realloc(s->slog, (size_t)s->slog_cap * sizeof *s->slog);
  }
  s->slog[s->slog_n++] = e;
}

static void push_restart(oracle_session* s, pdlp_restart_event e) {
  if (s->rlog_n == s->rlog_cap) {
    s->rlog_cap = s->rlog_cap ? 2 * s->rlog_cap : 64;
    s->rlog = (pdlp_restart_event*)realloc(s->rlog, (size_t)s->rlog_cap * sizeof *s->rlog);
  }
  s->rlog[s->rlog_n++] = e;
}

/* SolveLoop::finish (solver.hpp:741-757): takes ownership of x, y and red. */
static void finish(oracle_session* s, int status, double* x, double* y, const kkt_t* r,
                   reduced_t red, const char* msg) {
  pdlp_result_info* in = &s->info;
  memset(in, 0, sizeof *in);
  in->status = status;
  in->primal_objective_raw = r->pobj;
  in->dual_objective_raw = r->dobj;
  in->primal_objective = r->pobj + s->orig.c0;
  in->dual_objective = r->dobj + s->orig.c0;
  in->gap_abs = fabs(kkt_gap(r));
  in->primal_residual_norm = r->prn;
  in->dual_residual_norm = r->drn;
  in->relative_gap = in->gap_abs / (1.0 + fabs(r->dobj) + fabs(r->pobj));
  in->relative_primal_residual = r->prn / (1.0 + s->norms.rhs_norm);
  in->relative_dual_residual = r->drn / (1.0 + s->norms.obj_norm);
  in->kkt_omega = kkt_weighted(r, s->omega);
  in->iterations = s->total;
  in->restarts = s->outer;
  in->solve_seconds = elapsed(s);
  in->step_log_size = s->slog_n;
  in->restart_log_size = s->rlog_n;
  in->num_variables = s->n;
  in->num_constraints = s->m;
  in->trials = s->trials;
  if (msg) snprintf(in->message, sizeof in->message, "%s", msg);
  s->rx = x;
  s->ry = y;
  s->rred = red;
  s->finished = 1;
}

typedef struct {
  double *cand_x, *cand_y; /* scaled, owned */
  double *cand_ux, *cand_uy; /* unscaled, owned */
  point_eval_t cand_eval;
  int cand_is_avg;
  double kkt_cand;
  int terminated;
  double *other_ux, *other_uy;
  point_eval_t other_eval;
  int other_terminated;
} evaluation_t;

static void unscale(const oracle_session* s, const double* x, const double* y, double** ux, double** uy) {
  *ux = dvec(s->n);
  *uy = dvec(s->m);
  for (int64_t i = 0; i < s->n; ++i) (*ux)[i] = x[i] * s->s.col[i];
  for (int64_t i = 0; i < s->m; ++i) (*uy)[i] = y[i] * s->s.row[i];
}

/* SolveLoop::evaluate_candidates (solver.hpp:705-739) */
static evaluation_t evaluate_candidates(const oracle_session* s) {
  evaluation_t ev;
  memset(&ev, 0, sizeof ev);
  const int empty = s->wsum == 0.0;
  const double* avx = empty ? s->x : s->ax;
  const double* avy = empty ? s->y : s->ay;
  double *cux, *cuy, *aux, *auy;
  unscale(s, s->x, s->y, &cux, &cuy);
  unscale(s, avx, avy, &aux, &auy);
  point_eval_t ec = evaluate_point(&s->orig, cux, cuy);
  point_eval_t ea = evaluate_point(&s->orig, aux, auy);
  const double kc = kkt_weighted(&ec.res, s->omega);
  const double ka = kkt_weighted(&ea.res, s->omega);
  ev.cand_is_avg = !(kc < ka);
  if (ev.cand_is_avg) {
    ev.cand_x = dcopy(avx, s->n);
    ev.cand_y = dcopy(avy, s->m);
    ev.cand_ux = aux;
    ev.cand_uy = auy;
    ev.cand_eval = ea;
    ev.kkt_cand = ka;
    ev.other_ux = cux;
    ev.other_uy = cuy;
    ev.other_eval = ec;
  } else {
    ev.cand_x = dcopy(s->x, s->n);
    ev.cand_y = dcopy(s->y, s->m);
    ev.cand_ux = cux;
    ev.cand_uy = cuy;
    ev.cand_eval = ec;
    ev.kkt_cand = kc;
    ev.other_ux = aux;
    ev.other_uy = auy;
    ev.other_eval = ea;
  }
  ev.terminated = termination_met(&ev.cand_eval.res, s->p.eps_optimal, &s->norms);
  ev.other_terminated = termination_met(&ev.other_eval.res, s->p.eps_optimal, &s->norms);
  return ev;
}

static void evaluation_free(evaluation_t* ev) {
  free(ev->cand_x);
  free(ev->cand_y);
  free(ev->cand_ux);
  free(ev->cand_uy);
  free(ev->other_ux);
  free(ev->other_uy);
  reduced_free(&ev->cand_eval.red);
  reduced_free(&ev->other_eval.red);
}

/* finish with the candidate of an evaluation (limit / failure exits) */
static void finish_candidate(oracle_session* s, int status, const char* msg) {
  evaluation_t ev = evaluate_candidates(s);
  finish(s, status, ev.cand_ux, ev.cand_uy, &ev.cand_eval.res, ev.cand_eval.red, msg);
  ev.cand_ux = ev.cand_uy = NULL;
  ev.cand_eval.red.lambda = ev.cand_eval.red.pos = ev.cand_eval.red.neg = NULL;
  evaluation_free(&ev);
}

typedef struct {
  int failure;
  double eta_acc, eta_next, eta_bar, mov, inter;
  int trials;
} step_out_t;

/* detail::adaptive_step_cached (solver.hpp:381-467). On accept the new point
 * is in s->xn/s->yn/s->kxn and K'y' is written to kty_next. */
static step_out_t adaptive_step(oracle_session* s, int64_t k, double* kty_next) {
  step_out_t r;
  memset(&r, 0, sizeof r);
  const lp_t* sp = &s->scaled;
  const int64_t n = s->n, m = s->m;
  const double kp1 = (double)k + 1.0;
  const double reduction = 1.0 - pow(kp1, -s->p.step_reduction_exponent);
  const double growth = 1.0 + pow(kp1, -s->p.step_growth_exponent);
  double eta = s->eta_hat;
  for (int trial = 0; trial < 80; ++trial) {
    r.trials = trial + 1;
    s->trials += 1;
    const double tau = eta / s->omega, sigma = eta * s->omega;
    for (int64_t i = 0; i < n; ++i) {
      const double v = s->x[i] - tau * (sp->c[i] - s->kty[i]);
      s->xn[i] = smin(smax(v, sp->l[i]), sp->u[i]);
    }
    spmv(&s->K, s->xn, s->kxn);
    for (int64_t i = 0; i < m; ++i) s->yn[i] = s->y[i] + sigma * (s->q[i] - 2.0 * s->kxn[i] + s->kx[i]);
    project_dual(s->yn, s->m1);
    for (int64_t i = 0; i < n; ++i)
      if (!isfinite(s->xn[i])) {
        r.failure = 1;
        return r;
      }
    for (int64_t i = 0; i < m; ++i)
      if (!isfinite(s->yn[i])) {
        r.failure = 1;
        return r;
      }
    double dx = 0.0;
    double dy = 0.0, inter = 0.0;
    if (g_sum_order == 1) {
      double* t = (double*)xmalloc((size_t)(n > m ? n : m) * sizeof(double));
      for (int64_t i = 0; i < n; ++i) t[i] = (s->xn[i] - s->x[i]) * (s->xn[i] - s->x[i]);
      dx = pairwise(t, n);
      for (int64_t i = 0; i < m; ++i) t[i] = (s->yn[i] - s->y[i]) * (s->yn[i] - s->y[i]);
      dy = pairwise(t, m);
      for (int64_t i = 0; i < m; ++i) t[i] = (s->yn[i] - s->y[i]) * (s->kxn[i] - s->kx[i]);
      inter = pairwise(t, m);
      free(t);
    } else {
      for (int64_t i = 0; i < n; ++i) {
        const double d = s->xn[i] - s->x[i];
        dx += d * d;
      }
      for (int64_t i = 0; i < m; ++i) {
        const double d = s->yn[i] - s->y[i];
        dy += d * d;
        inter += d * (s->kxn[i] - s->kx[i]);
      }
    }
    const double mov = s->omega * dx + dy / s->omega;
    const double ia = fabs(inter);
    const double eta_bar = ia > 0.0 ? mov / (2.0 * ia) : INFINITY;
    const double eta_next = smin(reduction * eta_bar, growth * eta);
    if (eta <= eta_bar) {
      r.eta_acc = eta;
      r.eta_next = eta_next;
      r.eta_bar = eta_bar;
      r.mov = mov;
      r.inter = inter;
      spmv_t(&s->K, s->yn, kty_next);
      return r;
    }
    eta = eta_next;
    if (!(eta > 0.0) || !isfinite(eta)) {
      r.failure = 1;
      return r;
    }
  }
  r.failure = 1;
  return r;
}

/* WeightedAverage::add (vector_ops.hpp:95-107) */
static void avg_add(double* avg, const double* v, int64_t n, double w, double wsum) {
  if (wsum == w) {
    memcpy(avg, v, (size_t)n * sizeof(double));
    return;
  }
  const double ratio = w / wsum;
  for (int64_t i = 0; i < n; ++i) avg[i] += ratio * (v[i] - avg[i]);
}

oracle_session* oracle_begin(const pdlp_lp* lpin, const pdlp_params* params, int32_t* status) {
  if (params_validate(params)) return NULL;
  oracle_session* s = (oracle_session*)calloc(1, sizeof *s);
  s->p = *params;
  if (lp_from_abi(lpin, &s->orig)) {
    lp_free(&s->orig);
    free(s);
    return NULL;
  }
  const lp_t* o = &s->orig;
  s->n = o->n;
  s->m1 = o->m1;
  s->m = o->m1 + o->m2;
  /* SolveLoop ctor (solver.hpp:636-646) */
  s->norms.rhs_norm = sqrt(sqnorm(o->h, o->m1) + sqnorm(o->b, o->m2));
  s->norms.obj_norm = norm2(o->c, o->n);
  csr_t stacked = csr_vstack(&o->G, &o->A);
  s->s = make_scaling(&stacked, params->scaling, params->ruiz_iterations, params->pock_chambolle_alpha);
  csr_free(&stacked);
  s->scaled = apply_scaling(o, &s->s);
  s->K = csr_vstack(&s->scaled.G, &s->scaled.A);
  s->q = dvec(s->m);
  if (o->m1) memcpy(s->q, s->scaled.h, (size_t)o->m1 * sizeof(double));
  if (o->m2) memcpy(s->q + o->m1, s->scaled.b, (size_t)o->m2 * sizeof(double));

  /* run() prologue (solver.hpp:760-792) */
  clock_gettime(CLOCK_MONOTONIC, &s->t0);
  const int64_t n = s->n, m = s->m;
  s->x = dzeros(n);
  s->y = dzeros(m);
  s->xs = dzeros(n);
  s->ys = dzeros(m);
  s->kx = dvec(m);
  s->kty = dvec(n);
  spmv(&s->K, s->x, s->kx);
  spmv_t(&s->K, s->y, s->kty);
  const double mabs = max_abs_entry(&s->K);
  s->eta_hat = mabs > 0.0 ? 1.0 / mabs : 1.0;
  s->eta = s->eta_hat;
  {
    /* initialize_primal_weight (solver.hpp:293-300) on the scaled problem */
    const double cn = norm2(s->scaled.c, n), qn = norm2(s->q, m);
    const double w = (cn > params->eps_zero && qn > params->eps_zero) ? cn / qn : 1.0;
    s->omega = sclamp(w, params->omega_min, params->omega_max);
  }
  s->ax = dzeros(n);
  s->ay = dzeros(m);
  s->wsum = 0.0;
  s->dx_last = dzeros(n);
  s->dy_last = dzeros(m);
  s->xn = dvec(n);
  s->yn = dvec(m);
  s->kxn = dvec(m);
  {
    double *ux, *uy;
    unscale(s, s->x, s->y, &ux, &uy);
    point_eval_t ev0 = evaluate_point(o, ux, uy);
    s->kkt_epoch_start = kkt_weighted(&ev0.res, s->omega);
    s->kkt_last_candidate = s->kkt_epoch_start;
    if (termination_met(&ev0.res, params->eps_optimal, &s->norms)) {
      finish(s, PDLP_STATUS_OPTIMAL, ux, uy, &ev0.res, ev0.red, NULL);
    } else {
      free(ux);
      free(uy);
      reduced_free(&ev0.red);
    }
  }
  if (status) *status = s->finished ? s->info.status : PDLP_STATUS_RUNNING;
  return s;
}

/* Loop body of SolveLoop::run (solver.hpp:794-928), n accepted iterations. */
int oracle_run(oracle_session* s, int64_t count, int32_t* status) {
  const int64_t n = s->n, m = s->m;
  double* kty_next = dvec(n);
  for (int64_t done = 0; !s->finished && done < count; ++done) {
    if (s->total >= s->p.iteration_limit) {
      finish_candidate(s, PDLP_STATUS_ITERATION_LIMIT, NULL);
      break;
    }
    if (elapsed(s) >= s->p.time_limit_seconds) {
      finish_candidate(s, PDLP_STATUS_TIME_LIMIT, NULL);
      break;
    }
    step_out_t st = adaptive_step(s, s->total + 1, kty_next);
    if (st.failure) {
      char msg[128];
      snprintf(msg, sizeof msg, "non-finite iterate in adaptive step at iteration %lld",
               (long long)s->total);
      finish_candidate(s, PDLP_STATUS_NUMERICAL_ERROR, msg);
      break;
    }
    if (s->p.record_step_log) {
      pdlp_step_log_entry e = {s->total + 1, s->omega, st.eta_acc, st.eta_bar, st.eta_next, st.mov, st.inter};
      push_step(s, e);
    }
    for (int64_t i = 0; i < n; ++i) s->dx_last[i] = s->xn[i] - s->x[i];
    for (int64_t i = 0; i < m; ++i) s->dy_last[i] = s->yn[i] - s->y[i];
    double* t;
    t = s->x; s->x = s->xn; s->xn = t;
    t = s->y; s->y = s->yn; s->yn = t;
    t = s->kx; s->kx = s->kxn; s->kxn = t;
    t = s->kty; s->kty = kty_next; kty_next = t;
    s->eta = st.eta_acc;
    s->eta_hat = st.eta_next;
    s->total += 1;
    s->inner += 1;
    s->wsum += s->eta;
    avg_add(s->ax, s->x, n, s->eta, s->wsum);
    avg_add(s->ay, s->y, m, s->eta, s->wsum);

    if (s->inner % s->p.evaluation_frequency != 0) continue;

    evaluation_t ev = evaluate_candidates(s);
    if (ev.terminated) {
      finish(s, PDLP_STATUS_OPTIMAL, ev.cand_ux, ev.cand_uy, &ev.cand_eval.res, ev.cand_eval.red, NULL);
      ev.cand_ux = ev.cand_uy = NULL;
      memset(&ev.cand_eval.red, 0, sizeof ev.cand_eval.red);
      evaluation_free(&ev);
      break;
    }
    if (ev.other_terminated) {
      finish(s, PDLP_STATUS_OPTIMAL, ev.other_ux, ev.other_uy, &ev.other_eval.res, ev.other_eval.red, NULL);
      ev.other_ux = ev.other_uy = NULL;
      memset(&ev.other_eval.red, 0, sizeof ev.other_eval.red);
      evaluation_free(&ev);
      break;
    }
    {
      /* infeasibility rays (solver.hpp:853-885) */
      double* nx = dvec(n);
      double* ny = dvec(m);
      const double inv_t = 1.0 / (double)s->inner;
      for (int64_t i = 0; i < n; ++i) nx[i] = inv_t * (s->x[i] - s->xs[i]);
      for (int64_t i = 0; i < m; ++i) ny[i] = inv_t * (s->y[i] - s->ys[i]);
      double *dux, *duy, *nux, *nuy;
      unscale(s, s->dx_last, s->dy_last, &dux, &duy);
      unscale(s, nx, ny, &nux, &nuy);
      free(nx);
      free(ny);
      cert_t cert = certificate_from_ray(&s->orig, dux, duy, s->p.eps_infeasible, s->p.eps_zero);
      if (!cert.status) cert = certificate_from_ray(&s->orig, nux, nuy, s->p.eps_infeasible, s->p.eps_zero);
      free(dux);
      free(duy);
      free(nux);
      free(nuy);
      if (cert.status) {
        double* px;
        double* py;
        reduced_t red;
        if (cert.status == PDLP_STATUS_PRIMAL_INFEASIBLE) {
          px = dzeros(n);
          py = cert.ray_y;
          red = cert.red;
        } else {
          px = cert.ray_x;
          py = dzeros(m);
          double* slack = dual_slack(&s->orig, py);
          red = reduced_from_slack(slack, s->orig.l, s->orig.u, n);
          free(slack);
        }
        finish(s, cert.status, px, py, &ev.cand_eval.res, red, NULL);
        s->info.has_certificate = 1;
        evaluation_free(&ev);
        break;
      }
    }
    const double prev = s->kkt_last_candidate;
    const int crit = should_restart(ev.kkt_cand, prev, s->kkt_epoch_start, s->inner, s->total, &s->p);
    s->kkt_last_candidate = ev.kkt_cand;
    if (crit == PDLP_RESTART_NONE) {
      evaluation_free(&ev);
      continue;
    }
    pdlp_restart_event e;
    memset(&e, 0, sizeof e);
    e.total_iterations = s->total;
    e.epoch_length = s->inner;
    e.criterion = crit;
    e.candidate_is_average = ev.cand_is_avg;
    e.kkt_candidate = ev.kkt_cand;
    e.kkt_previous_candidate = prev;
    e.kkt_epoch_start = s->kkt_epoch_start;
    e.omega_before = s->omega;
    /* restart block (solver.hpp:907-927) */
    double dxs = 0.0, dys = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double d = ev.cand_x[i] - s->xs[i];
      dxs += d * d;
    }
    for (int64_t i = 0; i < m; ++i) {
      const double d = ev.cand_y[i] - s->ys[i];
      dys += d * d;
    }
    memcpy(s->xs, ev.cand_x, (size_t)n * sizeof(double));
    memcpy(s->ys, ev.cand_y, (size_t)m * sizeof(double));
    memcpy(s->x, ev.cand_x, (size_t)n * sizeof(double));
    memcpy(s->y, ev.cand_y, (size_t)m * sizeof(double));
    spmv(&s->K, s->x, s->kx);
    spmv_t(&s->K, s->y, s->kty);
    s->outer += 1;
    s->inner = 0;
    s->wsum = 0.0;
    memset(s->ax, 0, (size_t)n * sizeof(double));
    memset(s->ay, 0, (size_t)m * sizeof(double));
    {
      /* update_primal_weight (solver.hpp:305-325) */
      const double dx = sqrt(dxs), dy = sqrt(dys);
      double w = s->omega;
      if (dx > s->p.eps_zero && dy > s->p.eps_zero)
        w = exp(s->p.theta_smoothing * log(dy / dx) + (1.0 - s->p.theta_smoothing) * log(s->omega));
      s->omega = sclamp(w, s->p.omega_min, s->p.omega_max);
    }
    e.omega_after = s->omega;
    push_restart(s, e);
    s->kkt_epoch_start = kkt_weighted(&ev.cand_eval.res, s->omega);
    s->kkt_last_candidate = s->kkt_epoch_start;
    evaluation_free(&ev);
  }
  free(kty_next);
  if (status) *status = s->finished ? s->info.status : PDLP_STATUS_RUNNING;
  return PDLP_OK;
}

int oracle_get_iterate(oracle_session* s, double* x, double* y, double* kx, double* kty,
                       int64_t* counters, double* scalars) {
  if (x) memcpy(x, s->x, (size_t)s->n * sizeof(double));
  if (y) memcpy(y, s->y, (size_t)s->m * sizeof(double));
  if (kx) memcpy(kx, s->kx, (size_t)s->m * sizeof(double));
  if (kty) memcpy(kty, s->kty, (size_t)s->n * sizeof(double));
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
    scalars[3] = s->wsum;
  }
  return PDLP_OK;
}

int oracle_result(oracle_session* s, pdlp_result_info* info, double* x, double* y, double* lambda,
                  double* lambda_pos, double* lambda_neg, pdlp_step_log_entry* step_log,
                  int64_t step_cap, pdlp_restart_event* restart_log, int64_t restart_cap) {
  if (!s->finished) return fail(PDLP_ESTATE, "oracle_result: solve not finished");
  if (info) *info = s->info;
  if (x) memcpy(x, s->rx, (size_t)s->n * sizeof(double));
  if (y) memcpy(y, s->ry, (size_t)s->m * sizeof(double));
  if (lambda) memcpy(lambda, s->rred.lambda, (size_t)s->n * sizeof(double));
  if (lambda_pos) memcpy(lambda_pos, s->rred.pos, (size_t)s->n * sizeof(double));
  if (lambda_neg) memcpy(lambda_neg, s->rred.neg, (size_t)s->n * sizeof(double));
  if (step_log)
    for (int64_t i = 0; i < s->slog_n && i < step_cap; ++i) step_log[i] = s->slog[i];
  if (restart_log)
    for (int64_t i = 0; i < s->rlog_n && i < restart_cap; ++i) restart_log[i] = s->rlog[i];
  return PDLP_OK;
}

void oracle_end(oracle_session* s) {
  if (!s) return;
  lp_free(&s->orig);
  free(s->s.row);
  free(s->s.col);
  csr_free(&s->scaled.G);
  csr_free(&s->scaled.A);
  free(s->scaled.c);
  free(s->scaled.h);
  free(s->scaled.b);
  free(s->scaled.l);
  free(s->scaled.u);
  csr_free(&s->K);
  double* bufs[] = {s->q, s->x, s->y, s->kx, s->kty, s->xs, s->ys, s->ax, s->ay,
                    s->dx_last, s->dy_last, s->xn, s->yn, s->kxn, s->rx, s->ry};
  for (size_t i = 0; i < sizeof bufs / sizeof bufs[0]; ++i) free(bufs[i]);
  reduced_free(&s->rred);
  free(s->slog);
  free(s->rlog);
  free(s);
}

int oracle_solve(const pdlp_lp* lp, const pdlp_params* params, pdlp_result_info* info, double* x,
                 double* y, double* lambda, double* lambda_pos, double* lambda_neg,
                 pdlp_step_log_entry* step_log, int64_t step_cap, pdlp_restart_event* restart_log,
                 int64_t restart_cap) {
  int32_t st;
  oracle_session* s = oracle_begin(lp, params, &st);
  if (!s) return PDLP_EINVAL;
  while (!s->finished) oracle_run(s, INT64_MAX, &st);
  int rc = oracle_result(s, info, x, y, lambda, lambda_pos, lambda_neg, step_log, step_cap,
                         restart_log, restart_cap);
  oracle_end(s);
  return rc;
}

int oracle_scaling(const pdlp_lp* lpin, const pdlp_params* params, double* row_scale, double* col_scale) {
  lp_t lp;
  int rc = lp_from_abi(lpin, &lp);
  if (rc) {
    lp_free(&lp);
    return rc;
  }
  csr_t k = csr_vstack(&lp.G, &lp.A);
  scaling_t s = make_scaling(&k, params->scaling, params->ruiz_iterations, params->pock_chambolle_alpha);
  memcpy(row_scale, s.row, (size_t)k.rows * sizeof(double));
  memcpy(col_scale, s.col, (size_t)k.cols * sizeof(double));
  free(s.row);
  free(s.col);
  csr_free(&k);
  lp_free(&lp);
  return PDLP_OK;
}

int oracle_spmv(const pdlp_csr* a, const double* x, double* out) {
  csr_t m;
  int rc = csr_from_abi(a, &m);
  if (!rc) spmv(&m, x, out);
  csr_free(&m);
  return rc;
}

int oracle_spmv_transpose(const pdlp_csr* a, const double* y, double* out) {
  csr_t m;
  int rc = csr_from_abi(a, &m);
  if (!rc) spmv_t(&m, y, out);
  csr_free(&m);
  return rc;
}

int oracle_transpose(const pdlp_csr* a, int64_t* off, int64_t* col, double* val) {
  csr_t m, t;
  int rc = csr_from_abi(a, &m);
  if (!rc) rc = csr_transpose(&m, &t);
  if (!rc) {
    memcpy(off, t.off, (size_t)(t.rows + 1) * sizeof(int64_t));
    memcpy(col, t.col, (size_t)t.nnz * sizeof(int64_t));
    memcpy(val, t.val, (size_t)t.nnz * sizeof(double));
    csr_free(&t);
  }
  csr_free(&m);
  return rc;
}

int oracle_check_termination(const pdlp_lp* lpin, const double* x, const double* y, double eps,
                             double* out) {
  lp_t lp;
  int rc = lp_from_abi(lpin, &lp);
  if (rc) {
    lp_free(&lp);
    return rc;
  }
  term_norms_t nn;
  nn.rhs_norm = sqrt(sqnorm(lp.h, lp.m1) + sqnorm(lp.b, lp.m2));
  nn.obj_norm = norm2(lp.c, lp.n);
  point_eval_t ev = evaluate_point(&lp, x, y);
  out[0] = termination_met(&ev.res, eps, &nn);
  out[1] = ev.res.prn;
  out[2] = ev.res.drn;
  out[3] = ev.res.pobj;
  out[4] = ev.res.dobj;
  reduced_free(&ev.red);
  lp_free(&lp);
  return PDLP_OK;
}

/* pdhg_raw_step (solver.hpp:335-358) on to_saddle(lp) (lp_model.hpp:88-98):
 * x' = clamp(x - tau (c - K'y)), then y' = proj(y + sigma (q - K (2x' - x))). */
int oracle_pdhg_raw_step(const pdlp_lp* lpin, const double* x, const double* y, double tau, double sigma,
                         double* xo, double* yo) {
  lp_t lp;
  int rc = lp_from_abi(lpin, &lp);
  if (rc) {
    lp_free(&lp);
    return rc;
  }
  csr_t K = csr_vstack(&lp.G, &lp.A);
  const int64_t n = lp.n, m = lp.m1 + lp.m2;
  double* kty = dvec(n);
  double* ext = dvec(n);
  double* kext = dvec(m);
  spmv_t(&K, y, kty);
  for (int64_t i = 0; i < n; ++i) {
    const double v = x[i] - tau * (lp.c[i] - kty[i]);
    xo[i] = smin(smax(v, lp.l[i]), lp.u[i]); /* clamp_to_box, vector_ops.hpp:52-58 */
  }
  for (int64_t i = 0; i < n; ++i) ext[i] = 2.0 * xo[i] - x[i];
  spmv(&K, ext, kext);
  for (int64_t i = 0; i < m; ++i) {
    const double q = i < lp.m1 ? lp.h[i] : lp.b[i - lp.m1];
    yo[i] = y[i] + sigma * (q - kext[i]);
  }
  project_dual(yo, lp.m1);
  free(kty);
  free(ext);
  free(kext);
  csr_free(&K);
  lp_free(&lp);
  return PDLP_OK;
}

int oracle_from_triplets(int64_t rows, int64_t cols, int64_t nt, const int64_t* tr, const int64_t* tc,
                         const double* tv, int64_t* off, int64_t* col, double* val, int64_t* nnz_out) {
  csr_t m;
  int rc = csr_from_triplets(rows, cols, nt, tr, tc, tv, &m);
  if (rc) return rc;
  memcpy(off, m.off, (size_t)(rows + 1) * sizeof(int64_t));
  memcpy(col, m.col, (size_t)m.nnz * sizeof(int64_t));
  memcpy(val, m.val, (size_t)m.nnz * sizeof(double));
  *nnz_out = m.nnz;
  csr_free(&m);
  return PDLP_OK;
}
