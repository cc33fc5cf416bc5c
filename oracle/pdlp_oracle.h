/* pdlp_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference CPU solver's hot path (pdhglp,
 * /root/reference/proj/include/pdhglp/{sparse_matrix,vector_ops,lp_model,
 * scaling,solver}.hpp). It is the *checker* for the CUDA product path: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it. The product library never links it.
 *
 * Parity pin: oracle/ref_harness.cpp compiles the reference headers from
 * /root/reference into oracle/_ref/libpdhglp_ref.so exposing the same entry
 * points (prefix ref_ instead of oracle_); tests/test_oracle_pin.py checks the
 * two bitwise, and tests/golden/ holds vectors generated from the reference.
 *
 * Types are the product's C-ABI structs (include/pdlp_b200.h) so one ctypes
 * description drives the oracle, the reference harness and the GPU library.
 */
#ifndef PDLP_ORACLE_H_
#define PDLP_ORACLE_H_

#include "../include/pdlp_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_session oracle_session;

/* Full solve: pdhglp::solve (solver.hpp:935-940). Output buffers may be NULL. */
int oracle_solve(const pdlp_lp* lp, const pdlp_params* params, pdlp_result_info* info,
                 double* x, double* y, double* lambda, double* lambda_pos,
                 double* lambda_neg, pdlp_step_log_entry* step_log, int64_t step_cap,
                 pdlp_restart_event* restart_log, int64_t restart_cap);

/* Stepwise loop with the same semantics as pdlp_iterate_* of the product. */
oracle_session* oracle_begin(const pdlp_lp* lp, const pdlp_params* params, int32_t* status);
int oracle_run(oracle_session* s, int64_t n, int32_t* status);
int oracle_get_iterate(oracle_session* s, double* x, double* y, double* kx, double* kty,
                       int64_t* counters, double* scalars);
int oracle_result(oracle_session* s, pdlp_result_info* info, double* x, double* y,
                  double* lambda, double* lambda_pos, double* lambda_neg,
                  pdlp_step_log_entry* step_log, int64_t step_cap,
                  pdlp_restart_event* restart_log, int64_t restart_cap);
void oracle_end(oracle_session* s);

/* Preconditioner of vstack(G, A) (scaling.hpp:117-132). */
int oracle_scaling(const pdlp_lp* lp, const pdlp_params* params, double* row_scale,
                   double* col_scale);

/* Sequential kernels (sparse_matrix.hpp:117-178). */
int oracle_spmv(const pdlp_csr* a, const double* x, double* out);
int oracle_spmv_transpose(const pdlp_csr* a, const double* y, double* out);
/* Explicit transpose; outputs sized num_cols+1 / nnz / nnz. */
int oracle_transpose(const pdlp_csr* a, int64_t* row_offsets, int64_t* col_indices,
                     double* values);
/* CsrMatrix::from_triplets (sparse_matrix.hpp:57-108); outputs sized rows+1 / nt / nt;
 * *nnz_out receives the stored count. */
int oracle_from_triplets(int64_t rows, int64_t cols, int64_t nt, const int64_t* tr,
                         const int64_t* tc, const double* tv, int64_t* row_offsets,
                         int64_t* col_indices, double* values, int64_t* nnz_out);

/* check_termination + reduced_costs at an unscaled point (solver.hpp:231-249,
 * lp_model.hpp:192-195): out = {terminated, prn, drn, pobj_raw, dobj_raw}. */
int oracle_check_termination(const pdlp_lp* lp, const double* x, const double* y, double eps,
                             double* out);

/* pdhg_raw_step (solver.hpp:335-358) on the unscaled saddle problem. */
int oracle_pdhg_raw_step(const pdlp_lp* lp, const double* x, const double* y, double tau, double sigma,
                         double* x_out, double* y_out);

const char* oracle_last_error(void);

/* Summation-order probe: 0 (default) the reference's sequential step-size
 * sums, 1 pairwise trees (process-wide; tests only). */
void oracle_set_sum_order(int order);

#ifdef __cplusplus
}
#endif
#endif
