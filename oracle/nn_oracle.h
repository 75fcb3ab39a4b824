/* ORACLE — test infrastructure only (tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg are the only callers; the product never links
 * it).  Plain-C restatement of the reference's Nested Neumann hot path,
 * /root/reference/proj/src/{kernels,solver,factorized}.cpp, on interleaved
 * complex128 row-major arrays, with the reference's exact operation order
 * (ascending-k products, serial Frobenius sums) so that it reproduces the
 * reference bit-for-bit.  Pinned against the reference itself
 * (oracle/_ref/libnnref.so) and against tests/golden/ fixtures.
 *
 * Status codes follow include/nnb.h (0 ok, 1 shape, 2 domain, 3 divergence).
 */
#ifndef NN_ORACLE_H
#define NN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

void nno_set_threads(int threads);
int nno_matmul_z(const double* a, const double* b, int64_t m, int64_t k, int64_t n, double* c);
double nno_frobenius_z(const double* m, int64_t count);
int nno_residual_eps_z(const double* x, const double* a, int64_t n, double* eps);
int nno_nn_step_z(const double* x, const double* a, int64_t n, int64_t depth_l, double* out);
int nno_ns_sum_z(const double* x0, const double* a, int64_t n, int64_t order, double* out);
int nno_chain_z(const double* a, int64_t n, const double* x0, int p, int max_iters, double tol,
                double* x_out, double* eps_hist, int* iters_out, int* fail_iter);
int nno_batched_z(int mode, const double* a, int64_t batch, int64_t n, int p, int iters,
                  double* x_out, double* eps_last, int threads);
int nno_spmv_block_z(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n,
                     const double* x, int64_t k, double* out);
int nno_sparse_factorized_z(const int64_t* row_ptr, const int32_t* col, const double* val,
                            int64_t n, const double* b, int64_t k, int64_t gamma, double theta,
                            double* x_out, int64_t* spmv_count, int* fail_index);

void nno_gaussian(uint64_t seed, int64_t count, double* out);
int nno_random_spd(int64_t n, double cond, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif
#endif
