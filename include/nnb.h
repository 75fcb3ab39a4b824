/*
 * nnb.h — C-ABI of the B200-native Nested Neumann hot path (libnnb.so).
 *
 * This is the drop-in boundary: plain pointers and sizes, no torch or C++
 * types.  The reference C++ API (/root/reference/proj/include/nn/*.hpp) is
 * re-implemented on top of these entry points by the C++ layer in
 * paper_2212_02406_b200/dropin/ (namespace nn), and the Python mirror in
 * paper_2212_02406_b200/__init__.py binds them with ctypes.
 *
 * Conventions:
 *  - Matrices are row-major.  `_d` entry points take float64; `_z` entry
 *    points take complex128 interleaved (re, im), i.e. std::complex<double>.
 *  - Every matrix/vector pointer may be HOST or DEVICE memory; the library
 *    detects which (cudaPointerGetAttributes) and stages host data through
 *    device buffers itself.  Caller memory is never freed or retained.
 *  - `stream` is a cudaStream_t (NULL = the legacy default stream).
 *    Host outputs are complete when the call returns; device outputs are
 *    complete in stream order.
 *  - Return value: NNB_OK or an NNB_ERR_* code; nnb_last_error() gives a
 *    thread-local message.  There is no CPU fallback: without a CUDA device
 *    every compute entry point returns NNB_ERR_NODEVICE.
 *  - Reductions are deterministic (fixed order, no floating-point atomics):
 *    results are bit-reproducible run to run on a fixed device count.
 */
#ifndef NNB_H
#define NNB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NNB_ABI_VERSION 1

enum nnb_status {
  NNB_OK = 0,
  NNB_ERR_SHAPE = 1,        /* nn::ShapeError       proj/include/nn/errors.hpp:15-17 */
  NNB_ERR_DOMAIN = 2,       /* nn::DomainError      errors.hpp:20-22 */
  NNB_ERR_DIVERGENCE = 3,   /* nn::DivergenceError  errors.hpp:45-49 (index in result) */
  NNB_ERR_CONTRACTION = 4,  /* nn::ContractionError errors.hpp:40-42 */
  NNB_ERR_PLAN = 5,         /* nn::PlanError        errors.hpp:52-54 */
  NNB_ERR_BUDGET = 6,       /* nn::BudgetError      errors.hpp:57-59 */
  NNB_ERR_CUDA = 7,
  NNB_ERR_NCCL = 8,
  NNB_ERR_OOM = 9,
  NNB_ERR_NODEVICE = 10,
  NNB_ERR_SINGULAR = 11     /* nn::SingularMatrixError errors.hpp (pivot index out-param) */
};

/* Operand order of the nest ("Product order").
 * NORTHSTAR: R = I - A X,  X' = X (I + R + ... + R^p)  (right-multiply Horner)
 * REFERENCE: P = I - X A,  X' = (I + P + ... + P^p) X  (proj/src/solver.cpp:93-103) */
/* SYMMETRIC: the NORTHSTAR order for real A == A^T and X0 == X0^T (every
 *   built-in X0 of a symmetric A qualifies; a given X0 is checked).  The
 *   Horner products X·S(R)·R are then symmetric (push-through) and compute
 *   only their upper tile triangle, mirrored: p+1 products per nest cost
 *   about 1 + p/2.  R = I - A·X stays a full product.  Mirrored products
 *   run while eps >= 1e-4 and falling; later nests use full products, so
 *   the residual floor and the nest count to a tolerance are NORTHSTAR's
 *   (a mirrored nest's floor is ~kappa·u).  Results agree with NORTHSTAR
 *   to rounding.  NNB_ERR_DOMAIN when A or a given X0 is not
 *   symmetric, and for complex chains and the sharded chain. */
enum nnb_order { NNB_ORDER_NORTHSTAR = 0, NNB_ORDER_REFERENCE = 1, NNB_ORDER_SYMMETRIC = 2 };

/* Initial iterate. */
enum nnb_x0 {
  NNB_X0_GIVEN = 0,           /* caller's X0 */
  NNB_X0_SCALED_IDENTITY = 1, /* x0_scale * I (nn_invert: phi0 = I, proj/src/solver.cpp:138) */
  NNB_X0_TRANSPOSE_NORM = 2,  /* A^T / (||A||_1 ||A||_inf)   (BASELINE configs 0,2,3) */
  NNB_X0_JACOBI = 3           /* diag(A)^-1                  (BASELINE config 1) */
};

typedef struct nnb_chain_config {
  int32_t depth_p;        /* inception depth p (reference depth_L); 0 = identity map */
  int32_t max_iters;      /* nest budget (reference max_nests) */
  double tol;             /* stop when eps < tol; <= 0 runs exactly max_iters nests */
  int32_t order;          /* enum nnb_order */
  int32_t x0_kind;        /* enum nnb_x0 */
  double x0_scale;        /* NNB_X0_SCALED_IDENTITY only */
  int32_t final_residual; /* 1: eps after the last nest is computed (k(p+1)+1 products) */
} nnb_chain_config;

typedef struct nnb_chain_result {
  int32_t iters;      /* nests performed */
  int32_t fail_iter;  /* 1-based nest whose product went non-finite (NNB_ERR_DIVERGENCE) */
  int32_t stopped;    /* 0 = tolerance, 1 = max_iters */
  int32_t products;   /* dense N^3 products executed (incl. residual products) */
  double last_eps;    /* last recorded eps */
  double device_ms;   /* device time of the chain (CUDA events, excludes staging) */
} nnb_chain_result;

/* ---- library ---------------------------------------------------------- */
int nnb_abi_version(void);
const char* nnb_last_error(void);
int nnb_device_count(void);
/* Launch count of this library's kernels since load (for bench gpu_launches). */
uint64_t nnb_kernel_launches(void);
/* Returns the library's cached work buffers (the current device's stream-ordered pool,
 * kept across calls) to the driver, after a device synchronisation. */
int nnb_release_cached_memory(void);

/* Arithmetic mode of the calling thread.
 * NNB_ARITH_FAST (default): the faster of the two FP64-accurate product
 *   paths per product — the int8 emulation below for real products with
 *   M, N, K >= 1024 and M·N·K >= 3072^3, DMMA otherwise (complex and K-split
 *   products always DMMA); agrees with the reference to ~1e-15 relative.
 * NNB_ARITH_DMMA: every product on the FP64 tensor pipe (DMMA.8x8x4).
 * NNB_ARITH_REFERENCE: real dense products as ascending-k, explicitly
 *   rounded CUDA-core loops, serial Frobenius sums and the reference's own
 *   nest sequence — BIT-IDENTICAL to the reference for real data
 *   (a verification mode; complex products keep the 4-GEMM path).
 * NNB_ARITH_OZAKI: real dense products emulated on the int8 tensor cores
 *   (tcgen05.mma kind::i8, Ozaki scheme II with 16 moduli: csrc/ozaki.cu):
 *   every entry keeps 53 bits relative to its row's (column's) largest, the
 *   integer products are exact; same parity gate as FAST (X within 1e-10,
 *   identical nest counts).  Complex products keep the DMMA path.
 * The sparse path is bit-identical in every mode. */
enum nnb_arith { NNB_ARITH_FAST = 0, NNB_ARITH_REFERENCE = 1, NNB_ARITH_OZAKI = 2, NNB_ARITH_DMMA = 3 };
int nnb_set_arithmetic(int32_t mode);
int32_t nnb_get_arithmetic(void);
/* The next real nnb_nn_chain_d of the calling thread (with final_residual = 1) copies
 * its final residual R = I − A·X — the product eps_last is computed from — into the
 * device buffer R_out (n×n, leading dimension ldr).  A test hook for sampling the
 * chain's own R at sizes no CPU oracle reaches (SURVEY §8(c) C4 item iii). */
int nnb_chain_capture_residual(double* R_out, int64_t ldr);
/* Most moduli (= int8 GEMMs per product) NNB_ARITH_OZAKI uses for inner dimension k; a
 * product uses fewer when its operands' L1/max ratios bound the integer product lower. */
int32_t nnb_ozaki_moduli(int64_t k);
/* Live timing of the emulation's kernels (for roofline reporting): while on, every
 * int8 GEMM / operand split / reconstruction launch is bracketed by CUDA events on its
 * stream.  nnb_ozaki_stats fills ms[3], work[3] (int8 ops; algorithmic bytes; bytes)
 * and launches[3] for the three classes, synchronising the recorded events. */
void nnb_ozaki_profile(int32_t on);
void nnb_ozaki_stats(double* ms, double* work, int64_t* launches, int32_t reset);

/* ---- dense kernels ------------------------------------------------------ */
/* C = A·B.  Replaces nn::matmul (proj/include/nn/kernels.hpp:20-21,
 * proj/src/kernels.cpp:137-162).  ld* are leading dimensions in elements. */
int nnb_gemm_d(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
               int64_t ldc, int64_t m, int64_t k, int64_t n, void* stream);
int nnb_gemm_z(const double* A, const double* B, double* C, int64_t m, int64_t k, int64_t n,
               void* stream);
/* C = A·Bᵀ with Bᵀ given as the n×k row-major matrix Bt (K-major B operand:
 * conflict-free fragment loads; also the Gram product B·Bᵀ without a copy). */
int nnb_gemm_nt_d(const double* A, int64_t lda, const double* Bt, int64_t ldbt, double* C, int64_t ldc,
                  int64_t m, int64_t k, int64_t n, void* stream);

/* out = alpha*A + beta*B + gamma*I (B nullable).  Replaces nn::add / sub /
 * scale / identity_minus / plus_identity (proj/include/nn/kernels.hpp:26-35). */
int nnb_axpby_d(double alpha, const double* A, double beta, const double* B, double gamma,
                double* out, int64_t rows, int64_t cols, void* stream);
int nnb_axpby_z(const double* alpha2, const double* A, const double* beta2, const double* B,
                const double* gamma2, double* out, int64_t rows, int64_t cols, void* stream);

/* out (cols×rows) = M^T (real) or M^H (complex interleaved), a tiled device
 * transpose.  Replaces nn::conjugate_transpose (proj/include/nn/kernels.hpp:37,
 * proj/src/kernels.cpp:223-229); used by the normal-equations solve. */
int nnb_transpose_d(const double* M, int64_t rows, int64_t cols, double* out, void* stream);
int nnb_conj_transpose_z(const double* M, int64_t rows, int64_t cols, double* out, void* stream);

/* Seeded test-matrix generators.
 * nnb_gaussian_stream: `count` draws of the reference's GaussianStream
 *   (proj/include/nn/rng.hpp:15-52; host code, the stream is sequential).
 * nnb_householder_q_d/_z: Q of the Householder QR of the n×n matrix A
 *   (proj/src/kernels.cpp:64-105), on the device.
 * nnb_random_spd_d: W = (Q·diag(lam))·Q^T symmetrised, Q = householder_q(G);
 *   with G drawn row-major from GaussianStream(seed) and lam the reference's
 *   log_uniform_spectrum this is nn::random_spd (kernels.cpp:352-381),
 *   bit-identical.
 * nnb_random_conditioned_z: A = (U·diag(sigma))·V^H, U, V = householder_q of
 *   the complex Gaussians GU, GV — nn::random_conditioned_complex
 *   (kernels.cpp:383-407), equal to a few ulps. */
int nnb_gaussian_stream(uint64_t seed, int64_t count, double* out);
int nnb_householder_q_d(const double* A, int64_t n, double* Q, void* stream);
int nnb_householder_q_z(const double* A, int64_t n, double* Q, void* stream);
int nnb_random_spd_d(const double* G, const double* lam, int64_t n, double* W, void* stream);
int nnb_random_conditioned_z(const double* GU, const double* GV, const double* sigma, int64_t n, double* A,
                             void* stream);

/* Gauss–Jordan inverse with partial pivoting: nn::direct_inverse_oracle
 * (proj/include/nn/kernels.hpp:67, proj/src/kernels.cpp:317-350), on the
 * device; bit-identical to the reference for real input.  NNB_ERR_SINGULAR
 * with *pivot_index when a pivot magnitude is <= 1e-13·||M||_F. */
int nnb_direct_inverse_d(const double* M, int64_t n, double* out, int32_t* pivot_index, void* stream);
int nnb_direct_inverse_z(const double* M, int64_t n, double* out, int32_t* pivot_index, void* stream);

/* ||M||_F (proj/include/nn/kernels.hpp:42) and trace (:40). */
int nnb_frobenius_d(const double* M, int64_t count, double* out, void* stream);
int nnb_frobenius_z(const double* M, int64_t count, double* out, void* stream);
int nnb_trace_z(const double* M, int64_t n, double* out2, void* stream);

/* eps = ||I - X·A||_F / sqrt(n).  Replaces nn::residual_epsilon
 * (proj/include/nn/solver.hpp:55, proj/src/solver.cpp:72-75). */
int nnb_residual_eps_d(const double* X, const double* A, int64_t n, double* eps, void* stream);
int nnb_residual_eps_z(const double* X, const double* A, int64_t n, double* eps, void* stream);

/* X0 builders (not in the reference). */
int nnb_x0_d(const double* A, int64_t n, int32_t x0_kind, double x0_scale, double* X0,
             void* stream);

/* ---- the Nested Neumann chain ------------------------------------------- */
/* Runs nests of depth p on A from X0 until eps < tol or max_iters nests,
 * eps recorded before every nest (and after the last if final_residual):
 * the loop of nn_invert (proj/src/solver.cpp:138-159) / SURVEY.md §8(c).
 * eps_hist: host array of max_iters+1 doubles (nullable).
 * X0 is read only for NNB_X0_GIVEN.  X_out receives the final iterate. */
int nnb_nn_chain_d(const double* A, int64_t n, const double* X0, const nnb_chain_config* cfg,
                   double* X_out, double* eps_hist, nnb_chain_result* result, void* stream);
int nnb_nn_chain_z(const double* A, int64_t n, const double* X0, const nnb_chain_config* cfg,
                   double* X_out, double* eps_hist, nnb_chain_result* result, void* stream);

/* One nest in reference order on (phi, W~): nn::nn_step
 * (proj/include/nn/solver.hpp:68-69).  depth 0 copies phi. */
int nnb_nn_step_d(const double* phi, const double* w, int64_t n, int32_t depth, double* out,
                  void* stream);
int nnb_nn_step_z(const double* phi, const double* w, int64_t n, int32_t depth, double* out,
                  void* stream);

/* Truncated Neumann series sum_{j=0}^{order} P^j phi0, P = I - phi0 W~:
 * nn::ns_sum (proj/include/nn/solver.hpp:61-62, proj/src/solver.cpp:77-91).
 * products_out (nullable) receives the reference's product tally. */
int nnb_ns_sum_d(const double* phi0, const double* w, int64_t n, int64_t order, double* out,
                 double* products_out, void* stream);
int nnb_ns_sum_z(const double* phi0, const double* w, int64_t n, int64_t order, double* out,
                 double* products_out, void* stream);

/* ---- product-form schedules on the same GEMM -- */
/* Factorized Neumann series of order gamma = 2^s − 1,
 * prod_{n<s} (I + P^{2^n}) phi0 with P = I − phi0 W~: nn::ns_factorized
 * (proj/include/nn/factorized.hpp:48-54, proj/src/factorized.cpp:42-61). */
int nnb_ns_factorized_d(const double* phi0, const double* w, int64_t n, int64_t gamma, double* out,
                        double* products_out, void* stream);
int nnb_ns_factorized_z(const double* phi0, const double* w, int64_t n, int64_t gamma, double* out,
                        double* products_out, void* stream);
/* p^exponent by square-and-multiply: nn::power_ladder (kernels.hpp:86-89). */
int nnb_power_ladder_d(const double* p, int64_t n, uint64_t exponent, double* out, double* products_out,
                       void* stream);
int nnb_power_ladder_z(const double* p, int64_t n, uint64_t exponent, double* out, double* products_out,
                       void* stream);
/* Non-recursive product form of i nests of depth L: nn::nn_explicit
 * (proj/include/nn/solver.hpp:87-92, proj/src/solver.cpp:176-199). */
int nnb_nn_explicit_d(const double* phi0, const double* w, int64_t n, int64_t nests_i, int64_t depth_L,
                      double* out, double* products_out, void* stream);
int nnb_nn_explicit_z(const double* phi0, const double* w, int64_t n, int64_t nests_i, int64_t depth_L,
                      double* out, double* products_out, void* stream);

/* ---- batched small complex systems (massive-MIMO Gram inversion) ------- */
/* batch independent n×n complex128 systems (n == 16), X0 = diag(A)^-1,
 * `iters` nests of depth p in reference order (nn_step per system) and the
 * residual after the last nest in eps_last (nullable, host or device).
 * A system whose A is stored exactly Hermitian (A == A^H bit for bit, as
 * the massive-MIMO Gram H^H·H + s²·I is) runs its Horner products on three
 * of four 8×8 tiles: each is Hermitian by push-through.  Results agree with
 * the full products to rounding; other systems take the full products. */
int nnb_nn_batched_z(const double* A, int64_t batch, int32_t n, int32_t p, int32_t iters,
                     double* X_out, double* eps_last, void* stream);
/* Neumann-series baseline of `order` terms from the same X0 (ns_sum). */
int nnb_ns_batched_z(const double* A, int64_t batch, int32_t n, int32_t order, double* X_out,
                     void* stream);

/* Fused massive-MIMO detection: per system
 * A = Hᴴ·H + sigma2·I (H: antennas × users, row-major complex128), z = Hᴴ·y,
 * X = NN inverse of A (Jacobi X0, `iters` nests of depth p), x̂ = X·z.
 * users == 16, antennas % 4 == 0.  X_out / eps_last nullable. */
int nnb_mimo_detect_z(const double* H, const double* y, int64_t batch, int32_t antennas, int32_t users,
                      double sigma2, int32_t p, int32_t iters, double* xhat_out, double* X_out,
                      double* eps_last, void* stream);

/* ---- sparse matrix-free factorized solve -------------------------------- */
/* Y = W·X for CSR W (int64 row_ptr, int32 col, float64 values) and an n×k
 * row-major block X: nn::spmv_block (proj/include/nn/kernels.hpp:91-92). */
int nnb_spmv_block_d(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n,
                     int64_t nnz, const double* X, int64_t k, double* Y, void* stream);
/* x = theta * prod_{f<s} (I + P^{2^f}) b with P = I - theta W, gamma = 2^s - 1
 * sparse applications per column: nn::solve_sparse_factorized
 * (proj/include/nn/factorized.hpp:74-76, proj/src/factorized.cpp:101-140).
 * spmv_count_out (nullable) = gamma*k; fail_factor_out gets the 0-based
 * factor index on NNB_ERR_DIVERGENCE. */
int nnb_sparse_factorized_d(const int64_t* row_ptr, const int32_t* col, const double* val,
                            int64_t n, int64_t nnz, const double* B, int64_t k, int64_t gamma,
                            double theta, double* X_out, int64_t* spmv_count_out,
                            int32_t* fail_factor_out, void* stream);
/* Bytes per nonzero of the CSR format the calling thread's last
 * nnb_sparse_factorized_d consumed: 1 when the operator has <= 256 distinct
 * (column - row, value) pairs (a pair dictionary, CSR-VI style: stencils and
 * other structured operators), 10 with int16 column deltas from the row, 12
 * with int32 columns; 0 before any solve.  Every format is bit-identical. */
int nnb_sparse_last_bytes_per_nnz(void);
/* Operator bytes one application of that solve streams from HBM: one code per row
 * (row dictionary: n bytes), the pair codes (slot-major ELL: width*n bytes, no row
 * offsets) or values and columns, plus row offsets. */
int64_t nnb_sparse_last_matrix_bytes(void);
/* That format by name: "row-dictionary-stencil-tb" (5-point stencils: row codes over
 * temporal-blocked passes of up to 8 applications, on one GPU or across row slabs of
 * whole grid rows), "row-dictionary" (<= 256 distinct whole rows over the ELL pair
 * codes, e.g. stencils: one uint8 code per row), "pair-dictionary-ell",
 * "pair-dictionary-csr", "csr-int16-delta", "csr-int32", "csr-int64-offsets";
 * "" before any solve. */
const char* nnb_sparse_last_format(void);
/* Device time (ms, CUDA events) of the calling thread's last row-slab solve without its
 * slab setup (the factor schedule and its halo exchanges); 0 before any. */
double nnb_sparse_last_solve_ms(void);

/* ---- contraction measurement (theta_trace's spectral estimate) ---------- */
/* Power iteration on M^H M from the unit probe v0 (complex128, length n):
 * nn::spectral_norm_estimate (proj/include/nn/kernels.hpp:51-53,
 * proj/src/kernels.cpp:244-269).  M complex128 n×n, host or device. */
int nnb_spectral_norm_z(const double* M, int64_t n, const double* v0, double tol,
                        int32_t max_iters, double* value, int32_t* converged, int32_t* iterations,
                        void* stream);
/* The same for the matrix-free shifted operator I − theta·W, W real CSR
 * (symmetric): nn::spectral_norm_estimate_shifted (kernels.hpp:57-61). */
int nnb_spectral_norm_shifted_csr(const int64_t* row_ptr, const int32_t* col, const double* val,
                                  int64_t n, int64_t nnz, double theta, const double* v0,
                                  double tol, int32_t max_iters, double* value,
                                  int32_t* converged, int32_t* iterations, void* stream);

/* ---- row-sharded chain across GPUs (one process per GPU) ---------------- */
/* rank g owns rows [row0_g, row0_g+rows_g) of A and X.  Per
 * nest: ring all-gather of X (NCCL send/recv on a side stream) overlapped
 * block by block with the K-split partial GEMMs of R_g = I_g − A_g·X, eps from
 * the per-rank Σ‖R_g‖² gathered and summed in rank order (identical on every
 * rank), ring all-gather of R overlapped with V_g = X_g + V_g·R (p×).
 * Not in the reference (single-process). */
typedef struct nnb_comm* nnb_comm_t;
#define NNB_UNIQUE_ID_BYTES 128
/* Partition used by the sharded entry points: blocks of whole 16-row units,
 * balanced, rank order.  Pure host arithmetic (no device needed). */
void nnb_partition_rows(int64_t n, int32_t world, int32_t rank, int64_t* row0, int64_t* rows);
int nnb_comm_unique_id(void* id_out /* NNB_UNIQUE_ID_BYTES */);
/* NCCL communicator on the calling thread's current CUDA device. */
int nnb_comm_init(const void* id, int32_t world, int32_t rank, nnb_comm_t* comm_out);
int nnb_comm_destroy(nnb_comm_t comm);
/* A_rows / X0_rows / X_rows_out: this rank's rows_g × n block (row-major).
 * X0 kinds: GIVEN, SCALED_IDENTITY, JACOBI, and TRANSPOSE_NORM (which
 * gathers A to form the transposed block).  Where the int8 emulation applies
 * (NNB_ARITH_FAST at n >= 3072, NNB_ARITH_OZAKI) the ranks exchange column
 * statistics and int8 residue blocks instead of FP64 rows, and X equals the
 * single-GPU chain's bit for bit; otherwise an FP64 ring feeds K-split DMMA
 * products.  Replaces the nn_invert loop (proj/src/solver.cpp:138-159) across GPUs. */
int nnb_nn_chain_sharded_d(nnb_comm_t comm, const double* A_rows, int64_t n,
                           const double* X0_rows, const nnb_chain_config* cfg, double* X_rows_out,
                           double* eps_hist, nnb_chain_result* result, void* stream);
/* The same schedule with `world` virtual ranks executed by this process on
 * this GPU (shared buffers replace the ring): validates the partition, the
 * K-split accumulation and the rank-ordered eps on one device. */
int nnb_nn_chain_sharded_emulated_d(const double* A, int64_t n, int32_t world, const double* X0,
                                    const nnb_chain_config* cfg, double* X_out, double* eps_hist,
                                    nnb_chain_result* result, void* stream);

/* ---- row-slab sharded sparse solve (one process per GPU) ---------------- */
/* rank g owns the rows nnb_partition_rows(n, world, g) of W,
 * B and x.  row_ptr: this rank's rows_g+1 offsets into col/val (col holds
 * GLOBAL column indices); B_rows / X_rows: rows_g × k.  Per application the
 * halo rows (the columns a slab references in its neighbours' slabs) move by
 * NCCL send/recv while the interior rows compute.  Bit-identical to
 * nnb_sparse_factorized_d for any world size.  The operator's bandwidth must
 * not exceed a neighbour slab (halos come from adjacent ranks only). */
int nnb_sparse_factorized_sharded_d(nnb_comm_t comm, const int64_t* row_ptr, const int32_t* col,
                                    const double* val, int64_t n, const double* B_rows, int64_t k,
                                    int64_t gamma, double theta, double* X_rows,
                                    int64_t* spmv_count_out, int32_t* fail_factor_out, void* stream);
/* Reusable form for repeated solves on one operator: the slab's staged CSR,
 * remapped columns, halo sizes and extended vectors are built once
 * (k right-hand-side columns fixed at creation). */
typedef struct nnb_sparse_plan* nnb_sparse_plan_t;
int nnb_sparse_plan_create(nnb_comm_t comm, const int64_t* row_ptr, const int32_t* col, const double* val,
                           int64_t n, int64_t k, nnb_sparse_plan_t* plan_out, void* stream);
int nnb_sparse_plan_solve(nnb_sparse_plan_t plan, const double* B_rows, int64_t gamma, double theta,
                          double* X_rows, int64_t* spmv_count_out, int32_t* fail_factor_out,
                          void* stream);
int nnb_sparse_plan_destroy(nnb_sparse_plan_t plan);
/* The same schedule with `world` virtual ranks (device copies move the halos). */
int nnb_sparse_factorized_sharded_emulated_d(const int64_t* row_ptr, const int32_t* col,
                                             const double* val, int64_t n, int64_t nnz,
                                             const double* B, int64_t k, int64_t gamma,
                                             double theta, int32_t world, double* X_out,
                                             int64_t* spmv_count_out, int32_t* fail_factor_out,
                                             void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NNB_H */
