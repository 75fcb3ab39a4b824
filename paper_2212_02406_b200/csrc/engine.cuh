// Internal engine API shared by the C-ABI translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "gemm_f64.cuh"

namespace nnb {

// ---- error plumbing (thread-local message, status codes of include/nnb.h) --
void set_error(const std::string& msg);
const char* last_error();

int cuda_fail(cudaError_t e, const char* what, const char* file, int line);
#define NNB_CUDA(x)                                                            \
  do {                                                                         \
    cudaError_t _e = (x);                                                      \
    if (_e != cudaSuccess) return ::nnb::cuda_fail(_e, #x, __FILE__, __LINE__); \
  } while (0)
#define NNB_TRY(x)              \
  do {                          \
    int _s = (x);               \
    if (_s != 0) return _s;     \
  } while (0)

int fail(int code, const std::string& msg);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-device setting:
// remember, per kernel and device, the largest size already set (thread-safe),
// so a second GPU driven from the same process gets its own call.
template <auto Kernel>
int ensure_smem(int bytes) {
  static std::atomic<int> done[64] = {};
  int dev = 0;
  NNB_CUDA(cudaGetDevice(&dev));
  std::atomic<int>& d = done[dev & 63];
  int cur = d.load(std::memory_order_acquire);
  if (cur >= bytes) return 0;
  NNB_CUDA(cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  while (cur < bytes && !d.compare_exchange_weak(cur, bytes, std::memory_order_acq_rel)) {
  }
  return 0;
}
void count_launch(uint64_t n = 1);
uint64_t launches();

// ---- device staging --------------------------------------------------------
bool is_device_ptr(const void* p);
int require_device();
cudaStream_t resolve(void* stream);

// Device buffer owned by one call (stream-ordered allocation).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  int alloc(size_t b, cudaStream_t st);
  void release();
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

// Either the caller's device pointer or a staged device copy of a host array.
struct In {
  const double* d = nullptr;
  DevBuf own;
  int stage(const double* src, size_t count, cudaStream_t s);
};
struct Out {
  double* d = nullptr;
  double* host = nullptr;
  size_t count = 0;
  DevBuf own;
  int prepare(double* dst, size_t count, cudaStream_t s);
  int finish(cudaStream_t s);  // copies back to host when staged
};

// ---- GEMM ------------------------------------------------------------------
// Reduction workspace: per-tile partials + the last-CTA counter.
struct RedWs {
  DevBuf buf;
  double* ss_partial = nullptr;
  int* nf_partial = nullptr;
  unsigned* counter = nullptr;
  int capacity = 0;
  int init(int max_tiles, cudaStream_t s);
};

struct GemmOp {
  const double* A = nullptr;
  int64_t lda = 0;
  const double* B = nullptr;
  int64_t ldb = 0;
  int64_t M = 0, N = 0, K = 0;
  GemmEpilogue ep;
  bool b_kmajor = false;  // B points at Bᵀ (N×K row-major, leading dimension ldb)
};

int max_tiles_for(int64_t M, int64_t N);
// 2D FP64 TMA descriptor over a row-major rows×cols matrix (leading dimension ld):
// box_rows×box_cols boxes, 128B swizzle or none, zero fill out of bounds.
int make_tmap(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld, int box_rows,
              int box_cols, bool swizzle128);
// Arithmetic mode (thread-local): 0 = fast DMMA path, 1 = reference-exact (exact.cu).
void set_arith(int mode);
int arith();
int gemm_exact(const GemmOp& op, cudaStream_t s);
// Ozaki-II emulation of a real product on the int8 tensor cores (ozaki.cu).
int gemm_ozaki(const GemmOp& op, cudaStream_t s);
int ozaki_moduli_for(int64_t k);
// moduli the whole product op needs (stats passes only), and a thread-local floor that
// a chunked product's pieces then use (0 = off)
int ozaki_plan_moduli(const GemmOp& op, cudaStream_t st, int* s_out);
void ozaki_force_moduli(int s);
void ozaki_profile(int on);
void ozaki_stats(double* ms, double* work, int64_t* launches, int reset);
// NNB_ARITH_FAST routes a real product to the int8 emulation where it beats DMMA
// (measured crossover between N=2048 and 4096): M, N >= 1024 and M·N·K >= 3072^3.
inline bool ozaki_pays(int64_t M, int64_t N, int64_t K) {
  return M >= 1024 && N >= 1024 && K >= 1024 && K <= 131071 && (double)M * N * K >= 3072.0 * 3072.0 * 3072.0;
}
// A chain operand that stays unchanged while pinned: its int8 splits are reused.
// returns false (and changes nothing) when p is already pinned
bool oz_pin(const double* p, int64_t ld, int64_t rows, int64_t cols);
void oz_unpin(const double* p);
// RAII pin for a scope in which p's contents do not change (no-op when off)
struct OzPinScope {
  const double* p = nullptr;
  OzPinScope(bool on, const double* ptr, int64_t ld, int64_t rows, int64_t cols) {
    if (on && oz_pin(ptr, ld, rows, cols)) p = ptr;
  }
  ~OzPinScope() {
    if (p) oz_unpin(p);
  }
};
// ---- int8 emulation of a row-sharded product (ozaki.cu; sharded.cu drives it) ----------
// C_g = epilogue(L_g·F) with F = [F_0; …; F_{G−1}] row-block sharded.  F's column exponents
// come from every rank's column statistics (gathered, combined in rank order), each rank
// splits its own block into K-major residues, the residue blocks are all-gathered, and the
// G block products accumulate mod m_l (oz_gemm_block, `accumulate`) before one
// reconstruction — every element then equals the single-GPU emulated product's.
// ratio slots (float bits, as the single-GPU path): [L1 left, L1 right, L2 left, L2 right].
int oz_col_partials(const double* F, int64_t ld, int64_t rows, int64_t n, double* out /*[3][n]*/, cudaStream_t s);
int oz_col_combine(const double* gathered /*[world][stride]*/, int world, int64_t stride, int64_t n, int* exps,
                   unsigned* ratio /*right slots: ratio + 1*/, cudaStream_t s);
int oz_row_stats(const double* L, int64_t ld, int64_t rows, int64_t k, int* exps, unsigned* ratio, cudaStream_t s);
int oz_read_ratios(const unsigned* ratio_dev, double out[4], cudaStream_t s);  // synchronises s
int oz_moduli(double a1, double a2, double b1, double b2, int64_t K);
int oz_split_left(const double* L, int64_t ld, int64_t rows, int64_t k, const int* exps, int s, int8_t* out,
                  int64_t kp, cudaStream_t st);
int oz_split_right(const double* F, int64_t ld, int64_t k_rows, int64_t n, const int* exps, int s, int8_t* out,
                   int64_t kp, cudaStream_t st);
// s int8 GEMMs over nblk K blocks in one launch: block b multiplies the left residues' columns
// from a_k0[b] by the right residue array's rows from b_row0[b] (b_kp bytes each, zero-padded);
// `accumulate` adds to the residues in `out` (mod m); persistent grid of SMs − reserve_sms CTAs
int oz_gemm_blocks(const int8_t* a_res, int64_t M, int64_t a_kp, const int64_t* a_k0, const int8_t* b_res, int64_t N,
                   int64_t b_rows, int64_t b_kp, const int64_t* b_row0, int nblk, int s, uint8_t* out, int64_t ldr,
                   bool accumulate, cudaStream_t st, int reserve_sms = 0);
int oz_reconstruct(int s, const uint8_t* res, int64_t ldr, int64_t M, int64_t N, const int* ea, const int* eb,
                   GemmEpilogue ep, struct RedWs* red, cudaStream_t st);
// the next real chain of the calling thread copies its final residual I − A·X to r (device, ld)
void set_chain_capture(double* r, int64_t ld);
// 2D uint8 TMA descriptor (rows × cols bytes, leading dimension ld bytes), 128B swizzle.
int make_tmap_u8(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                 int box_cols);
// Launches C = epilogue(A·B).  If `red` is non-null the Σ C² / non-finite
// reduction is wired to it (ep.ss_out / nf_out / eps_out chosen by caller).
int gemm(GemmOp op, RedWs* red, cudaStream_t s);

// Complex product on planar operands, 3M on the DMMA GEMM (engine.cu).
struct ZGemm {
  int64_t M = 0, N = 0, K = 0;
  const double *Ar = nullptr, *Ai = nullptr;
  int64_t lda = 0;
  const double *Br = nullptr, *Bi = nullptr;
  int64_t ldb = 0;
  double alpha = 1.0, beta = 0.0, gamma = 0.0;
  const double *Dr = nullptr, *Di = nullptr;  // may alias Cr / Ci
  int64_t ldd = 0;
  int64_t diag_offset = 0;
  double *Cr = nullptr, *Ci = nullptr;
  int64_t ldc = 0;
  double* ss_out = nullptr;   // Σ |C|² (with nf_out and a reduction workspace)
  int* nf_out = nullptr;
  double* eps_out = nullptr;  // sqrt(Σ|C|²)·eps_scale
  double eps_scale = 1.0;
};
int zgemm3m(const ZGemm& z, RedWs* red, cudaStream_t s);

// ---- auxiliary kernels ----------------------------------------------------------
int axpby(double alpha, const double* A, int64_t lda, double beta, const double* B, int64_t ldb,
          double gamma, int64_t diag_offset, double* out, int64_t ldo, int64_t rows, int64_t cols,
          cudaStream_t s);
int copy2d(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int64_t cols,
           cudaStream_t s);
int x0_build(const double* A, int64_t lda, int64_t n, int kind, double scale, double* X0,
             int64_t ldx, cudaStream_t s);
// deterministic Σ v² over `count` doubles (stride 1) into *out_dev
int sumsq(const double* v, int64_t count, double* out_dev, cudaStream_t s);
int trace_dev(const double* M, int64_t n, int64_t ld, int complex_stride, double* out_dev,
              cudaStream_t s);
int deinterleave(const double* z, int64_t count, double* re, double* im, cudaStream_t s);
int interleave(const double* re, const double* im, int64_t count, double* z, cudaStream_t s);
int fill_identity(double* X, int64_t n, int64_t ld, double val, cudaStream_t s);
// generators.cu: Householder Q (device in/out, cplx: interleaved), random_spd / random_conditioned_complex
int householder_q(const double* A, int64_t n, int cplx, double* Q, cudaStream_t s);
int random_spd_dev(const double* G, const double* lam, int64_t n, double* W, cudaStream_t s);
// Gauss–Jordan inverse (direct_inverse_oracle); *singular_col = first singular pivot column or −1
int direct_inverse(const double* M, int64_t n, int cplx, double pivot_floor, double* inv, int* singular_col,
                   cudaStream_t s);
int random_conditioned_dev(const double* GU, const double* GV, const double* sigma, int64_t n, double* A,
                           cudaStream_t s);
// out (cols×rows) = Mᵀ (cplx = 0) or Mᴴ of interleaved complex M (cplx = 1)
int transpose(const double* M, int64_t rows, int64_t cols, int cplx, double* out, cudaStream_t s);

// ---- dense chain -----------------------------------------------------------------
struct ChainCfg {
  int p = 1;
  int max_iters = 1;
  double tol = 0.0;
  int order = 0;
  int final_residual = 1;
};
struct ChainOut {
  int iters = 0;
  int fail_iter = 0;
  int stopped = 1;
  int products = 0;
  double last_eps = 0.0;
  float device_ms = 0.f;
  int x_index = 0;  // sharded driver: which ping-pong buffer holds the final X
};
// Host-streaming hooks of the real chain (nnb_nn_chain_d with host buffers):
// the first residual product runs split along K as A's column blocks and
// X0's row blocks land (NORTHSTAR order, R = I − A·X0; bit-identical to one
// launch through the accumulator seed), and the last
// Horner product runs in row chunks whose rows go device→host on `copy` as
// soon as they are written.  PCIe then overlaps the DMMA work instead of
// bracketing it.
struct ChainIo {
  int chunks = 0;
  int64_t chunk_rows = 0;
  cudaEvent_t* a_ready = nullptr;  // [chunks] A's columns and X0's rows of chunk q are on the device; null: all present
  double* host_out = nullptr;      // row-major n×n host destination of the final X (nullable)
  cudaStream_t copy = nullptr;
  cudaEvent_t* out_done = nullptr; // [chunks] scratch
  cudaEvent_t copy_done = nullptr; // scratch
  bool out_streamed = false;       // run_chain delivered the final X to host_out (X itself is then stale)
  // int8-emulation streaming: A arrives by row chunks and X0 by column chunks, and the first
  // product R = I − A·X0 runs by blocks as their chunks land (chain.cu product_2d)
  cudaEvent_t* a_rows_ready = nullptr;  // [chunks] A's row chunk i landed
  cudaEvent_t* x_cols_ready = nullptr;  // [chunks] X0's column chunk j landed
};
// Real chain on device buffers with ld == ldn (ldn even, >= n).  X holds X0
// on entry and the final iterate on exit.  eps_hist host (nullable).
int chain_real(const double* A, int64_t n, int64_t ldn, double* X, const ChainCfg& cfg,
               double* eps_hist, ChainOut* out, cudaStream_t s, ChainIo* io = nullptr);
// Small real chains (n <= small_chain_max_n(), NNB_SMALL_CHAIN_MAX, 0 = off): the
// nn_invert loop as one cooperative kernel (chain_small.cu).  X holds X0 on entry
// and the final iterate on exit; R, w1, w2 are n×ld scratch; eps_dev / nf_dev
// are filled as run_chain fills them; status_dev = {k, products, stopped, recorded}
// (device ints, read by the caller after its own synchronisation).
int small_chain_max_n();
bool small_chain_eligible(int64_t n, int64_t ld, const ChainCfg& cfg);
int small_chain_real(const double* A, double* X, double* R, double* w1, double* w2, int64_t n, int64_t ld,
                     const ChainCfg& cfg, double* eps_dev, int* nf_dev, int* status_dev, cudaStream_t s);
// Page-locked host block of at least `bytes` (per thread, grown on demand; null on failure).
void* pinned_stage(size_t bytes);
// Complex chain on planar device buffers (re/im each n×ldn).
int chain_complex(const double* Ar, const double* Ai, int64_t n, int64_t ldn, double* Xr,
                  double* Xi, const ChainCfg& cfg, double* eps_hist, ChainOut* out,
                  cudaStream_t s);

// ns_sum on device planes (im pointers null for real); identity_start as the
// reference decides it (phi0 exactly I).
int ns_sum_dev(const double* phi0_re, const double* phi0_im, const double* w_re,
               const double* w_im, int64_t n, int64_t ldn, int64_t order, bool identity_start,
               double* out_re, double* out_im, double* products, cudaStream_t s);
int ns_factorized_dev(const double* phi_re, const double* phi_im, const double* w_re, const double* w_im,
                      int64_t n, int64_t ldn, int s_factors, bool identity_start, double* out_re, double* out_im,
                      double* products, cudaStream_t s);
int power_ladder_dev(const double* p_re, const double* p_im, int64_t n, int64_t ldn, uint64_t e, double* out_re,
                     double* out_im, double* products, cudaStream_t s);
int nn_explicit_dev(const double* phi_re, const double* phi_im, const double* w_re, const double* w_im, int64_t n,
                    int64_t ldn, int nests_i, int depth_L, bool identity_start, double* out_re, double* out_im,
                    double* products, cudaStream_t s);
int is_identity_dev(const double* re, const double* im, int64_t n, int64_t ld, bool* result,
                    cudaStream_t s);
// A == Aᵀ exactly (synchronises s)
int is_symmetric_dev(const double* A, int64_t n, int64_t ld, bool* result, cudaStream_t s);
int deinterleave2d(const double* z, int64_t rows, int64_t cols, double* re, double* im,
                   int64_t ldp, cudaStream_t s);
int interleave2d(const double* re, const double* im, int64_t rows, int64_t cols, int64_t ldp,
                 double* z, cudaStream_t s);
int axpby_z(double ar, double ai, const double* A, double br, double bi, const double* B,
            double gr, double gi, double* out, int64_t rows, int64_t cols, cudaStream_t s);

// ---- batched / sparse (separate translation units) -------------------------------
int batched_nn_z16(const double* A, int64_t batch, int p, int iters, int ns_order, double* X,
                   double* eps_last, cudaStream_t s);
// n = 8, 24, 32 (batched_generic.cu): one warp per system, iterates in shared memory
int batched_nn_gen(const double* A, int64_t batch, int n, int p, int iters, int ns_order, double* X, double* eps,
                   cudaStream_t s);
int mimo_detect_gen(const double* H, const double* y, int64_t batch, int antennas, int users, double sigma2, int p,
                    int iters, double* xhat, double* X, double* eps, cudaStream_t s);
int mimo_detect_z16(const double* H, const double* y, int64_t batch, int antennas, double sigma2, int p,
                    int iters, double* xhat, double* X, double* eps_last, cudaStream_t s);
int spmv_csr(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n,
             const double* X, int64_t k, double* Y, cudaStream_t s);
int sparse_factorized(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n,
                      const double* B, int64_t k, int s_factors, double theta, double* X,
                      int* fail_factor, cudaStream_t s);

}  // namespace nnb
