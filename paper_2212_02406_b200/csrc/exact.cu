// Reference-exact arithmetic mode (nnb_set_arithmetic(NNB_ARITH_REFERENCE)).
//
// The fast path runs products on DMMA (k-blocked, fused multiply-adds) and
// reduces ‖R‖² per tile, so it agrees with the reference to ~1e-15 relative
// but not bit for bit.  This mode reproduces the reference's rounding
// exactly for real data, so the GPU can be checked bit-for-bit against it:
//   * gemm_exact_kernel: C[i][j] = Σ_k a_ik·b_kj in ascending k, one rounded
//     multiply and one rounded add per term starting from 0.0 — the
//     reference's `sum += a(i,k)*b(k,j)` (proj/src/kernels.cpp:143-150) for
//     zero imaginary parts; the epilogue's "I −" / "+ I" are the reference's
//     identity_minus / plus_identity roundings (kernels.cpp:203-221);
//   * serial_sumsq_kernel: ‖C‖² summed serially in row-major order and
//     eps = sqrt(s) / sqrt(N) — frobenius_norm / residual_epsilon
//     (kernels.cpp:238-242, solver.cpp:72-75);
//   * the chain driver switches to the reference's own nest sequence
//     P = I − X·W, S = I + P, S = I + P·S (L−1×), X' = S·X (solver.cpp:93-103).
// CUDA-core FP64 (no tensor cores): a verification mode, not the fast path.
#include <cstdlib>

#include "engine.cuh"

namespace nnb {

// 0 fast (per product: int8 emulation where it pays, else DMMA), 1 reference-exact,
// 2 Ozaki int8 emulation for every real product (ozaki.cu), 3 DMMA only.
// NNB_ARITHMETIC=reference|ozaki|dmma selects the mode for every thread (e.g. for the C++ drop-in without code changes).
static int initial_arith() {
  const char* e = std::getenv("NNB_ARITHMETIC");
  return (e && e[0] == 'r') ? 1 : (e && e[0] == 'o') ? 2 : (e && e[0] == 'd') ? 3 : 0;
}
static thread_local int g_arith = initial_arith();
void set_arith(int mode) { g_arith = mode; }
int arith() { return g_arith; }

namespace {

constexpr int kT = 64, kKc = 16;

__global__ void __launch_bounds__(256) gemm_exact_kernel(const double* __restrict__ A, int64_t lda,
                                                         const double* __restrict__ B, int64_t ldb, int M, int N,
                                                         int K, GemmEpilogue ep) {
  __shared__ double As[kT][kKc + 1];
  __shared__ double Bs[kKc][kT + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * kT, n0 = blockIdx.x * kT;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int k0 = 0; k0 < K; k0 += kKc) {
    const int kc = min(kKc, K - k0);
    for (int e = threadIdx.x; e < kT * kKc; e += 256) {
      const int r = e / kKc, k = e % kKc;
      As[r][k] = (m0 + r < M && k < kc) ? A[(int64_t)(m0 + r) * lda + k0 + k] : 0.0;
    }
    for (int e = threadIdx.x; e < kKc * kT; e += 256) {
      const int k = e / kT, c = e % kT;
      Bs[k][c] = (n0 + c < N && k < kc) ? B[(int64_t)(k0 + k) * ldb + n0 + c] : 0.0;
    }
    __syncthreads();
    for (int k = 0; k < kc; ++k) {  // ascending k, no contraction
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double a = As[ty * 4 + i][k];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a, Bs[k][tx * 4 + j]));
      }
    }
    __syncthreads();
  }
  int nf = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + ty * 4 + i;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = n0 + tx * 4 + j;
      if (c >= N) continue;
      double v = ep.alpha == 1.0 ? acc[i][j] : (ep.alpha == -1.0 ? -acc[i][j] : __dmul_rn(ep.alpha, acc[i][j]));
      if (ep.D) v = __dadd_rn(v, ep.beta == 1.0 ? ep.D[(int64_t)r * ep.ldd + c] : __dmul_rn(ep.beta, ep.D[(int64_t)r * ep.ldd + c]));
      if ((int64_t)r + ep.diag_offset == c) v = __dadd_rn(ep.gamma, v);
      ep.C[(int64_t)r * ep.ldc + c] = v;
      nf += !isfinite(v);
    }
  }
  if (ep.nf_out && nf) atomicAdd(ep.nf_out, nf);  // integer: order-free
}

__global__ void serial_sumsq_kernel(const double* __restrict__ C, int64_t ldc, int M, int N, double* ss_out,
                                    double* eps_out, double n_div) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0;
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < N; ++c) {
      const double v = C[(int64_t)r * ldc + c];
      s = __dadd_rn(s, __dmul_rn(v, v));  // std::norm = re*re + 0*0, then s += it
    }
  if (ss_out) *ss_out = s;
  if (eps_out) *eps_out = __ddiv_rn(__dsqrt_rn(s), __dsqrt_rn(n_div));
}

}  // namespace

int gemm_exact(const GemmOp& op, cudaStream_t s) {
  if (op.b_kmajor) return fail(7, "exact mode: K-major B operand is not supported");
  if (op.ep.nf_out) NNB_CUDA(cudaMemsetAsync(op.ep.nf_out, 0, sizeof(int), s));
  dim3 grid(static_cast<unsigned>((op.N + kT - 1) / kT), static_cast<unsigned>((op.M + kT - 1) / kT));
  gemm_exact_kernel<<<grid, 256, 0, s>>>(op.A, op.lda, op.B, op.ldb, static_cast<int>(op.M), static_cast<int>(op.N),
                                         static_cast<int>(op.K), op.ep);
  count_launch();
  if (op.ep.ss_out || op.ep.eps_out) {
    const double n_div = op.ep.eps_scale > 0.0 ? 1.0 / (op.ep.eps_scale * op.ep.eps_scale) : 1.0;
    serial_sumsq_kernel<<<1, 32, 0, s>>>(op.ep.C, op.ep.ldc, static_cast<int>(op.M), static_cast<int>(op.N),
                                         op.ep.ss_out, op.ep.eps_out, std::nearbyint(n_div));
    count_launch();
  }
  NNB_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace nnb
