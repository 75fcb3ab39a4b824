// Batched Nested Neumann for the other massive-MIMO system sizes: n = 8, 24 and 32
// users (BASELINE config 1 is 16 users and runs the specialised batched_z16_kernel).
// The reference's nn_step / ns_sum / residual_epsilon take any n
// (proj/src/solver.cpp:77-103); this kernel keeps the 16-user kernel's contract —
// Jacobi X0 = diag(A)^-1 (Smith's complex reciprocal, as libgcc's __divdc3), `iters`
// nests of depth p in the reference operand order (P = I − X·A, X' = X + P·(X + P·…)),
// eps = ‖I − X·A‖_F/√n after the last nest; or the NS series of a given order —
// with one warp per system and the iterates in shared memory.
//
// Products are complex 4M on DMMA.8x8x4: for each 8×8 output tile, n/4 k-steps of
// four DMMAs (re·re, −im·im, re·im, im·re) into two register accumulators.  Operands
// live planar in per-warp shared memory with a row stride of n + 2 doubles, which
// keeps the m8n8k4 fragment loads at their 2-wavefront minimum.
// The fused detector (Gram Hᴴ·H + σ²I and z = Hᴴ·y from one pass over H, the NN
// inverse, x̂ = X·z) has the same shape for n users.
#include <algorithm>
#include <cmath>
#include <cstdint>

#include "common.cuh"
#include "engine.cuh"

namespace nnb {
namespace {

template <int N>
struct Gen {
  static constexpr int kLd = N + 2;            // planar row stride (doubles)
  static constexpr int kMat = N * kLd;         // one plane
  static constexpr int kT = N / 8;             // 8×8 tiles per dimension
  static constexpr int kMats = 4;              // A, X, P, V
  static constexpr int kBytesPerWarp = kMats * 2 * kMat * 8;
};

struct Pl {
  double* re;
  double* im;
};

// C(8×8 tile ti,tj) of L·R, 4M: acc_re = Σ lr·rr − li·ri, acc_im = Σ lr·ri + li·rr
template <int N>
__device__ __forceinline__ void tile_mma(const Pl& L, const Pl& R, int ti, int tj, int g, int t, double (&cr)[2],
                                         double (&ci)[2]) {
  constexpr int ld = Gen<N>::kLd;
  cr[0] = cr[1] = ci[0] = ci[1] = 0.0;
#pragma unroll
  for (int kb = 0; kb < N / 4; ++kb) {
    const int ar = 8 * ti + g, ac = 4 * kb + t;   // A fragment: L[ar][ac]
    const int br = 4 * kb + t, bc = 8 * tj + g;   // B fragment: R[br][bc]
    const double lr = L.re[ar * ld + ac], li = L.im[ar * ld + ac];
    const double rr = R.re[br * ld + bc], ri = R.im[br * ld + bc];
    dmma_8x8x4(cr[0], cr[1], lr, rr);
    dmma_8x8x4(cr[0], cr[1], -li, ri);
    dmma_8x8x4(ci[0], ci[1], lr, ri);
    dmma_8x8x4(ci[0], ci[1], li, rr);
  }
}

// 3M (Gauss) for one 8×8 tile: P1 = Σ lr·rr, P2 = Σ li·ri, P3 = Σ (lr+li)(rr+ri);
// re = P1 − P2, im = P3 − P1 − P2 — 3 DMMA and 2 pre-sum DADDs per k-step instead of 4 DMMA
template <int N>
__device__ __forceinline__ void tile_mma3(const Pl& L, const Pl& R, int ti, int tj, int g, int t, double (&cr)[2],
                                          double (&ci)[2]) {
  constexpr int ld = Gen<N>::kLd;
  double p1[2] = {0.0, 0.0}, p2[2] = {0.0, 0.0}, p3[2] = {0.0, 0.0};
#pragma unroll
  for (int kb = 0; kb < N / 4; ++kb) {
    const int ar = 8 * ti + g, ac = 4 * kb + t;
    const int br = 4 * kb + t, bc = 8 * tj + g;
    const double lr = L.re[ar * ld + ac], li = L.im[ar * ld + ac];
    const double rr = R.re[br * ld + bc], ri = R.im[br * ld + bc];
    dmma_8x8x4(p1[0], p1[1], lr, rr);
    dmma_8x8x4(p2[0], p2[1], li, ri);
    dmma_8x8x4(p3[0], p3[1], lr + li, rr + ri);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    cr[h] = p1[h] - p2[h];
    ci[h] = p3[h] - p1[h] - p2[h];
  }
}

// out = alpha·(L·R) + beta·D + gamma·I over all tiles (out may alias any operand: every
// tile is formed in registers before the first store);
// returns this lane's Σ |out|² when want_ss
template <int N>
__device__ double product(const Pl& L, const Pl& R, double alpha, const Pl* D, double beta, double gamma, const Pl& out,
                          int g, int t, bool want_ss) {
  constexpr int ld = Gen<N>::kLd;
  double ss = 0.0;
  double keep_r[Gen<N>::kT * Gen<N>::kT][2], keep_i[Gen<N>::kT * Gen<N>::kT][2];
#pragma unroll
  for (int ti = 0; ti < Gen<N>::kT; ++ti)
#pragma unroll
    for (int tj = 0; tj < Gen<N>::kT; ++tj) {
      double cr[2], ci[2];
      tile_mma3<N>(L, R, ti, tj, g, t, cr, ci);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 8 * ti + g, c = 8 * tj + 2 * t + h;
        double vr = alpha * cr[h], vi = alpha * ci[h];
        if (D) {
          vr = fma(beta, D->re[r * ld + c], vr);
          vi = fma(beta, D->im[r * ld + c], vi);
        }
        if (r == c) vr += gamma;
        keep_r[ti * Gen<N>::kT + tj][h] = vr;
        keep_i[ti * Gen<N>::kT + tj][h] = vi;
        if (want_ss) ss += vr * vr + vi * vi;
      }
    }
  __syncwarp();  // every lane has read L, R and D before `out` is overwritten
#pragma unroll
  for (int ti = 0; ti < Gen<N>::kT; ++ti)
#pragma unroll
    for (int tj = 0; tj < Gen<N>::kT; ++tj)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 8 * ti + g, c = 8 * tj + 2 * t + h;
        out.re[r * ld + c] = keep_r[ti * Gen<N>::kT + tj][h];
        out.im[r * ld + c] = keep_i[ti * Gen<N>::kT + tj][h];
      }
  __syncwarp();
  return ss;
}

// X0 = diag(A)^-1, Smith's reciprocal (libgcc's __divdc3 for 1/(c + di))
template <int N>
__device__ void jacobi_x0(const Pl& A, const Pl& X, int lane) {
  constexpr int ld = Gen<N>::kLd;
  for (int i = lane; i < N * ld; i += 32) {
    X.re[i] = 0.0;
    X.im[i] = 0.0;
  }
  __syncwarp();
  if (lane < N) {
    const double c = A.re[lane * ld + lane], d = A.im[lane * ld + lane];
    double xr, xi;
    if (fabs(c) >= fabs(d)) {
      const double r = d / c, den = c + d * r;
      xr = (1.0 + 0.0 * r) / den;
      xi = (0.0 - 1.0 * r) / den;
    } else {
      const double r = c / d, den = c * r + d;
      xr = (1.0 * r + 0.0) / den;
      xi = (0.0 * r - 1.0) / den;
    }
    X.re[lane * ld + lane] = xr;
    X.im[lane * ld + lane] = xi;
  }
  __syncwarp();
}

// NN (ns_order < 0) or NS of order ns_order on the system in A; X written to X.
template <int N>
__device__ double solve(const Pl& A, const Pl& X, const Pl& P, const Pl& V, int p, int iters, int ns_order, int g,
                        int t, int lane, bool want_eps) {
  constexpr int ld = Gen<N>::kLd;
  jacobi_x0<N>(A, X, lane);
  if (ns_order < 0) {
    for (int it = 0; it < iters; ++it) {
      product<N>(X, A, -1.0, nullptr, 0.0, 1.0, P, g, t, false);  // P = I − X·A
      // Horner V = X + P·V (V starts at X); product() forms the whole tile set in
      // registers before it stores, so the output may alias an operand
      const Pl* v = &X;
      for (int j = 1; j <= p; ++j) {
        product<N>(P, *v, 1.0, &X, 1.0, 0.0, V, g, t, false);
        v = &V;
      }
      for (int i = lane; i < N * ld; i += 32) {
        X.re[i] = V.re[i];
        X.im[i] = V.im[i];
      }
      __syncwarp();
    }
    if (!want_eps) return 0.0;
    const double ss = warp_sum(product<N>(X, A, -1.0, nullptr, 0.0, 1.0, P, g, t, true));
    return sqrt(ss) / sqrt(static_cast<double>(N));
  }
  // NS: P = I − X0·A, T = I + P, T = T·P + I (order−1 times), X = T·X0
  if (ns_order == 0) return 0.0;  // X = X0
  product<N>(X, A, -1.0, nullptr, 0.0, 1.0, P, g, t, false);
  for (int i = lane; i < N * ld; i += 32) {
    V.re[i] = P.re[i];
    V.im[i] = P.im[i];
  }
  __syncwarp();
  if (lane < N) V.re[lane * ld + lane] += 1.0;
  __syncwarp();
  for (int step = 2; step <= ns_order; ++step) product<N>(V, P, 1.0, nullptr, 0.0, 1.0, V, g, t, false);
  // X = T·X0 into P (X is an operand), then back
  product<N>(V, X, 1.0, nullptr, 0.0, 0.0, P, g, t, false);
  for (int i = lane; i < N * ld; i += 32) {
    X.re[i] = P.re[i];
    X.im[i] = P.im[i];
  }
  __syncwarp();
  return 0.0;
}

template <int N>
__device__ __forceinline__ void warp_planes(double* smem_warp, Pl& A, Pl& X, Pl& P, Pl& V) {
  constexpr int m = Gen<N>::kMat;
  A = {smem_warp + 0 * m, smem_warp + 1 * m};
  X = {smem_warp + 2 * m, smem_warp + 3 * m};
  P = {smem_warp + 4 * m, smem_warp + 5 * m};
  V = {smem_warp + 6 * m, smem_warp + 7 * m};
}

template <int N>
__device__ void store_x(const Pl& X, double2* Xs, int lane) {
  constexpr int ld = Gen<N>::kLd;
  for (int e = lane; e < N * N; e += 32) Xs[e] = make_double2(X.re[(e / N) * ld + e % N], X.im[(e / N) * ld + e % N]);
  __syncwarp();
}

template <int N>
__global__ void __launch_bounds__(128) batched_gen_kernel(const double2* __restrict__ A, int64_t batch, int p,
                                                          int iters, int ns_order, double2* __restrict__ Xout,
                                                          double* __restrict__ eps_last) {
  extern __shared__ __align__(16) double gsm[];
  constexpr int ld = Gen<N>::kLd;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  Pl Am, X, P, V;
  warp_planes<N>(gsm + (size_t)warp * Gen<N>::kMats * 2 * Gen<N>::kMat, Am, X, P, V);
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t s = blockIdx.x * wpb + warp; s < batch; s += (int64_t)gridDim.x * wpb) {
    const double2* As = A + s * N * N;
    for (int e = lane; e < N * N; e += 32) {
      const double2 v = __ldg(As + e);
      Am.re[(e / N) * ld + e % N] = v.x;
      Am.im[(e / N) * ld + e % N] = v.y;
    }
    __syncwarp();
    const double eps = solve<N>(Am, X, P, V, p, iters, ns_order, g, t, lane, eps_last != nullptr);
    if (eps_last && lane == 0 && ns_order < 0) eps_last[s] = eps;
    store_x<N>(X, Xout + s * N * N, lane);
  }
}

// Fused detector for N users: A = Hᴴ·H + σ²I, z = Hᴴ·y, NN inverse, x̂ = X·z
template <int N>
__global__ void __launch_bounds__(128) detect_gen_kernel(const double2* __restrict__ H, const double2* __restrict__ Y,
                                                         int64_t batch, int ant, double sigma2, int p, int iters,
                                                         double2* __restrict__ xhat, double2* __restrict__ Xout,
                                                         double* __restrict__ eps_last) {
  extern __shared__ __align__(16) double gsm[];
  constexpr int ld = Gen<N>::kLd;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  Pl Am, X, P, V;
  warp_planes<N>(gsm + (size_t)warp * Gen<N>::kMats * 2 * Gen<N>::kMat, Am, X, P, V);
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t s = blockIdx.x * wpb + warp; s < batch; s += (int64_t)gridDim.x * wpb) {
    const double2* Hs = H + s * (int64_t)ant * N;
    const double2* Ys = Y + s * (int64_t)ant;
    // Gram by DMMA over the antennas: A-operand conj(H)[i][a], B-operand H[a][j]
#pragma unroll
    for (int ti = 0; ti < Gen<N>::kT; ++ti)
#pragma unroll
      for (int tj = 0; tj < Gen<N>::kT; ++tj) {
        double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
        for (int kb = 0; kb < ant / 4; ++kb) {
          const int a = 4 * kb + t;
          const double2 hl = __ldg(Hs + (int64_t)a * N + 8 * ti + g);  // conj → (x, −y)
          const double2 hr = __ldg(Hs + (int64_t)a * N + 8 * tj + g);
          dmma_8x8x4(cr[0], cr[1], hl.x, hr.x);
          dmma_8x8x4(cr[0], cr[1], hl.y, hr.y);   // −(−y)·y
          dmma_8x8x4(ci[0], ci[1], hl.x, hr.y);
          dmma_8x8x4(ci[0], ci[1], -hl.y, hr.x);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = 8 * ti + g, c = 8 * tj + 2 * t + h;
          Am.re[r * ld + c] = cr[h] + (r == c ? sigma2 : 0.0);
          Am.im[r * ld + c] = ci[h];
        }
      }
    __syncwarp();
    // z = Hᴴ·y (lane i < N: row i), kept in V's first column
    if (lane < N) {
      double zr = 0.0, zi = 0.0;
      for (int a = 0; a < ant; ++a) {
        const double2 h = __ldg(Hs + (int64_t)a * N + lane), y = __ldg(Ys + a);
        zr = fma(h.x, y.x, fma(h.y, y.y, zr));
        zi = fma(h.x, y.y, fma(-h.y, y.x, zi));
      }
      V.re[lane * ld + N] = zr;  // spare padding column (ld = N + 2)
      V.im[lane * ld + N] = zi;
    }
    __syncwarp();
    double zr_l = 0.0, zi_l = 0.0;
    if (lane < N) {
      zr_l = V.re[lane * ld + N];
      zi_l = V.im[lane * ld + N];
    }
    const double eps = solve<N>(Am, X, P, V, p, iters, -1, g, t, lane, eps_last != nullptr);
    if (eps_last && lane == 0) eps_last[s] = eps;
    // x̂ = X·z: lane i < N computes row i
    double xr = 0.0, xi = 0.0;
    for (int j = 0; j < N; ++j) {
      const double zjr = __shfl_sync(0xffffffffu, zr_l, j), zji = __shfl_sync(0xffffffffu, zi_l, j);
      if (lane < N) {
        const double a = X.re[lane * ld + j], b = X.im[lane * ld + j];
        xr = fma(a, zjr, fma(-b, zji, xr));
        xi = fma(a, zji, fma(b, zjr, xi));
      }
    }
    if (lane < N) xhat[s * N + lane] = make_double2(xr, xi);
    if (Xout) store_x<N>(X, Xout + s * N * N, lane);
    __syncwarp();
  }
}

// ---- n = 24, 32: one block of n/8 warps per system ---------------------------------
// With one warp per system a 32-user system's four planar 32×34 matrix pairs (70 KB) left 3
// warps per SM, and the warp's 16 output tiles did not fit its registers.  Here warp w owns
// the 8-row stripe w of every product (n/8 tiles, formed in registers), the system's warps
// meet at a block barrier before the stripe is stored (the output may alias an operand)
// and after; 3 (n=32) or 5 (n=24) systems per SM, 12-15 warps.  Products are 3M (Gauss):
// 25 % fewer DMMAs than the one-warp kernel's 4M, within the parity tolerance.
template <int N>
__device__ double product_coop(const Pl& L, const Pl& R, double alpha, const Pl* D, double beta, double gamma,
                               const Pl& out, int w, int g, int t, bool want_ss) {
  constexpr int ld = Gen<N>::kLd, kT = Gen<N>::kT;
  double ss = 0.0;
  double keep_r[kT][2], keep_i[kT][2];
#pragma unroll
  for (int tj = 0; tj < kT; ++tj) {
    double cr[2], ci[2];
    tile_mma3<N>(L, R, w, tj, g, t, cr, ci);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = 8 * w + g, c = 8 * tj + 2 * t + h;
      double vr = alpha * cr[h], vi = alpha * ci[h];
      if (D) {
        vr = fma(beta, D->re[r * ld + c], vr);
        vi = fma(beta, D->im[r * ld + c], vi);
      }
      if (r == c) vr += gamma;
      keep_r[tj][h] = vr;
      keep_i[tj][h] = vi;
      if (want_ss) ss += vr * vr + vi * vi;
    }
  }
  __syncthreads();  // every warp has read L, R and D before `out` is overwritten
#pragma unroll
  for (int tj = 0; tj < kT; ++tj)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = 8 * w + g, c = 8 * tj + 2 * t + h;
      out.re[r * ld + c] = keep_r[tj][h];
      out.im[r * ld + c] = keep_i[tj][h];
    }
  __syncthreads();
  return ss;
}

// Jacobi X0 and the NN (ns_order < 0) or NS (ns_order > 0) iteration on the system in Am,
// by the block's n/8 warps; returns eps = ‖I − X·A‖_F/√n after the last nest (NN, want_eps)
template <int N>
__device__ double solve_coop(const Pl& Am, const Pl& X, const Pl& P, const Pl& V, int p, int iters, int ns_order,
                             int w, int g, int t, bool want_eps, double* red) {
  constexpr int ld = Gen<N>::kLd, kW = N / 8, kThreadsC = 32 * kW;
  const int lane = threadIdx.x & 31;
  // X0 = diag(A)^-1 (Smith's reciprocal, as jacobi_x0)
  for (int i = threadIdx.x; i < N * ld; i += kThreadsC) {
    X.re[i] = 0.0;
    X.im[i] = 0.0;
  }
  __syncthreads();
  if (threadIdx.x < N) {
    const int r = threadIdx.x;
    const double c = Am.re[r * ld + r], d = Am.im[r * ld + r];
    double xr, xi;
    if (fabs(c) >= fabs(d)) {
      const double q = d / c, den = c + d * q;
      xr = (1.0 + 0.0 * q) / den;
      xi = (0.0 - 1.0 * q) / den;
    } else {
      const double q = c / d, den = c * q + d;
      xr = (1.0 * q + 0.0) / den;
      xi = (0.0 * q - 1.0) / den;
    }
    X.re[r * ld + r] = xr;
    X.im[r * ld + r] = xi;
  }
  __syncthreads();
  double eps = 0.0;
  if (ns_order < 0) {
    for (int it = 0; it < iters; ++it) {
      product_coop<N>(X, Am, -1.0, nullptr, 0.0, 1.0, P, w, g, t, false);  // P = I − X·A
      const Pl* v = &X;
      for (int j = 1; j <= p; ++j) {  // V = X + P·V, V starting at X
        product_coop<N>(P, *v, 1.0, &X, 1.0, 0.0, V, w, g, t, false);
        v = &V;
      }
      for (int i = threadIdx.x; i < N * ld; i += kThreadsC) {
        X.re[i] = V.re[i];
        X.im[i] = V.im[i];
      }
      __syncthreads();
    }
    if (want_eps) {
      const double ss = warp_sum(product_coop<N>(X, Am, -1.0, nullptr, 0.0, 1.0, P, w, g, t, true));
      if (lane == 0) red[w] = ss;
      __syncthreads();
      double tot = 0.0;
      for (int i = 0; i < kW; ++i) tot += red[i];
      eps = sqrt(tot) / sqrt(static_cast<double>(N));
      __syncthreads();  // red is reused by the next system
    }
  } else if (ns_order > 0) {
    // NS: P = I − X0·A, T = I + P, T = T·P + I (order−1 times), X = T·X0
    product_coop<N>(X, Am, -1.0, nullptr, 0.0, 1.0, P, w, g, t, false);
    for (int i = threadIdx.x; i < N * ld; i += kThreadsC) {
      V.re[i] = P.re[i];
      V.im[i] = P.im[i];
    }
    __syncthreads();
    if (threadIdx.x < N) V.re[threadIdx.x * ld + threadIdx.x] += 1.0;
    __syncthreads();
    for (int step = 2; step <= ns_order; ++step) product_coop<N>(V, P, 1.0, nullptr, 0.0, 1.0, V, w, g, t, false);
    product_coop<N>(V, X, 1.0, nullptr, 0.0, 0.0, P, w, g, t, false);
    for (int i = threadIdx.x; i < N * ld; i += kThreadsC) {
      X.re[i] = P.re[i];
      X.im[i] = P.im[i];
    }
    __syncthreads();
  }
  return eps;
}

template <int N>
__global__ void __launch_bounds__(32 * (N / 8)) batched_gen_coop_kernel(const double2* __restrict__ A, int64_t batch,
                                                                        int p, int iters, int ns_order,
                                                                        double2* __restrict__ Xout,
                                                                        double* __restrict__ eps_last) {
  extern __shared__ __align__(16) double gsm[];
  constexpr int ld = Gen<N>::kLd, kW = N / 8, kThreadsC = 32 * kW;
  __shared__ double red[kW];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  Pl Am, X, P, V;
  warp_planes<N>(gsm, Am, X, P, V);
  for (int64_t s = blockIdx.x; s < batch; s += gridDim.x) {
    const double2* As = A + s * N * N;
    for (int e = threadIdx.x; e < N * N; e += kThreadsC) {
      const double2 v = __ldg(As + e);
      Am.re[(e / N) * ld + e % N] = v.x;
      Am.im[(e / N) * ld + e % N] = v.y;
    }
    // (solve_coop's first barrier orders these stores before any read)
    const double eps = solve_coop<N>(Am, X, P, V, p, iters, ns_order, w, g, t, eps_last != nullptr, red);
    if (eps_last && threadIdx.x == 0 && ns_order < 0) eps_last[s] = eps;
    double2* Xs = Xout + s * N * N;
    for (int e = threadIdx.x; e < N * N; e += kThreadsC)
      Xs[e] = make_double2(X.re[(e / N) * ld + e % N], X.im[(e / N) * ld + e % N]);
    __syncthreads();  // X, A are rewritten by the next system
  }
}

// Fused detector for n = 24, 32 users, one block of n/8 warps per uplink: warp w forms the
// 8-row stripe w of A = Hᴴ·H + σ²I (4M DMMA over the antennas), threads < n form z = Hᴴ·y,
// then the NN inverse (solve_coop) and x̂ = X·z.
template <int N>
__global__ void __launch_bounds__(32 * (N / 8)) detect_gen_coop_kernel(const double2* __restrict__ H,
                                                                       const double2* __restrict__ Y, int64_t batch,
                                                                       int ant, double sigma2, int p, int iters,
                                                                       double2* __restrict__ xhat,
                                                                       double2* __restrict__ Xout,
                                                                       double* __restrict__ eps_last) {
  extern __shared__ __align__(16) double gsm[];
  constexpr int ld = Gen<N>::kLd, kW = N / 8, kThreadsC = 32 * kW;
  __shared__ double red[kW];
  __shared__ double zs[2][N];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  Pl Am, X, P, V;
  warp_planes<N>(gsm, Am, X, P, V);
  for (int64_t s = blockIdx.x; s < batch; s += gridDim.x) {
    const double2* Hs = H + s * (int64_t)ant * N;
    const double2* Ys = Y + s * (int64_t)ant;
#pragma unroll 1
    for (int tj = 0; tj < Gen<N>::kT; ++tj) {
      double cr[2] = {0.0, 0.0}, ci[2] = {0.0, 0.0};
      for (int kb = 0; kb < ant / 4; ++kb) {
        const int a = 4 * kb + t;
        const double2 hl = __ldg(Hs + (int64_t)a * N + 8 * w + g);  // conj → (x, −y)
        const double2 hr = __ldg(Hs + (int64_t)a * N + 8 * tj + g);
        dmma_8x8x4(cr[0], cr[1], hl.x, hr.x);
        dmma_8x8x4(cr[0], cr[1], hl.y, hr.y);  // −(−y)·y
        dmma_8x8x4(ci[0], ci[1], hl.x, hr.y);
        dmma_8x8x4(ci[0], ci[1], -hl.y, hr.x);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 8 * w + g, c = 8 * tj + 2 * t + h;
        Am.re[r * ld + c] = cr[h] + (r == c ? sigma2 : 0.0);
        Am.im[r * ld + c] = ci[h];
      }
    }
    if (threadIdx.x < N) {
      double zr = 0.0, zi = 0.0;
      for (int a = 0; a < ant; ++a) {
        const double2 h = __ldg(Hs + (int64_t)a * N + threadIdx.x), y = __ldg(Ys + a);
        zr = fma(h.x, y.x, fma(h.y, y.y, zr));
        zi = fma(h.x, y.y, fma(-h.y, y.x, zi));
      }
      zs[0][threadIdx.x] = zr;
      zs[1][threadIdx.x] = zi;
    }
    const double eps = solve_coop<N>(Am, X, P, V, p, iters, -1, w, g, t, eps_last != nullptr, red);
    if (eps_last && threadIdx.x == 0) eps_last[s] = eps;
    if (threadIdx.x < N) {  // x̂ = X·z, row threadIdx.x
      double xr = 0.0, xi = 0.0;
      for (int j = 0; j < N; ++j) {
        const double a = X.re[threadIdx.x * ld + j], b = X.im[threadIdx.x * ld + j];
        xr = fma(a, zs[0][j], fma(-b, zs[1][j], xr));
        xi = fma(a, zs[1][j], fma(b, zs[0][j], xi));
      }
      xhat[s * N + threadIdx.x] = make_double2(xr, xi);
    }
    if (Xout) {
      double2* Xs = Xout + s * N * N;
      for (int e = threadIdx.x; e < N * N; e += kThreadsC)
        Xs[e] = make_double2(X.re[(e / N) * ld + e % N], X.im[(e / N) * ld + e % N]);
    }
    __syncthreads();  // A, X, z are rewritten by the next uplink
  }
}

template <int N, auto K>
int launch_coop(int64_t batch, cudaStream_t s, void** args) {
  constexpr int threads = 32 * (N / 8);
  const int smem = static_cast<int>(Gen<N>::kBytesPerWarp);  // one system's matrices
  NNB_TRY(ensure_smem<K>(smem));
  int per_sm = 0, dev = 0, sms = 0;
  NNB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, K, threads, smem));
  NNB_CUDA(cudaGetDevice(&dev));
  NNB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const unsigned grid =
      static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(batch, (int64_t)sms * std::max(1, per_sm))));
  NNB_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(K), dim3(grid), dim3(threads), args, smem, s));
  count_launch();
  return 0;
}

template <auto K>
int launch_gen(size_t smem_per_warp, int64_t batch, cudaStream_t s, void** args) {
  int warps = static_cast<int>(std::min<size_t>(4, (200 * 1024) / smem_per_warp));
  if (warps < 1) warps = 1;
  const int smem = static_cast<int>(smem_per_warp * warps);
  NNB_TRY(ensure_smem<K>(smem));
  int per_sm = 0, dev = 0, sms = 0;
  NNB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, K, 32 * warps, smem));
  NNB_CUDA(cudaGetDevice(&dev));
  NNB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t want = (batch + warps - 1) / warps;
  const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * std::max(1, per_sm))));
  NNB_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(K), dim3(grid), dim3(32 * warps), args, smem, s));
  count_launch();
  return 0;
}

}  // namespace

int batched_nn_gen(const double* A, int64_t batch, int n, int p, int iters, int ns_order, double* X, double* eps,
                   cudaStream_t s) {
  if (batch == 0) return 0;
  const double2* a = reinterpret_cast<const double2*>(A);
  double2* x = reinterpret_cast<double2*>(X);
  void* args[] = {&a, &batch, &p, &iters, &ns_order, &x, &eps};
  switch (n) {
    case 8: return launch_gen<batched_gen_kernel<8>>(Gen<8>::kBytesPerWarp, batch, s, args);
    case 24: return launch_coop<24, batched_gen_coop_kernel<24>>(batch, s, args);
    case 32: return launch_coop<32, batched_gen_coop_kernel<32>>(batch, s, args);
    default: return fail(1, "batched: n must be 8, 16, 24 or 32");
  }
}

int mimo_detect_gen(const double* H, const double* y, int64_t batch, int antennas, int users, double sigma2, int p,
                    int iters, double* xhat, double* X, double* eps, cudaStream_t s) {
  if (batch == 0) return 0;
  const double2* h = reinterpret_cast<const double2*>(H);
  const double2* yy = reinterpret_cast<const double2*>(y);
  double2* xh = reinterpret_cast<double2*>(xhat);
  double2* x = reinterpret_cast<double2*>(X);
  void* args[] = {&h, &yy, &batch, &antennas, &sigma2, &p, &iters, &xh, &x, &eps};
  switch (users) {
    case 8: return launch_gen<detect_gen_kernel<8>>(Gen<8>::kBytesPerWarp, batch, s, args);
    case 24: return launch_coop<24, detect_gen_coop_kernel<24>>(batch, s, args);
    case 32: return launch_coop<32, detect_gen_coop_kernel<32>>(batch, s, args);
    default: return fail(1, "mimo detect: users must be 8, 16, 24 or 32");
  }
}

}  // namespace nnb
