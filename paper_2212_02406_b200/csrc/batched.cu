// Batched Nested Neumann inversion of small complex systems (massive-MIMO
// Gram matrices, BASELINE config 1: 262144 × 16×16 complex128).
//
// One warp owns one system at a time (grid-stride over systems):
//   * A is read once from HBM (coalesced 16-byte loads) straight into the
//     DMMA B-operand registers it occupies for the whole solve;
//   * X0 = diag(A)^-1 (Jacobi) is formed in shared memory;
//   * every iterate (X, P, V) stays in per-warp shared memory, planar re/im,
//     16×16 doubles with the XOR swizzle  (r, c) -> r*16 + (c ^ 4*(r&3)),
//     which makes both the A-operand (row=g, col=t) and the B-operand
//     (row=t, col=g) fragment loads of mma.m8n8k4 conflict-free (2
//     wavefronts per 32 doubles) and keeps the epilogue's double2 stores
//     at the 4-wavefront minimum;
//   * each complex 16×16×16 product is 64 DMMA.8x8x4 (4M: re·re − im·im,
//     re·im + im·re) with the "I −", "+X" and ‖·‖² terms in the epilogue;
//   * X is written once (coalesced) and, for the NN chain, eps of the final
//     residual is written per system.
// The nest follows the reference's operand order (proj/src/solver.cpp:93-103):
//   P = I − X·A;  V = X + P·X;  V = X + P·V (p−1 more);  X = V,
// and the Neumann-series baseline follows ns_sum (proj/src/solver.cpp:77-91):
//   P = I − X0·A;  T = I + P;  T = T·P + I (order−1 times);  X = T·X0.
#include "engine.cuh"

namespace nnb {
namespace {

constexpr int kN = 16;
constexpr int kMat = kN * kN;            // doubles per plane
constexpr int kWarpsPerCta = 4;
constexpr int kThreads = kWarpsPerCta * 32;

__device__ __forceinline__ int swz(int r, int c) { return r * kN + (c ^ (4 * (r & 3))); }

struct SMat {
  double* re;
  double* im;
};

// acc[mt][nt][plane][i]: C[8mt+g][8nt+2t+i] (plane 0 = re, 1 = im)
using Acc = double[2][2][2][2];

__device__ __forceinline__ void acc_zero(Acc& acc) {
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int p = 0; p < 2; ++p) acc[a][b][p][0] = acc[a][b][p][1] = 0.0;
}

// acc += L·R, L from shared (A-operand), R from shared (B-operand).
__device__ __forceinline__ void zmma_ss(Acc& acc, const SMat& L, const SMat& R, int g, int t) {
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    double lr[2], li[2], rr[2], ri[2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int idx = swz(8 * mt + g, 4 * kb + t);
      lr[mt] = L.re[idx];
      li[mt] = L.im[idx];
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int idx = swz(4 * kb + t, 8 * nt + g);
      rr[nt] = R.re[idx];
      ri[nt] = R.im[idx];
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const double nli = -li[mt];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        dmma_8x8x4(acc[mt][nt][0][0], acc[mt][nt][0][1], lr[mt], rr[nt]);
        dmma_8x8x4(acc[mt][nt][0][0], acc[mt][nt][0][1], nli, ri[nt]);
        dmma_8x8x4(acc[mt][nt][1][0], acc[mt][nt][1][1], lr[mt], ri[nt]);
        dmma_8x8x4(acc[mt][nt][1][0], acc[mt][nt][1][1], li[mt], rr[nt]);
      }
    }
  }
}

// acc += L·A with A's B-operand fragments held in registers:
// areg[nt][kb][plane] = A[4kb+t][8nt+g].
__device__ __forceinline__ void zmma_sr(Acc& acc, const SMat& L, const double (&areg)[2][4][2],
                                        int g, int t) {
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    double lr[2], li[2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int idx = swz(8 * mt + g, 4 * kb + t);
      lr[mt] = L.re[idx];
      li[mt] = L.im[idx];
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const double nli = -li[mt];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        dmma_8x8x4(acc[mt][nt][0][0], acc[mt][nt][0][1], lr[mt], areg[nt][kb][0]);
        dmma_8x8x4(acc[mt][nt][0][0], acc[mt][nt][0][1], nli, areg[nt][kb][1]);
        dmma_8x8x4(acc[mt][nt][1][0], acc[mt][nt][1][1], lr[mt], areg[nt][kb][1]);
        dmma_8x8x4(acc[mt][nt][1][0], acc[mt][nt][1][1], li[mt], areg[nt][kb][0]);
      }
    }
  }
}

// out = alpha·acc + (D ? D : 0) + gamma·I, stored to shared `out` (may alias D).
// Returns this lane's Σ|out|² when `want_ss`.
__device__ __forceinline__ double epilogue(const Acc& acc, double alpha, const SMat* D,
                                           double gamma, const SMat& out, int g, int t,
                                           bool want_ss) {
  double ss = 0.0;
  __syncwarp();  // every lane finished reading operands that `out` may overwrite
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int r = 8 * mt + g, c = 8 * nt + 2 * t;
      const int idx = swz(r, c);
      double2 vr = make_double2(alpha * acc[mt][nt][0][0], alpha * acc[mt][nt][0][1]);
      double2 vi = make_double2(alpha * acc[mt][nt][1][0], alpha * acc[mt][nt][1][1]);
      if (D) {
        const double2 dr = *reinterpret_cast<const double2*>(D->re + idx);
        const double2 di = *reinterpret_cast<const double2*>(D->im + idx);
        vr.x += dr.x; vr.y += dr.y;
        vi.x += di.x; vi.y += di.y;
      }
      if (r == c) vr.x += gamma;
      if (r == c + 1) vr.y += gamma;
      *reinterpret_cast<double2*>(out.re + idx) = vr;
      *reinterpret_cast<double2*>(out.im + idx) = vi;
      if (want_ss) {
        ss = fma(vr.x, vr.x, ss); ss = fma(vi.x, vi.x, ss);
        ss = fma(vr.y, vr.y, ss); ss = fma(vi.y, vi.y, ss);
      }
    }
  __syncwarp();
  return ss;
}

// Σ|I − X·A|² without storing the residual.
__device__ __forceinline__ double residual_ss(const Acc& acc, int g, int t) {
  double ss = 0.0;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int r = 8 * mt + g, c = 8 * nt + 2 * t;
      double v0 = -acc[mt][nt][0][0], v1 = -acc[mt][nt][0][1];
      if (r == c) v0 += 1.0;
      if (r == c + 1) v1 += 1.0;
      ss = fma(v0, v0, ss);
      ss = fma(v1, v1, ss);
      ss = fma(acc[mt][nt][1][0], acc[mt][nt][1][0], ss);
      ss = fma(acc[mt][nt][1][1], acc[mt][nt][1][1], ss);
    }
  return ss;
}

template <int P>
__global__ void __launch_bounds__(kThreads)
    batched_z16_kernel(const double2* __restrict__ A, int64_t batch, int iters, int ns_order,
                       double2* __restrict__ Xout, double* __restrict__ eps_last, int ns_mode) {
  __shared__ __align__(16) double smem[kWarpsPerCta][3][2][kMat];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  SMat X{smem[warp][0][0], smem[warp][0][1]};
  SMat Pm{smem[warp][1][0], smem[warp][1][1]};
  SMat V{smem[warp][2][0], smem[warp][2][1]};

  const int64_t gw = blockIdx.x * (int64_t)kWarpsPerCta + warp;
  const int64_t nw = (int64_t)gridDim.x * kWarpsPerCta;
  for (int64_t s = gw; s < batch; s += nw) {
    const double2* As = A + s * kMat;
    // A's B-operand fragments: A[4kb+t][8nt+g]
    double areg[2][4][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int kb = 0; kb < 4; ++kb) {
        const double2 v = __ldg(As + (4 * kb + t) * kN + 8 * nt + g);
        areg[nt][kb][0] = v.x;
        areg[nt][kb][1] = v.y;
      }
    // X0 = diag(A)^-1 (Smith's complex reciprocal, as libgcc's __divdc3)
    for (int i = lane; i < kMat; i += 32) {
      X.re[i] = 0.0;
      X.im[i] = 0.0;
    }
    __syncwarp();
    if (lane < kN) {
      const double2 d = __ldg(As + lane * kN + lane);
      double xr, xi;
      if (fabs(d.x) >= fabs(d.y)) {
        const double r = d.y / d.x, den = d.x + d.y * r;
        xr = 1.0 / den;
        xi = -r / den;
      } else {
        const double r = d.x / d.y, den = d.x * r + d.y;
        xr = r / den;
        xi = -1.0 / den;
      }
      X.re[swz(lane, lane)] = xr;
      X.im[swz(lane, lane)] = xi;
    }
    __syncwarp();

    Acc acc;
    if (!ns_mode) {
      // ---- Nested Neumann: `iters` nests of depth P ----
      for (int it = 0; it < iters; ++it) {
        acc_zero(acc);
        zmma_sr(acc, X, areg, g, t);                    // X·A
        epilogue(acc, -1.0, nullptr, 1.0, Pm, g, t, false);  // P = I − X·A
        const SMat* v = &X;
#pragma unroll
        for (int j = 1; j <= P; ++j) {
          acc_zero(acc);
          zmma_ss(acc, Pm, *v, g, t);                   // P·V
          const SMat& dst = (j == P) ? X : V;           // last Horner step lands in X
          epilogue(acc, 1.0, &X, 0.0, dst, g, t, false);  // V = X + P·V
          v = &V;
        }
      }
      // final residual eps = ‖I − X·A‖_F / √n
      acc_zero(acc);
      zmma_sr(acc, X, areg, g, t);
      double ss = warp_sum(residual_ss(acc, g, t));
      if (lane == 0 && eps_last) eps_last[s] = sqrt(ss) * 0.25;  // 1/sqrt(16)
    } else if (ns_order > 0) {
      // ---- Neumann-series baseline of `ns_order` terms from X0 ----
      acc_zero(acc);
      zmma_sr(acc, X, areg, g, t);
      epilogue(acc, -1.0, nullptr, 1.0, Pm, g, t, false);  // P = I − X0·A
      // T = I + P  (into V)
      for (int i = lane; i < kMat; i += 32) {
        V.re[i] = Pm.re[i];
        V.im[i] = Pm.im[i];
      }
      __syncwarp();
      if (lane < kN) V.re[swz(lane, lane)] += 1.0;
      __syncwarp();
      for (int step = 2; step <= ns_order; ++step) {
        acc_zero(acc);
        zmma_ss(acc, V, Pm, g, t);                      // T·P
        epilogue(acc, 1.0, nullptr, 1.0, V, g, t, false);  // T = T·P + I
      }
      acc_zero(acc);
      zmma_ss(acc, V, X, g, t);                         // T·X0
      epilogue(acc, 1.0, nullptr, 0.0, X, g, t, false);
    }
    // store X (planar swizzled shared -> interleaved global, coalesced 16B)
    double2* Xs = Xout + s * kMat;
#pragma unroll
    for (int q = 0; q < kMat / 32; ++q) {
      const int e = q * 32 + lane;
      const int idx = swz(e / kN, e % kN);
      Xs[e] = make_double2(X.re[idx], X.im[idx]);
    }
    __syncwarp();
  }
}

}  // namespace

int batched_nn_z16(const double* A, int64_t batch, int p, int iters, int ns_order, double* X,
                   double* eps_last, cudaStream_t s) {
  // ns_order < 0: Nested Neumann chain; ns_order >= 0: Neumann series of that order
  const int ns_mode = ns_order >= 0 ? 1 : 0;
  if (batch <= 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (batch + kWarpsPerCta - 1) / kWarpsPerCta;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(want, (int64_t)sms * 4));
  const double2* a = reinterpret_cast<const double2*>(A);
  double2* x = reinterpret_cast<double2*>(X);
  switch (ns_mode ? 1 : p) {
    case 1: batched_z16_kernel<1><<<grid, kThreads, 0, s>>>(a, batch, iters, ns_order, x, eps_last, ns_mode); break;
    case 2: batched_z16_kernel<2><<<grid, kThreads, 0, s>>>(a, batch, iters, ns_order, x, eps_last, ns_mode); break;
    case 3: batched_z16_kernel<3><<<grid, kThreads, 0, s>>>(a, batch, iters, ns_order, x, eps_last, ns_mode); break;
    case 4: batched_z16_kernel<4><<<grid, kThreads, 0, s>>>(a, batch, iters, ns_order, x, eps_last, ns_mode); break;
    default: return fail(2, "batched: depth p must be in 1..4");
  }
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace nnb
