// Batched Nested Neumann inversion of small complex systems (massive-MIMO
// Gram matrices, BASELINE config 1: 262144 × 16×16 complex128).
//
// One warp owns one system at a time (grid-stride over systems, persistent
// grid sized to the measured occupancy):
//   * A is read once from HBM (coalesced 16-byte loads) straight into the
//     DMMA B-operand registers it occupies for the whole solve; the next
//     system's A is prefetched into registers while the current one iterates
//     (PREFETCH), hiding the HBM latency behind ~13k cycles of DMMA work;
//   * X0 = diag(A)^-1 (Jacobi) is formed in shared memory;
//   * every iterate (X, P, V) stays in per-warp shared memory, planar re/im,
//     16×16 doubles with an XOR swizzle (swz below) that makes both the
//     A-operand (row=g, col=t) and the B-operand (row=t, col=g) fragment
//     loads of mma.m8n8k4 conflict-free (2 wavefronts per 32 doubles) and
//     keeps the epilogue's double2 stores at the 4-wavefront minimum;
//   * each complex 16×16×16 product runs on DMMA.8x8x4 either as 4M
//     (re·re − im·im, re·im + im·re: 64 DMMA) or as 3M (Gauss:
//     P1 = re·re, P2 = im·im, P3 = (re+im)·(re+im); re = P1 − P2,
//     im = P3 − P1 − P2: 48 DMMA), with the "I −", "+X" and ‖·‖² terms in
//     the epilogue;
//   * X is written once (coalesced) and, for the NN chain, eps of the final
//     residual is written per system.
// The nest follows the reference's operand order (proj/src/solver.cpp:93-103):
//   P = I − X·A;  V = X + P·X;  V = X + P·V (p−1 more);  X = V,
// and the Neumann-series baseline follows ns_sum (proj/src/solver.cpp:77-91):
//   P = I − X0·A;  T = I + P;  T = T·P + I (order−1 times);  X = T·X0.
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "engine.cuh"

namespace nnb {
namespace {

constexpr int kN = 16;
constexpr int kMat = kN * kN;  // doubles per plane
constexpr int kWarpsPerCta = 4;
constexpr int kThreads = kWarpsPerCta * 32;

// (r, c) -> 16r + (c ^ key(r)), key = 4·(r bits 0 and 1 swapped) ∈ {0, 8, 4, 12}:
// conflict-free for the m8n8k4 A- and B-fragment loads (2 wavefronts per 32
// doubles) and for the epilogue's double2 stores / seed loads (4 wavefronts),
// because rows 2q and 2q+1 differ in key bit 3 (ncu: the plain 4·(r&3) key
// doubled those 16-byte accesses).
__device__ __forceinline__ int swz(int r, int c) { return r * kN + (c ^ (4 * (((r & 1) << 1) | ((r >> 1) & 1)))); }

struct SMat {
  double* re;
  double* im;
};

// Accumulators for C[8mt+g][8nt+2t+i]: 4M keeps (re, im); 3M keeps (P1, P2, P3).
template <bool M3>
struct ZAcc {
  double v[2][2][M3 ? 3 : 2][2];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int p = 0; p < (M3 ? 3 : 2); ++p) v[a][b][p][0] = v[a][b][p][1] = 0.0;
  }
  // one k-step: L fragments (lr, li) for 2 m-tiles, R fragments (rr, ri) for 2 n-tiles
  __device__ __forceinline__ void step(const double (&lr)[2], const double (&li)[2], const double (&rr)[2],
                                       const double (&ri)[2]) {
    if constexpr (M3) {
      double ls[2], rs[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        ls[i] = lr[i] + li[i];
        rs[i] = rr[i] + ri[i];
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          dmma_8x8x4(v[mt][nt][0][0], v[mt][nt][0][1], lr[mt], rr[nt]);
          dmma_8x8x4(v[mt][nt][1][0], v[mt][nt][1][1], li[mt], ri[nt]);
          dmma_8x8x4(v[mt][nt][2][0], v[mt][nt][2][1], ls[mt], rs[nt]);
        }
    } else {
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const double nli = -li[mt];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          dmma_8x8x4(v[mt][nt][0][0], v[mt][nt][0][1], lr[mt], rr[nt]);
          dmma_8x8x4(v[mt][nt][0][0], v[mt][nt][0][1], nli, ri[nt]);
          dmma_8x8x4(v[mt][nt][1][0], v[mt][nt][1][1], lr[mt], ri[nt]);
          dmma_8x8x4(v[mt][nt][1][0], v[mt][nt][1][1], li[mt], rr[nt]);
        }
      }
    }
  }
  // 3M, Hermitian result (HᴴH): the upper tiles (0,0), (0,1), (1,1) only — the
  // (1,0) tile is the conjugate transpose of (0,1) (gram_epilogue mirrors it)
  __device__ __forceinline__ void step_herm(const double (&lr)[2], const double (&li)[2], const double (&rr)[2],
                                            const double (&ri)[2]) {
    const double ls[2] = {lr[0] + li[0], lr[1] + li[1]}, rs[2] = {rr[0] + ri[0], rr[1] + ri[1]};
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = mt; nt < 2; ++nt) {
        dmma_8x8x4(v[mt][nt][0][0], v[mt][nt][0][1], lr[mt], rr[nt]);
        dmma_8x8x4(v[mt][nt][1][0], v[mt][nt][1][1], li[mt], ri[nt]);
        dmma_8x8x4(v[mt][nt][2][0], v[mt][nt][2][1], ls[mt], rs[nt]);
      }
  }
  // 3M only: seed the accumulators with s·(D + γ·I), s = −1 when NEG, as
  // P1 = re, P2 = 0, P3 = re + im — the "+D" and "γI" then cost 2 DADD per
  // element pair instead of 4 after the product, and the sign folds into
  // epilogue_seeded's operand order (DADD shares the FP64 pipe with DMMA).
  template <bool NEG>
  __device__ __forceinline__ void seed(const SMat* D, double gamma, int g, int t) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int r = 8 * mt + g, c = 8 * nt + 2 * t;
        double2 dr = make_double2(0.0, 0.0), di = make_double2(0.0, 0.0);
        if (D) {
          const int idx = swz(r, c);
          dr = *reinterpret_cast<const double2*>(D->re + idx);
          di = *reinterpret_cast<const double2*>(D->im + idx);
        }
        if (r == c) dr.x += gamma;
        if (r == c + 1) dr.y += gamma;
        double2 ds = D ? make_double2(dr.x + di.x, dr.y + di.y) : dr;
        v[mt][nt][0][0] = NEG ? -dr.x : dr.x;
        v[mt][nt][0][1] = NEG ? -dr.y : dr.y;
        v[mt][nt][1][0] = v[mt][nt][1][1] = 0.0;
        v[mt][nt][2][0] = NEG ? -ds.x : ds.x;
        v[mt][nt][2][1] = NEG ? -ds.y : ds.y;
      }
  }
  __device__ __forceinline__ double re(int mt, int nt, int i) const {
    if constexpr (M3) return v[mt][nt][0][i] - v[mt][nt][1][i];
    else return v[mt][nt][0][i];
  }
  __device__ __forceinline__ double im(int mt, int nt, int i) const {
    if constexpr (M3) return v[mt][nt][2][i] - v[mt][nt][0][i] - v[mt][nt][1][i];
    else return v[mt][nt][1][i];
  }
};

// acc += L·R, L (A-operand) and R (B-operand) from shared memory.
template <bool M3>
__device__ __forceinline__ void zmma_ss(ZAcc<M3>& acc, const SMat& L, const SMat& R, int g, int t) {
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
    acc.step(lr, li, rr, ri);
  }
}

// 3M acc += L·R where L·R is Hermitian: tiles (0,0), (0,1), (1,1) only (36 DMMA
// instead of 48); epilogue_seeded_herm mirrors (0,1) into (1,0).
__device__ __forceinline__ void zmma_ss_herm(ZAcc<true>& acc, const SMat& L, const SMat& R, int g, int t) {
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
    acc.step_herm(lr, li, rr, ri);
  }
}

// acc += L·A with A's B-operand fragments in registers: areg[nt][kb][plane] = A[4kb+t][8nt+g].
template <bool M3>
__device__ __forceinline__ void zmma_sr(ZAcc<M3>& acc, const SMat& L, const double (&areg)[2][4][2], int g,
                                        int t) {
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    double lr[2], li[2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int idx = swz(8 * mt + g, 4 * kb + t);
      lr[mt] = L.re[idx];
      li[mt] = L.im[idx];
    }
    const double rr[2] = {areg[0][kb][0], areg[1][kb][0]};
    const double ri[2] = {areg[0][kb][1], areg[1][kb][1]};
    acc.step(lr, li, rr, ri);
  }
}

// out = alpha·acc + (D ? D : 0) + gamma·I, stored to shared `out` (may alias D).
template <bool M3>
__device__ __forceinline__ void epilogue(const ZAcc<M3>& acc, double alpha, const SMat* D, double gamma,
                                         const SMat& out, int g, int t) {
  __syncwarp();  // every lane finished reading operands that `out` may overwrite
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int r = 8 * mt + g, c = 8 * nt + 2 * t;
      const int idx = swz(r, c);
      double2 vr = make_double2(alpha * acc.re(mt, nt, 0), alpha * acc.re(mt, nt, 1));
      double2 vi = make_double2(alpha * acc.im(mt, nt, 0), alpha * acc.im(mt, nt, 1));
      if (D) {
        const double2 dr = *reinterpret_cast<const double2*>(D->re + idx);
        const double2 di = *reinterpret_cast<const double2*>(D->im + idx);
        vr.x += dr.x;
        vr.y += dr.y;
        vi.x += di.x;
        vi.y += di.y;
      }
      if (r == c) vr.x += gamma;
      if (r == c + 1) vr.y += gamma;
      *reinterpret_cast<double2*>(out.re + idx) = vr;
      *reinterpret_cast<double2*>(out.im + idx) = vi;
    }
  __syncwarp();
}

// A = HᴴH + σ²·I from step_herm's three tiles; tile (1,0) = conj(tile (0,1))ᵀ.
__device__ __forceinline__ void gram_epilogue(const ZAcc<true>& acc, double sigma2, const SMat& out, int g, int t) {
  __syncwarp();
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = mt; nt < 2; ++nt) {
      const int r = 8 * mt + g, c = 8 * nt + 2 * t;
      double2 vr = make_double2(acc.re(mt, nt, 0), acc.re(mt, nt, 1));
      const double2 vi = make_double2(acc.im(mt, nt, 0), acc.im(mt, nt, 1));
      if (r == c) vr.x += sigma2;
      if (r == c + 1) vr.y += sigma2;
      *reinterpret_cast<double2*>(out.re + swz(r, c)) = vr;
      *reinterpret_cast<double2*>(out.im + swz(r, c)) = vi;
      if (mt != nt) {  // mirror: A[c+i][r] = conj(A[r][c+i])
        out.re[swz(c, r)] = vr.x;
        out.im[swz(c, r)] = -vi.x;
        out.re[swz(c + 1, r)] = vr.y;
        out.im[swz(c + 1, r)] = -vi.y;
      }
    }
  __syncwarp();
}

// Largest |x| of a few doubles, to within a factor 2, by integer ops on their high words
// (sign cleared; IEEE order = integer order) — kept off the FP64 pipe, which DMMA uses.
__device__ __forceinline__ uint32_t mag_hi(double x) {
  return static_cast<uint32_t>(__double2hiint(x)) & 0x7fffffffu;
}

// 3M with seeded accumulators: out = s·acc (s = −1 when NEG), stored to shared `out`.
// Returns the high word of this lane's largest |out| entry (dead code unless used).
template <bool NEG>
__device__ __forceinline__ uint32_t epilogue_seeded(const ZAcc<true>& acc, const SMat& out, int g, int t) {
  uint32_t mx = 0;
  __syncwarp();  // every lane finished reading operands that `out` may overwrite
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int idx = swz(8 * mt + g, 8 * nt + 2 * t);
      double2 vr, vi;
      const double* p0 = acc.v[mt][nt][0];
      const double* p1 = acc.v[mt][nt][1];
      const double* p2 = acc.v[mt][nt][2];
      if (NEG) {
        vr = make_double2(p1[0] - p0[0], p1[1] - p0[1]);
        vi = make_double2((p0[0] + p1[0]) - p2[0], (p0[1] + p1[1]) - p2[1]);
      } else {
        vr = make_double2(p0[0] - p1[0], p0[1] - p1[1]);
        vi = make_double2(p2[0] - (p0[0] + p1[0]), p2[1] - (p0[1] + p1[1]));
      }
      *reinterpret_cast<double2*>(out.re + idx) = vr;
      *reinterpret_cast<double2*>(out.im + idx) = vi;
      mx = max(max(max(mx, mag_hi(vr.x)), max(mag_hi(vr.y), mag_hi(vi.x))), mag_hi(vi.y));
    }
  __syncwarp();
  return mx;
}

// epilogue_seeded<false> for a Hermitian result from zmma_ss_herm: tiles (0,0),
// (0,1), (1,1) stored, (1,0) = conj((0,1))ᵀ.
__device__ __forceinline__ void epilogue_seeded_herm(const ZAcc<true>& acc, const SMat& out, int g, int t) {
  __syncwarp();  // every lane finished reading operands that `out` may overwrite
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = mt; nt < 2; ++nt) {
      const int r = 8 * mt + g, c = 8 * nt + 2 * t;
      const double* p0 = acc.v[mt][nt][0];
      const double* p1 = acc.v[mt][nt][1];
      const double* p2 = acc.v[mt][nt][2];
      const double2 vr = make_double2(p0[0] - p1[0], p0[1] - p1[1]);
      const double2 vi = make_double2(p2[0] - (p0[0] + p1[0]), p2[1] - (p0[1] + p1[1]));
      *reinterpret_cast<double2*>(out.re + swz(r, c)) = vr;
      *reinterpret_cast<double2*>(out.im + swz(r, c)) = vi;
      if (mt != nt) {
        out.re[swz(c, r)] = vr.x;
        out.im[swz(c, r)] = -vi.x;
        out.re[swz(c + 1, r)] = vr.y;
        out.im[swz(c + 1, r)] = -vi.y;
      }
    }
  __syncwarp();
}

// One Horner step V' = X + P·V (3M, seeded).  For Hermitian A and X every such
// product is Hermitian — P·V = poly(P)·X and (I − XA)^k X = X (I − AX)^k — so
// `herm` computes three of its four 8×8 tiles and mirrors the fourth.
__device__ __forceinline__ void horner_step(ZAcc<true>& acc, const SMat& X, const SMat& Pm, const SMat& v,
                                            const SMat& out, bool herm, int g, int t) {
  acc.template seed<false>(&X, 0.0, g, t);
  if (herm) {
    zmma_ss_herm(acc, Pm, v, g, t);
    epilogue_seeded_herm(acc, out, g, t);
  } else {
    zmma_ss(acc, Pm, v, g, t);
    epilogue_seeded<false>(acc, out, g, t);
  }
}

// A == Aᴴ exactly (NaN never equal: such systems take the full products), from
// A's register fragments alone: lane (g, t) holds A[4kb+t][8nt+g]; the
// transposed element A[8nt+g][4kb+t] sits in lane (4(kb&1)+t, g&3) as its
// fragment [kb>>1][2nt + (g>>2)], fetched by shuffles (both candidates, then
// selected).  Called once the fragments are in use anyway, so it adds no wait.
__device__ __forceinline__ bool is_hermitian(const double (&areg)[2][4][2], int g, int t) {
  bool ok = true;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
      if (nt == 1 && kb < 2) continue;  // the tile above the diagonal: its mirror (nt 0, kb 2..3) checked it
      const int src = (4 * (kb & 1) + t) * 4 + (g & 3);
      const double r0 = __shfl_sync(0xffffffffu, areg[kb >> 1][2 * nt][0], src);
      const double i0 = __shfl_sync(0xffffffffu, areg[kb >> 1][2 * nt][1], src);
      const double r1 = __shfl_sync(0xffffffffu, areg[kb >> 1][2 * nt + 1][0], src);
      const double i1 = __shfl_sync(0xffffffffu, areg[kb >> 1][2 * nt + 1][1], src);
      const bool hi = (g >> 2) != 0;
      ok &= (hi ? r1 : r0) == areg[nt][kb][0] && (hi ? i1 : i0) == -areg[nt][kb][1];
    }
  return __all_sync(0xffffffffu, ok);
}

// Σ|I − X·A|² without storing the residual.
template <bool M3>
__device__ __forceinline__ double residual_ss(const ZAcc<M3>& acc, int g, int t) {
  double ss = 0.0;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int r = 8 * mt + g, c = 8 * nt + 2 * t;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        double vr = -acc.re(mt, nt, i);
        if (r == c + i) vr += 1.0;
        const double vi = acc.im(mt, nt, i);
        ss = fma(vr, vr, ss);
        ss = fma(vi, vi, ss);
      }
    }
  return ss;
}

__device__ __forceinline__ void load_a_frags(const double2* __restrict__ As, int g, int t, double (&areg)[2][4][2]) {
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
      const double2 v = __ldg(As + (4 * kb + t) * kN + 8 * nt + g);
      areg[nt][kb][0] = v.x;
      areg[nt][kb][1] = v.y;
    }
}

// Nest 0 from the diagonal (Jacobi) X0: P = I − X0·A is a row scaling of A and
// V1 = X0 + P·X0 a column scaling of P, so both are elementwise on the lane's
// A fragments (rows 4kb+t, columns 8nt+g) — the reference's products add only
// zeros to x_r·a_rc and p_rc·x_c.  The remaining p − 1 Horner steps are
// products: nest 0 costs p − 1 products instead of p + 1 (11 instead of 13 per
// C2 system).  Returns with X = X1 and P holding I − X0·A.
template <int P, bool M3>
__device__ __forceinline__ void first_nest_diag(ZAcc<M3>& acc, const SMat& X, const SMat& Pm, const SMat& V,
                                                const double (&areg)[2][4][2], int g, int t, bool herm_ok,
                                                bool* herm_out) {
  double2 xr[4], xc[2], pv[2][4];
#pragma unroll
  for (int kb = 0; kb < 4; ++kb) {
    const int r = 4 * kb + t;
    xr[kb] = make_double2(X.re[swz(r, r)], X.im[swz(r, r)]);
  }
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int c = 8 * nt + g;
    xc[nt] = make_double2(X.re[swz(c, c)], X.im[swz(c, c)]);
  }
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
      const int r = 4 * kb + t, c = 8 * nt + g, idx = swz(r, c);
      const double ar = areg[nt][kb][0], ai = areg[nt][kb][1];
      const double2 p = make_double2((r == c ? 1.0 : 0.0) - (xr[kb].x * ar - xr[kb].y * ai),
                                     -(xr[kb].x * ai + xr[kb].y * ar));
      Pm.re[idx] = p.x;
      Pm.im[idx] = p.y;
      pv[nt][kb] = p;
    }
  __syncwarp();  // every lane has read X0's diagonal before V1 (X itself when p = 1) is written
  const SMat& d1 = (P == 1) ? X : V;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
      const int r = 4 * kb + t, c = 8 * nt + g, idx = swz(r, c);
      const double2 p = pv[nt][kb];
      double vr = p.x * xc[nt].x - p.y * xc[nt].y, vi = p.x * xc[nt].y + p.y * xc[nt].x;
      if (r == c) {
        vr += xr[kb].x;
        vi += xr[kb].y;
      }
      d1.re[idx] = vr;
      d1.im[idx] = vi;
    }
  __syncwarp();
  // A's fragments have arrived (used above): the Hermitian test costs no wait here;
  // the caller passes the result on to the later nests
  const bool herm = herm_ok && (herm_out ? is_hermitian(areg, g, t) : true);
  if (herm_out) *herm_out = herm;
  const SMat* v = &V;
#pragma unroll
  for (int j = 2; j <= P; ++j) {  // V = X0 + P·V; the last step lands in X
    if constexpr (M3) {
      horner_step(acc, X, Pm, *v, (j == P) ? X : V, herm, g, t);
    } else {
      acc.zero();
      zmma_ss(acc, Pm, *v, g, t);
      epilogue(acc, 1.0, &X, 0.0, (j == P) ? X : V, g, t);
    }
  }
}

// Mirrored (Hermitian) Horner products leave a κ·u residual floor — the dense chain's
// NNB_ORDER_SYMMETRIC measured it.  Keep them while ε = ‖I − X·A‖_F/√n, formed for
// free from the nest's P, falls at the nest's order: the first nest whose ε stops
// falling, or lands 1e3× above ε_prev^(p+1) once ε_prev < 1e-2, is at that floor, and
// from there on every product is full (sticky).  The last nest is also full when the
// system is ill-conditioned and the nest would land where the floor decides it
// (ε^(p+1) < 1e-13): κ is estimated from the nest k at which ε first fell below 1e-2
// — (1 − 1/κ)^((p+1)^k) ≈ 1e-2 gives κ ≈ (p+1)^k / 4.6 — and "ill-conditioned" is
// κ > 100, where the mirrored floor (~κ·u) would exceed the parity gate's 1e-12.  One
// full nest restores Newton's self-correction (a κ = 1e5 batch: ε 6.8e-8 with a
// mirrored last nest against the reference's 4.7e-12).  Config 1 (κ <= 4, ε < 1e-2
// after one or two nests) keeps the 25 % cheaper products throughout: 2.40 ms against
// 2.61 with a full last nest.
struct MirrorState {
  float eps_prev = INFINITY;
  int k_drop = -1;  // first nest with ε < 1e-2
};
// Called one nest late (its warp reduction then costs no latency): eps is the size of
// nest `it`'s P — max |P_ij| from the high words (an integer warp max, no FP64 work:
// the FP64 pipe is the one DMMA issues on), which tracks ‖P‖_F/√n within a small
// factor, ample for these thresholds — and the decision is for nest it + 1, which
// would land near ε^((p+1)^2).
template <int P>
__device__ __forceinline__ bool keep_mirrored(float eps, MirrorState& st, int it, bool last) {
  float expect = st.eps_prev, next = eps;
#pragma unroll
  for (int j = 0; j < P; ++j) {
    expect *= st.eps_prev;  // ε_prev^(p+1)
    next *= eps;            // ε^(p+1)
  }
  float next2 = next;
#pragma unroll
  for (int j = 0; j < P; ++j) next2 *= next;  // ε^((p+1)^2), 0 when it underflows
  if (st.k_drop < 0 && eps < 1e-2f) st.k_drop = it;
  float kappa = 1.0f;
  for (int k = 0; k < (st.k_drop < 0 ? it + 1 : st.k_drop); ++k) kappa *= (P + 1);
  const bool ill = kappa > 460.0f;  // κ ≈ (p+1)^k / 4.6 > 100
  const bool ok = eps < st.eps_prev && !(st.eps_prev < 1e-2f && eps > 1e3f * expect) &&
                  !(last && ill && next2 < 1e-13f);
  st.eps_prev = eps;
  return ok;
}
// ε proxy of a P from every lane's high-word maximum
__device__ __forceinline__ float p_size(uint32_t mx) {
  const uint32_t w = __reduce_max_sync(0xffffffffu, mx);
  return static_cast<float>(__hiloint2double(static_cast<int>(w), 0));
}

// NNB_BATCHED_MINB (compile-time) caps registers so that MINB CTAs fit per SM.
#ifndef NNB_BATCHED_MINB
#define NNB_BATCHED_MINB 4
#endif
template <int P, bool M3, bool PREFETCH>
__global__ void __launch_bounds__(kThreads, NNB_BATCHED_MINB)
    batched_z16_kernel(const double2* __restrict__ A, int64_t batch, int iters, int ns_order,
                       double2* __restrict__ Xout, double* __restrict__ eps_last, int ns_mode, int herm_ok) {
  __shared__ __align__(16) double smem[kWarpsPerCta][3][2][kMat];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  SMat X{smem[warp][0][0], smem[warp][0][1]};
  SMat Pm{smem[warp][1][0], smem[warp][1][1]};
  SMat V{smem[warp][2][0], smem[warp][2][1]};

  const int64_t gw = blockIdx.x * (int64_t)kWarpsPerCta + warp;
  const int64_t nw = (int64_t)gridDim.x * kWarpsPerCta;
  double areg[2][4][2], anext[2][4][2];
  if (PREFETCH && gw < batch) load_a_frags(A + gw * kMat, g, t, anext);
  for (int64_t s = gw; s < batch; s += nw) {
    const double2* As = A + s * kMat;
    if (PREFETCH) {
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
          areg[nt][kb][0] = anext[nt][kb][0];
          areg[nt][kb][1] = anext[nt][kb][1];
        }
      if (s + nw < batch) load_a_frags(A + (s + nw) * kMat, g, t, anext);
    } else {
      load_a_frags(As, g, t, areg);
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

    ZAcc<M3> acc;
    if (!ns_mode) {
      // ---- Nested Neumann: `iters` nests of depth P (nest 0 from the diagonal X0) ----
      // Hermitian A (and so X0): the Horner products compute three of four tiles
      bool herm = false;
      if (iters > 0) first_nest_diag<P, M3>(acc, X, Pm, V, areg, g, t, M3 && herm_ok, &herm);
      MirrorState mst;
      float eps_pending = INFINITY;
      for (int it = 1; it < iters; ++it) {
        const SMat* v = &X;
        if constexpr (M3) {
          acc.template seed<true>(nullptr, 1.0, g, t);  // −I
          zmma_sr(acc, X, areg, g, t);                  // −I + X·A
          const uint32_t pss = epilogue_seeded<true>(acc, Pm, g, t);  // P = I − X·A
          // decide this nest from the previous nest's ε (its reduction is long done), then
          // start this nest's reduction — nothing waits on it until the next nest
          if (herm && it >= 2) herm = keep_mirrored<P>(eps_pending, mst, it - 1, it == iters - 1);
          eps_pending = p_size(pss);
#pragma unroll
          for (int j = 1; j <= P; ++j) {
            horner_step(acc, X, Pm, *v, (j == P) ? X : V, herm, g, t);  // X + P·V; the last lands in X
            v = &V;
          }
        } else {
          acc.zero();
          zmma_sr(acc, X, areg, g, t);                  // X·A
          epilogue(acc, -1.0, nullptr, 1.0, Pm, g, t);  // P = I − X·A
#pragma unroll
          for (int j = 1; j <= P; ++j) {
            acc.zero();
            zmma_ss(acc, Pm, *v, g, t);                 // P·V
            const SMat& dst = (j == P) ? X : V;         // last Horner step lands in X
            epilogue(acc, 1.0, &X, 0.0, dst, g, t);     // V = X + P·V
            v = &V;
          }
        }
      }
      // final residual eps = ‖I − X·A‖_F / √n
      acc.zero();
      zmma_sr(acc, X, areg, g, t);
      const double ss = warp_sum(residual_ss(acc, g, t));
      if (lane == 0 && eps_last) eps_last[s] = sqrt(ss) * 0.25;  // 1/sqrt(16)
    } else if (ns_order > 0) {
      // ---- Neumann-series baseline of `ns_order` terms from X0 (the same
      // diagonal-X0 shortcuts: P = I − X0·A and X = T·X0 are scalings) ----
      double2 xc[2];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) xc[nt] = make_double2(X.re[swz(8 * nt + g, 8 * nt + g)], X.im[swz(8 * nt + g, 8 * nt + g)]);
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {  // P = I − X0·A
          const int r = 4 * kb + t, c = 8 * nt + g, idx = swz(r, c);
          const double xr = X.re[swz(r, r)], xi = X.im[swz(r, r)];
          const double ar = areg[nt][kb][0], ai = areg[nt][kb][1];
          Pm.re[idx] = (r == c ? 1.0 : 0.0) - (xr * ar - xi * ai);
          Pm.im[idx] = -(xr * ai + xi * ar);
        }
      __syncwarp();
      for (int i = lane; i < kMat; i += 32) {      // T = I + P (into V)
        V.re[i] = Pm.re[i];
        V.im[i] = Pm.im[i];
      }
      __syncwarp();
      if (lane < kN) V.re[swz(lane, lane)] += 1.0;
      __syncwarp();
      for (int step = 2; step <= ns_order; ++step) {
        acc.zero();
        zmma_ss(acc, V, Pm, g, t);                  // T·P
        epilogue(acc, 1.0, nullptr, 1.0, V, g, t);  // T = T·P + I
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {  // X = T·X0: column c scaled by x_c
          const int r = 4 * kb + t, c = 8 * nt + g, idx = swz(r, c);
          const double tr = V.re[idx], ti = V.im[idx];
          X.re[idx] = tr * xc[nt].x - ti * xc[nt].y;
          X.im[idx] = tr * xc[nt].y + ti * xc[nt].x;
        }
      __syncwarp();
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

// ---------------------------------------------------------------------------
// Fused massive-MIMO detection (the step either side
// of the batched inversion; §4 motivates NN with mMIMO detection):
//   A = Hᴴ·H + σ²·I        (16×128 · 128×16, DMMA from coalesced H fragments)
//   z = Hᴴ·y               (accumulated from the same H fragments)
//   X = NN inverse of A    (Jacobi X0, `iters` nests of depth P, as above)
//   x̂ = X·z                (written per system; X and eps optional)
// H (32 KB per system) is read exactly once; A never touches HBM.
template <int P>
__global__ void __launch_bounds__(kThreads, NNB_BATCHED_MINB)
    mimo_detect_kernel(const double2* __restrict__ H, const double2* __restrict__ Y, int64_t batch, int ant,
                       double sigma2, int iters, double2* __restrict__ xhat, double2* __restrict__ Xout,
                       double* __restrict__ eps_last, int herm_ok) {
  constexpr bool M3 = true;
  __shared__ __align__(16) double smem[kWarpsPerCta][3][2][kMat];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  SMat X{smem[warp][0][0], smem[warp][0][1]};
  SMat Pm{smem[warp][1][0], smem[warp][1][1]};
  SMat V{smem[warp][2][0], smem[warp][2][1]};
  const int64_t gw = blockIdx.x * (int64_t)kWarpsPerCta + warp;
  const int64_t nw = (int64_t)gridDim.x * kWarpsPerCta;
  for (int64_t s = gw; s < batch; s += nw) {
    const double2* Hs = H + s * (int64_t)ant * kN;
    const double2* Ys = Y + s * (int64_t)ant;
    // ---- Gram A = Hᴴ·H and z = Hᴴ·y from one pass over H ----
    ZAcc<M3> acc;
    acc.zero();
    double zr[2] = {0.0, 0.0}, zi[2] = {0.0, 0.0};  // z[8mt+g], partial over this lane's antennas
#pragma unroll 4
    for (int kb = 0; kb < ant / 4; ++kb) {
      const int a = 4 * kb + t;
      const double2 h0 = __ldg(Hs + a * kN + g), h1 = __ldg(Hs + a * kN + 8 + g), y = __ldg(Ys + a);
      const double lr[2] = {h0.x, h1.x}, li[2] = {-h0.y, -h1.y};  // A-operand: conj(H)[i][a]
      const double rr[2] = {h0.x, h1.x}, ri[2] = {h0.y, h1.y};    // B-operand: H[a][j]
      acc.step_herm(lr, li, rr, ri);  // HᴴH is Hermitian: three of the four 8×8 tiles
      // conj(h)·y
      zr[0] = fma(h0.x, y.x, fma(h0.y, y.y, zr[0]));
      zi[0] = fma(h0.x, y.y, fma(-h0.y, y.x, zi[0]));
      zr[1] = fma(h1.x, y.x, fma(h1.y, y.y, zr[1]));
      zi[1] = fma(h1.x, y.y, fma(-h1.y, y.x, zi[1]));
    }
#pragma unroll
    for (int o = 1; o < 4; o <<= 1)  // sum the 4 antenna phases t (lanes with equal g)
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        zr[m] += __shfl_xor_sync(0xffffffffu, zr[m], o);
        zi[m] += __shfl_xor_sync(0xffffffffu, zi[m], o);
      }
    gram_epilogue(acc, sigma2, V, g, t);  // A = HᴴH + σ²I (shared, planar)
    // A's B-operand fragments in registers and X0 = diag(A)^-1
    double areg[2][4][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int kb = 0; kb < 4; ++kb) {
        const int idx = swz(4 * kb + t, 8 * nt + g);
        areg[nt][kb][0] = V.re[idx];
        areg[nt][kb][1] = V.im[idx];
      }
    for (int i = lane; i < kMat; i += 32) {
      X.re[i] = 0.0;
      X.im[i] = 0.0;
    }
    __syncwarp();
    if (lane < kN) {
      const double dr = V.re[swz(lane, lane)], di = V.im[swz(lane, lane)];
      double xr, xi;
      if (fabs(dr) >= fabs(di)) {
        const double r = di / dr, den = dr + di * r;
        xr = 1.0 / den;
        xi = -r / den;
      } else {
        const double r = dr / di, den = dr * r + di;
        xr = r / den;
        xi = -1.0 / den;
      }
      X.re[swz(lane, lane)] = xr;
      X.im[swz(lane, lane)] = xi;
    }
    __syncwarp();
    // ---- Nested Neumann inversion (seeded 3M products, nest 0 from the diagonal X0) ----
    // A = HᴴH + σ²I is Hermitian by construction (gram_epilogue mirrors it)
    bool herm = herm_ok != 0;
    if (iters > 0) first_nest_diag<P, true>(acc, X, Pm, V, areg, g, t, herm, nullptr);
    MirrorState mst;
    float eps_pending = INFINITY;
    for (int it = 1; it < iters; ++it) {
      acc.template seed<true>(nullptr, 1.0, g, t);
      zmma_sr(acc, X, areg, g, t);
      const uint32_t pss = epilogue_seeded<true>(acc, Pm, g, t);  // P = I − X·A
      if (herm && it >= 2) herm = keep_mirrored<P>(eps_pending, mst, it - 1, it == iters - 1);
      eps_pending = p_size(pss);
      const SMat* v = &X;
#pragma unroll
      for (int j = 1; j <= P; ++j) {
        horner_step(acc, X, Pm, *v, (j == P) ? X : V, herm, g, t);  // V = X + P·V
        v = &V;
      }
    }
    if (eps_last) {
      acc.zero();
      zmma_sr(acc, X, areg, g, t);
      const double ss = warp_sum(residual_ss(acc, g, t));
      if (lane == 0) eps_last[s] = sqrt(ss) * 0.25;
    }
    // ---- x̂ = X·z: two lanes per row, 8 columns each ----
    {
      const int row = lane & 15, half = lane >> 4;
      double sr = 0.0, si = 0.0;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const int j = 8 * half + jj;
        const double z0r = __shfl_sync(0xffffffffu, zr[0], 4 * jj), z1r = __shfl_sync(0xffffffffu, zr[1], 4 * jj);
        const double z0i = __shfl_sync(0xffffffffu, zi[0], 4 * jj), z1i = __shfl_sync(0xffffffffu, zi[1], 4 * jj);
        const double vr = half ? z1r : z0r, vi = half ? z1i : z0i;
        const double xr = X.re[swz(row, j)], xi = X.im[swz(row, j)];
        sr = fma(xr, vr, fma(-xi, vi, sr));
        si = fma(xr, vi, fma(xi, vr, si));
      }
      sr += __shfl_xor_sync(0xffffffffu, sr, 16);
      si += __shfl_xor_sync(0xffffffffu, si, 16);
      if (lane < kN) xhat[s * kN + lane] = make_double2(sr, si);
    }
    if (Xout) {
      double2* Xs = Xout + s * kMat;
#pragma unroll
      for (int q = 0; q < kMat / 32; ++q) {
        const int e = q * 32 + lane;
        const int idx = swz(e / kN, e % kN);
        Xs[e] = make_double2(X.re[idx], X.im[idx]);
      }
    }
    __syncwarp();
  }
}

// NNB_BATCHED_HERM=0: full products for Hermitian systems too (A/B measurement)
int herm_enabled() {
  static const int on = !(debug_env("NNB_BATCHED_HERM") && std::strcmp(debug_env("NNB_BATCHED_HERM"), "0") == 0);
  return on;
}

template <int P, bool M3, bool PF>
int launch_variant(const double2* a, int64_t batch, int iters, int ns_order, double2* x, double* eps,
                   int ns_mode, cudaStream_t s) {
  static int blocks_per_sm = 0;
  static int sms = 0;
  if (!blocks_per_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, batched_z16_kernel<P, M3, PF>, kThreads, 0);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  const int64_t want = (batch + kWarpsPerCta - 1) / kWarpsPerCta;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(want, (int64_t)sms * blocks_per_sm));
  batched_z16_kernel<P, M3, PF><<<grid, kThreads, 0, s>>>(a, batch, iters, ns_order, x, eps, ns_mode, herm_enabled());
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}

// Product method: 3M (default, 25 % fewer DMMA) or 4M; register prefetch of the
// next A off by default (measured on B200: 3M 3.16-3.21 ms, 3M+prefetch 3.26-3.29,
// 4M 3.45, 4M+prefetch 3.47-3.57 ms per 262144-system batch).
// NNB_BATCHED_VARIANT = "4m", "3m", "4m_nopf", "3m_nopf" overrides (A/B measurement).
template <int P>
int launch_p(const double2* a, int64_t batch, int iters, int ns_order, double2* x, double* eps, int ns_mode,
             cudaStream_t s) {
  static const char* env = debug_env("NNB_BATCHED_VARIANT");
  const bool m4 = env && env[0] == '4';
  const bool nopf = !env || std::strstr(env, "nopf");
  if (m4) {
    return nopf ? launch_variant<P, false, false>(a, batch, iters, ns_order, x, eps, ns_mode, s)
                : launch_variant<P, false, true>(a, batch, iters, ns_order, x, eps, ns_mode, s);
  }
  return nopf ? launch_variant<P, true, false>(a, batch, iters, ns_order, x, eps, ns_mode, s)
              : launch_variant<P, true, true>(a, batch, iters, ns_order, x, eps, ns_mode, s);
}

template <int P>
int launch_mimo(const double2* h, const double2* y, int64_t batch, int ant, double sigma2, int iters,
                double2* xhat, double2* X, double* eps, cudaStream_t s) {
  static int blocks_per_sm = 0, sms = 0;
  if (!blocks_per_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, mimo_detect_kernel<P>, kThreads, 0);
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  const int64_t want = (batch + kWarpsPerCta - 1) / kWarpsPerCta;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(want, (int64_t)sms * blocks_per_sm));
  mimo_detect_kernel<P><<<grid, kThreads, 0, s>>>(h, y, batch, ant, sigma2, iters, xhat, X, eps, herm_enabled());
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace

int mimo_detect_z16(const double* H, const double* y, int64_t batch, int antennas, double sigma2, int p, int iters,
                    double* xhat, double* X, double* eps_last, cudaStream_t s) {
  if (batch <= 0) return 0;
  const double2* h = reinterpret_cast<const double2*>(H);
  const double2* yy = reinterpret_cast<const double2*>(y);
  double2* xh = reinterpret_cast<double2*>(xhat);
  double2* x = reinterpret_cast<double2*>(X);
  switch (p) {
    case 1: return launch_mimo<1>(h, yy, batch, antennas, sigma2, iters, xh, x, eps_last, s);
    case 2: return launch_mimo<2>(h, yy, batch, antennas, sigma2, iters, xh, x, eps_last, s);
    case 3: return launch_mimo<3>(h, yy, batch, antennas, sigma2, iters, xh, x, eps_last, s);
    case 4: return launch_mimo<4>(h, yy, batch, antennas, sigma2, iters, xh, x, eps_last, s);
    default: return fail(2, "mimo detect: depth p must be in 1..4");
  }
}

int batched_nn_z16(const double* A, int64_t batch, int p, int iters, int ns_order, double* X,
                   double* eps_last, cudaStream_t s) {
  if (batch <= 0) return 0;
  // ns_order < 0: Nested Neumann chain; ns_order >= 0: Neumann series of that order
  const int ns_mode = ns_order >= 0 ? 1 : 0;
  const double2* a = reinterpret_cast<const double2*>(A);
  double2* x = reinterpret_cast<double2*>(X);
  switch (ns_mode ? 1 : p) {
    case 1: return launch_p<1>(a, batch, iters, ns_order, x, eps_last, ns_mode, s);
    case 2: return launch_p<2>(a, batch, iters, ns_order, x, eps_last, ns_mode, s);
    case 3: return launch_p<3>(a, batch, iters, ns_order, x, eps_last, ns_mode, s);
    case 4: return launch_p<4>(a, batch, iters, ns_order, x, eps_last, ns_mode, s);
    default: return fail(2, "batched: depth p must be in 1..4");
  }
}

}  // namespace nnb
