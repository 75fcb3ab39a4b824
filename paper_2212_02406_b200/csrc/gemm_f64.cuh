// FP64 DMMA GEMM with the Nested Neumann epilogues fused in.
//
//   C = alpha * (A·B) + beta * D + gamma * I_shifted        (row-major, FP64)
//
// plus, optionally, a deterministic Σ C² / non-finite count over the whole
// output (per-tile partials, then the last CTA to finish sums them in fixed
// tile order — no floating-point atomics, so eps is bit-reproducible run to
// run).  One kernel therefore covers every dense product of the chain:
//   R = I − A·X      alpha=-1, gamma=1, Σ‖R‖² → eps   (residual + first product)
//   V = X + V·R      alpha= 1, beta=1, D=X           (Horner step of X·S(R))
//   P = I − X·A, V = X + P·V                          (reference operand order)
// replacing the reference's matmul + identity_minus + plus_identity +
// frobenius_norm passes (/root/reference/proj/src/kernels.cpp:137-242,
// /root/reference/proj/src/solver.cpp:27-36,72-75,93-103): no separate
// elementwise or norm kernel touches HBM.
//
// Structure (sm_100a): one TMA producer warp streams BMxBK tiles of A
// (128B-swizzled) and BKxBN tiles of B (linear) into a STAGES-deep shared
// ring guarded by full/empty mbarriers; WM×WN consumer warps run
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) out of shared memory with the
// accumulators in registers; the epilogue runs from registers.
#pragma once

#include "common.cuh"

namespace nnb {

struct GemmEpilogue {
  double alpha = 1.0;
  double beta = 0.0;
  const double* D = nullptr;  // may alias C (read-before-write per element)
  int64_t ldd = 0;
  double gamma = 0.0;         // added where (row + diag_offset) == col
  int64_t diag_offset = 0;
  double* C = nullptr;
  int64_t ldc = 0;
  // optional second output from the same product P (3M complex products):
  // C2 = alpha2·P + beta2·D2 (D2 may alias C2); the Σ C² reduction then covers
  // both outputs
  double* C2 = nullptr;
  int64_t ldc2 = 0;
  const double* D2 = nullptr;
  int64_t ldd2 = 0;
  double alpha2 = 0.0, beta2 = 0.0;
  // symmetric output (square C, no C2, D symmetric and not aliasing C,
  // diag_offset 0): only tiles tm <= tn are computed and only their r <= c
  // elements stored, each with its mirror (counted twice in the Σ C² /
  // non-finite reduction).  Valid when A·B is symmetric in exact arithmetic
  // for the operands given — e.g. X·(I − A·X)^j for symmetric X and A, by
  // push-through (DESIGN.md §3 K1-K3).
  int sym = 0;
  // accumulator seed (nullable, may alias C): the K loop starts from acc_in's
  // tile instead of 0.  A product split along K into launches whose non-final
  // parts store the raw accumulator (alpha 1, beta 0, gamma 0) then runs the
  // same DMMA sequence as one launch, bit for bit.
  const double* acc_in = nullptr;
  int64_t ld_acc_in = 0;
  // Σ C² / non-finite reduction (all nullable => skipped)
  double* ss_partial = nullptr;  // [num_tiles]
  int* nf_partial = nullptr;     // [num_tiles]
  unsigned* tile_counter = nullptr;  // zero on entry, reset to zero by the last CTA
  double* ss_out = nullptr;      // Σ C²
  int* nf_out = nullptr;         // Σ non-finite
  double* eps_out = nullptr;     // sqrt(Σ C²) * eps_scale
  double eps_scale = 1.0;
};

// B_KMAJOR: the B operand is supplied transposed (Bᵀ, N×K row-major) and its
// tiles are 128B-swizzled like A's, which makes the B-fragment loads
// conflict-free (2 wavefronts instead of 4 per 32 doubles).
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool B_KMAJOR = false>
struct GemmCfg {
  static constexpr bool kBKMajor = B_KMAJOR;
  static constexpr int kBM = BM, kBN = BN, kBK = BK, kWM = WM, kWN = WN, kStages = STAGES;
  static constexpr int kConsumerWarps = WM * WN;
  static constexpr int kThreads = (kConsumerWarps + 1) * 32;
  static constexpr int kWarpM = BM / WM, kWarpN = BN / WN;
  static constexpr int kMI = kWarpM / 8, kNI = kWarpN / 8;
  static constexpr int kABytes = BM * BK * 8, kBBytes = BK * BN * 8;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kSmemBytes = STAGES * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(BK == 16, "A tile rows are one 128-byte swizzle row");
  static_assert(kWarpM % 8 == 0 && kWarpN % 8 == 0, "warp tile must be a multiple of 8x8");
  static_assert(kABytes % 1024 == 0 && kBBytes % 1024 == 0, "stages must stay 1024B aligned");
};

template <class Cfg>
__global__ void __launch_bounds__(Cfg::kThreads, 1)
    gemm_f64_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    int M, int N, int K, GemmEpilogue ep) {
  constexpr int BM = Cfg::kBM, BN = Cfg::kBN, BK = Cfg::kBK, STAGES = Cfg::kStages;
  constexpr int MI = Cfg::kMI, NI = Cfg::kNI, NCW = Cfg::kConsumerWarps;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty = full + STAGES;
  double* red = reinterpret_cast<double*>(empty + STAGES);  // [NCW]
  int* redi = reinterpret_cast<int*>(red + NCW);            // [NCW]
  int* last_flag = redi + NCW;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // grouped raster: GROUP_M tile-rows sweep the tile-columns together (L2 reuse)
  constexpr int GROUP_M = 8;
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const int pid = blockIdx.x;
  int tm, tn;
  if (!ep.sym) {
    const int group = pid / (GROUP_M * tiles_n);
    const int first_m = group * GROUP_M;
    const int gsz = min(tiles_m - first_m, GROUP_M);
    tm = first_m + (pid % gsz);
    tn = (pid % (GROUP_M * tiles_n)) / gsz;
  } else {
    // upper-triangular tiles, same grouping: a group of gsz tile-rows starting
    // at f owns a gsz-row triangle (column-major) then a gsz-row rectangle
    int f = 0, rem = pid, gsz = min(tiles_m, GROUP_M);
    for (;;) {
      gsz = min(tiles_m - f, GROUP_M);
      const int cnt = gsz * (gsz + 1) / 2 + gsz * (tiles_n - f - gsz);
      if (rem < cnt) break;
      rem -= cnt;
      f += gsz;
    }
    const int tri = gsz * (gsz + 1) / 2;
    if (rem < tri) {
      int c = 0;
      while (rem >= c + 1) rem -= ++c;
      tn = f + c;
      tm = f + rem;
    } else {
      rem -= tri;
      tn = f + gsz + rem / gsz;
      tm = f + rem % gsz;
    }
  }
  const int m0 = tm * BM, n0 = tn * BN;
  const int KT = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == NCW) {
    // ===== TMA producer (one elected lane) =====
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        const uint32_t ph = (kt / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * Cfg::kStageBytes;
        uint8_t* sb = sa + Cfg::kABytes;
        mbar_arrive_expect_tx(&full[s], Cfg::kStageBytes);
        tma_load_2d(sa, &tmA, &full[s], kt * BK, m0);
        if (Cfg::kBKMajor)
          tma_load_2d(sb, &tmB, &full[s], kt * BK, n0);
        else
          tma_load_2d(sb, &tmB, &full[s], n0, kt * BK);
      }
    }
    return;
  }

  // ===== DMMA consumers =====
  const int wm = warp / Cfg::kWN, wn = warp % Cfg::kWN;
  const int g = lane >> 2, t = lane & 3;
  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (ep.acc_in) {
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int r = m0 + wm * Cfg::kWarpM + i * 8 + g;
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int c = n0 + wn * Cfg::kWarpN + j * 8 + 2 * t;
        if (r < M && c < N) {
          const double* ap = ep.acc_in + (int64_t)r * ep.ld_acc_in + c;
          acc[i][j][0] = ap[0];
          if (c + 1 < N) acc[i][j][1] = ap[1];
        }
      }
    }
  }

  // Per-thread fragment byte offsets inside a stage.
  // A (128B swizzle): (r,k) -> r*128 + ((k>>1) ^ (r&7))*16 + (k&1)*8, r&7 == g.
  // B (linear):       (k,n) -> (k*BN + n)*8.
  const uint32_t a_row_off = (wm * Cfg::kWarpM + g) * 128;
  // B (K-major, swizzled as A): (n,k) -> n*128 + ((k>>1) ^ (n&7))*16 + (k&1)*8.
  const uint32_t b_col_off = Cfg::kBKMajor ? (wn * Cfg::kWarpN + g) * 128 : (wn * Cfg::kWarpN + g) * 8 + t * BN * 8;

  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % STAGES;
    const uint32_t ph = (kt / STAGES) & 1;
    mbar_wait(&full[s], ph);
    const uint8_t* sa = smem + s * Cfg::kStageBytes;
    const uint8_t* sb = sa + Cfg::kABytes;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double af[MI], bf[NI];
      const uint32_t a_chunk = (((kk * 2 + (t >> 1)) ^ g) << 4) | ((t & 1) << 3);
#pragma unroll
      for (int i = 0; i < MI; ++i)
        af[i] = *reinterpret_cast<const double*>(sa + a_row_off + i * 8 * 128 + a_chunk);
#pragma unroll
      for (int j = 0; j < NI; ++j)
        bf[j] = Cfg::kBKMajor ? *reinterpret_cast<const double*>(sb + b_col_off + j * 8 * 128 + a_chunk)
                              : *reinterpret_cast<const double*>(sb + b_col_off + kk * 4 * BN * 8 + j * 64);
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    fence_proxy_async_smem();  // fragment reads of stage s complete before the TMA refill
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // ===== fused epilogue from registers =====
  double ss = 0.0;
  int nf = 0;
  const bool want_red = ep.ss_partial != nullptr;
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int r = m0 + wm * Cfg::kWarpM + i * 8 + g;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const int c = n0 + wn * Cfg::kWarpN + j * 8 + 2 * t;
      if (c >= N) continue;
      const bool two = (c + 1) < N;
      double v0 = ep.alpha * acc[i][j][0];
      double v1 = ep.alpha * acc[i][j][1];
      if (ep.D) {
        const double* dp = ep.D + (int64_t)r * ep.ldd + c;
        if (two) {
          const double2 d = *reinterpret_cast<const double2*>(dp);
          v0 = fma(ep.beta, d.x, v0);
          v1 = fma(ep.beta, d.y, v1);
        } else {
          v0 = fma(ep.beta, dp[0], v0);
        }
      }
      const int64_t dr = (int64_t)r + ep.diag_offset;
      if (dr == c) v0 += ep.gamma;
      if (dr == c + 1) v1 += ep.gamma;
      if (ep.sym) {
        // upper triangle (r <= c) stored with its mirror, so C is symmetric bit
        // for bit; r > c inside a diagonal tile belongs to (c, r)'s thread
        auto put = [&](int cc, double v) {
          if (r > cc) return;
          ep.C[(int64_t)r * ep.ldc + cc] = v;
          if (r < cc) ep.C[(int64_t)cc * ep.ldc + r] = v;
          if (want_red) {
            const double w = r < cc ? 2.0 : 1.0;
            ss = fma(w * v, v, ss);
            nf += (r < cc ? 2 : 1) * !isfinite(v);
          }
        };
        put(c, v0);
        if (two) put(c + 1, v1);
        continue;
      }
      double* cp = ep.C + (int64_t)r * ep.ldc + c;
      if (two) {
        *reinterpret_cast<double2*>(cp) = make_double2(v0, v1);
      } else {
        cp[0] = v0;
      }
      if (want_red) {
        ss = fma(v0, v0, ss);
        nf += !isfinite(v0);
        if (two) {
          ss = fma(v1, v1, ss);
          nf += !isfinite(v1);
        }
      }
      if (ep.C2) {
        double w0 = ep.alpha2 * acc[i][j][0];
        double w1 = ep.alpha2 * acc[i][j][1];
        if (ep.D2) {
          const double* dp = ep.D2 + (int64_t)r * ep.ldd2 + c;
          if (two) {
            const double2 d = *reinterpret_cast<const double2*>(dp);
            w0 = fma(ep.beta2, d.x, w0);
            w1 = fma(ep.beta2, d.y, w1);
          } else {
            w0 = fma(ep.beta2, dp[0], w0);
          }
        }
        double* cp2 = ep.C2 + (int64_t)r * ep.ldc2 + c;
        if (two) {
          *reinterpret_cast<double2*>(cp2) = make_double2(w0, w1);
        } else {
          cp2[0] = w0;
        }
        if (want_red) {
          ss = fma(w0, w0, ss);
          nf += !isfinite(w0);
          if (two) {
            ss = fma(w1, w1, ss);
            nf += !isfinite(w1);
          }
        }
      }
    }
  }
  if (!want_red) return;

  // deterministic tile reduction: fixed shuffle tree, fixed warp order
  ss = warp_sum(ss);
  nf = warp_sum_i(nf);
  if (lane == 0) {
    red[warp] = ss;
    redi[warp] = nf;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32));
  const int ntiles = gridDim.x;
  if (threadIdx.x == 0) {
    double tss = 0.0;
    int tnf = 0;
    for (int w = 0; w < NCW; ++w) {
      tss += red[w];
      tnf += redi[w];
    }
    ep.ss_partial[pid] = tss;
    ep.nf_partial[pid] = tnf;
    __threadfence();
    const unsigned done = atomicAdd(ep.tile_counter, 1u);
    *last_flag = (done == (unsigned)(ntiles - 1));
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32));
  if (!*last_flag) return;

  // last CTA: sum all tile partials in a fixed order
  __threadfence();
  double s2 = 0.0;
  int n2 = 0;
  for (int k = threadIdx.x; k < ntiles; k += NCW * 32) {
    s2 += __ldcg(ep.ss_partial + k);
    n2 += __ldcg(ep.nf_partial + k);
  }
  s2 = warp_sum(s2);
  n2 = warp_sum_i(n2);
  asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32));
  if (lane == 0) {
    red[warp] = s2;
    redi[warp] = n2;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32));
  if (threadIdx.x == 0) {
    double tot = 0.0;
    int ntot = 0;
    for (int w = 0; w < NCW; ++w) {
      tot += red[w];
      ntot += redi[w];
    }
    if (ep.ss_out) *ep.ss_out = tot;
    if (ep.nf_out) *ep.nf_out = ntot;
    if (ep.eps_out) *ep.eps_out = sqrt(tot) * ep.eps_scale;
    *ep.tile_counter = 0u;
  }
}

}  // namespace nnb
