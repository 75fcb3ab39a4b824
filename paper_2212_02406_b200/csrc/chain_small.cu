// Device-resident Nested Neumann chain for small N (config 0, N = 256).
//
// The launch-per-product chain (chain.cu) pays ≈11 µs per N=256 product: a
// launch, 16 TMA round trips of a 16-k-step ring and the last-CTA ε
// reduction, for 34 MFLOP that the DMMA pipes finish in ≈1 µs.  Here the
// whole `nn_invert` loop (proj/src/solver.cpp:138-159: residual ε, stop test,
// nn_step) runs inside ONE cooperative kernel:
//
//  * every product C = α·(L·Rm) + β·D + γ·I is split into TM×16 output tiles
//    (TM = 32 while the tiles fit one per SM, else 16); a CTA pulls its TM×K
//    row panel of L and K×16 column panel of Rm (plus the D tile) with TMA
//    from L2 (the working set is < 3 MB of the 126 MB L2), in 64-k chunks
//    with one mbarrier each; A's row panel stays resident in shared memory
//    when every CTA owns one tile; its 8 warps split K (k-steps w, w+8, …) on
//    DMMA.8x8x4 and the 8 partial tiles are summed in fixed warp order;
//  * products are separated by a grid barrier (gpu-scope release/acquire
//    counter); the next product's loads are issued right after it, before any
//    ε bookkeeping;
//  * Σ C² and the non-finite count go to per-(product, tile) partials.  In
//    tolerance mode every CTA sums the residual's partials in the same fixed
//    order right after its barrier and takes the same stop decision; all ε /
//    non-finite slots are summed once at the end.  No host round trip.
//
// Control flow is run_chain()'s (chain.cu): the same products, the same ε /
// non-finite slots, the same stop rules and iteration counts; the K-split
// changes only FP64 rounding, inside the 1e-10 parity bar.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "engine.cuh"

namespace nnb {
namespace {

constexpr int kT = 16;          // output tile columns
constexpr int kWarps = 8;       // K-split warps per CTA
constexpr int kThreads = kWarps * 32;
constexpr int kBoxK = 64;       // k rows per column-panel TMA box
constexpr int kBufs = 5;
constexpr int kMaxChunks = 8;   // n <= 512        // 0 = A, 1 = X (caller), 2/3 = Horner scratch, 4 = R

struct SmallMaps {
  CUtensorMap row[kBufs];  // row-panel boxes: 16 (k) × TM (rows), 128B swizzle
  CUtensorMap col[kBufs];  // column-panel boxes: 16 (n) × 64 (k), 128B swizzle
};

struct SmallArgs {
  double* ptr[kBufs];
  int n;
  int64_t ld;
  int p, max_iters, final_residual, order, tol_mode;
  double tol, eps_scale;
  double* eps_dev;  // [max_iters + 1]
  int* nf_dev;      // [(max_iters + 1)·(p + 1)]
  double* ss_part;  // [2][tiles]
  int* nf_part;     // [2][tiles]
  unsigned* bar;    // grid barrier counter (zero at launch)
  int* status;      // k, products, stopped, recorded
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// All CTAs are co-resident (cooperative launch); the counter only grows.  The
// bar.sync orders the CTA's C stores before thread 0's gpu-scope release; the
// acquiring CTAs' TMA reads of them follow a fence.proxy.async.global in issue().
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& epoch) {
  __syncthreads();
  ++epoch;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    const unsigned target = epoch * gridDim.x;
    while (ld_acquire(bar) < target) {
    }
  }
  __syncthreads();
}

struct Totals {
  double ss;
  int nf;
};

// One product of the chain: C = α·(L·Rm) + β·D + γ·I on buffers by index
// (db < 0: no D term).
struct Op {
  int li, ri, db, cb;
  double alpha, beta, gamma;
};

template <int TM>
__global__ void __launch_bounds__(kThreads) small_chain_kernel(const __grid_constant__ SmallMaps maps, SmallArgs a) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  __shared__ double wss[kWarps];
  __shared__ int wnf[kWarps];
  __shared__ Totals tot_s;
  __shared__ __align__(8) uint64_t full[kMaxChunks];  // one per 64-k chunk: MMAs start as chunk 0 lands
  constexpr int MI = TM / 8;

  const int n = a.n;
  const int64_t ld = a.ld;
  const int tiles_m = (n + TM - 1) / TM, tiles_n = (n + kT - 1) / kT;
  const int tiles = tiles_m * tiles_n;
  const int kp = (n + kBoxK - 1) / kBoxK * kBoxK;
  uint8_t* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);  // stays a shared-window pointer
  // panels (1024-B aligned for the 128B swizzle): L rows, resident A rows, Rm columns, the D tile
  uint8_t* As = sm;                  // kp/16 boxes of TM×128 B (at least kWarps·TM·16 doubles: `red`)
  uint8_t* Ares = As + TM * (kp > 128 ? kp : 128) * 8;  // A's row panel, loaded once when every CTA owns one tile
  uint8_t* Bs = Ares + TM * kp * 8;  // kp/64 boxes of 64×128 B
  uint8_t* Ds = Bs + kp * 128;       // TM×128 B
  double* red = reinterpret_cast<double*>(As);  // [kWarps][TM×16], after the MMA loop
  const bool resident = gridDim.x == (unsigned)tiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  unsigned epoch = 0;
  uint32_t phase = 0;
  bool a_loaded = false;  // tracked identically by every thread
  const int chunks = kp / kBoxK;
  if (threadIdx.x == 0) {
    for (int c = 0; c < chunks; ++c) mbar_init(&full[c], 1);
    fence_barrier_init();
    for (int b = 0; b < kBufs; ++b) {
      tma_prefetch_desc(&maps.row[b]);
      tma_prefetch_desc(&maps.col[b]);
    }
  }
  __syncthreads();

  auto use_res = [&](const Op& op) { return resident && op.li == 0; };
  // one thread: the TMA loads of `op`'s tile
  auto issue = [&](const Op& op, int tile) {
    const int m0 = (tile / tiles_n) * TM, n0 = (tile % tiles_n) * kT;
    asm volatile("fence.proxy.async.global;" ::: "memory");
    fence_proxy_async_smem();  // earlier generic accesses of the panels before the refill
    const bool res = use_res(op);
    const bool load_l = !res || !a_loaded;
    uint8_t* ldst = res ? Ares : As;
    for (int c = 0; c < chunks; ++c) {
      const bool d = c == 0 && op.db >= 0;  // the D tile rides with chunk 0
      mbar_arrive_expect_tx(&full[c], (load_l ? TM * kBoxK * 8 : 0) + kBoxK * 128 + (d ? TM * 128 : 0));
      if (load_l)
        for (int kb = 4 * c; kb < 4 * c + 4; ++kb)
          tma_load_2d(ldst + kb * (TM * 128), &maps.row[op.li], &full[c], kb * 16, m0);
      tma_load_2d(Bs + c * (kBoxK * 128), &maps.col[op.ri], &full[c], n0, c * kBoxK);
      if (d) tma_load_2d(Ds, &maps.row[op.db], &full[c], n0, m0);
    }
  };

  // All tiles of `op` (the first tile's loads already issued), then the grid barrier.
  auto run = [&](const Op& op, int q) {
    double* ssp = a.ss_part + (int64_t)q * tiles;
    int* nfp = a.nf_part + (int64_t)q * tiles;
    double* C = a.ptr[op.cb];
    const uint8_t* Lp = use_res(op) ? Ares : As;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
      const int m0 = (tile / tiles_n) * TM, n0 = (tile % tiles_n) * kT;
      if (tile != (int)blockIdx.x && threadIdx.x == 0) issue(op, tile);
      double acc[MI][2][2] = {};
      for (int s = warp; s < kp / 4; s += kWarps) {
        if ((s & 15) == warp) mbar_wait(&full[s >> 4], phase);  // first k-step of a chunk
        const int k0 = s * 4;
        const int k = k0 + t;
        const uint8_t* ab = Lp + (k0 >> 4) * (TM * 128);
        const uint32_t achunk = ((((k & 15) >> 1) ^ g) << 4) | ((k & 1) << 3);
        const uint8_t* bb = Bs + (k >> 6) * (kBoxK * 128) + (k & 63) * 128 + ((g & 1) << 3);
        double af[MI];
#pragma unroll
        for (int i = 0; i < MI; ++i) af[i] = *reinterpret_cast<const double*>(ab + (i * 8 + g) * 128 + achunk);
        const double b0 = *reinterpret_cast<const double*>(bb + (((g >> 1) ^ (k & 7)) << 4));
        const double b1 = *reinterpret_cast<const double*>(bb + ((((8 + g) >> 1) ^ (k & 7)) << 4));
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          dmma_8x8x4(acc[i][0][0], acc[i][0][1], af[i], b0);
          dmma_8x8x4(acc[i][1][0], acc[i][1][1], af[i], b1);
        }
      }
      phase ^= 1;
      __syncthreads();  // panel reads done before `red` overwrites As
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          double* q = red + warp * (TM * kT) + (i * 8 + g) * kT + j * 8 + 2 * t;
          q[0] = acc[i][j][0];
          q[1] = acc[i][j][1];
        }
      __syncthreads();

      // output elements: fixed warp order, then the fused epilogue
      double ss = 0.0;
      int nf = 0;
#pragma unroll
      for (int q = 0; q < TM * kT / kThreads; ++q) {
        const int e = q * kThreads + threadIdx.x;
        const int r = e / kT, c = e % kT;
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) v += red[w * (TM * kT) + e];
        const int gr = m0 + r, gc = n0 + c;
        if (gr < n && gc < n) {
          v = op.alpha * v;
          if (op.db >= 0)
            v = fma(op.beta, *reinterpret_cast<const double*>(Ds + r * 128 + ((((c >> 1) ^ (r & 7))) << 4) + ((c & 1) << 3)),
                    v);
          if (gr == gc) v += op.gamma;
          C[(int64_t)gr * ld + gc] = v;
          ss = fma(v, v, ss);
          nf += !isfinite(v);
        }
      }
      ss = warp_sum(ss);
      nf = warp_sum_i(nf);
      if (lane == 0) {
        wss[warp] = ss;
        wnf[warp] = nf;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double ts = 0.0;
        int tn = 0;
        for (int w = 0; w < kWarps; ++w) {
          ts += wss[w];
          tn += wnf[w];
        }
        ssp[tile] = ts;
        nfp[tile] = tn;
      }
    }
    if (use_res(op)) a_loaded = true;
    grid_barrier(a.bar, epoch);
  };

  // run_chain()'s loop (chain.cu) as a schedule of products, decided identically in
  // every CTA.  The next product's loads go out before the ε / non-finite totals of
  // the current one are read (a residual's successor is speculative: if the stop
  // test fires, its loads are drained and it is not run).
  const int p = a.p;
  auto residual_op = [&](int xi) {
    const int xb = 1 + xi;
    return a.order == 0 ? Op{0, xb, -1, 4, -1.0, 0.0, 1.0} : Op{xb, 0, -1, 4, -1.0, 0.0, 1.0};
  };
  auto horner_op = [&](int xi, int vi, int dst_i) {
    return a.order == 0 ? Op{1 + vi, 4, 1 + xi, 1 + dst_i, 1.0, 1.0, 0.0}
                        : Op{4, 1 + vi, 1 + xi, 1 + dst_i, 1.0, 1.0, 0.0};
  };
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  int k = 0, j = 0, xi = 0, vi = 0, dst_i = 1, products = 0, stopped = 1, recorded = 0;
  if (a.max_iters > 0 || a.final_residual) {
    Op cur = residual_op(xi);
    if (threadIdx.x == 0) issue(cur, blockIdx.x);
    for (;;) {
      run(cur, products);
      // the successor (k, j) -> (nk, nj) and its operands
      bool has_next = true;
      int nk = k, nj = j + 1, nxi = xi, nvi = vi, ndst = dst_i;
      if (j == 0) {
        if (k >= a.max_iters) {
          has_next = false;
        } else if (p > 0) {
          nvi = xi;
          ndst = (xi + 1) % 3;
        } else {
          nk = k + 1;
          nj = 0;
          has_next = nk < a.max_iters || a.final_residual;
        }
      } else {
        nvi = dst_i;
        ndst = 3 - xi - nvi;
        if (j == p) {
          nxi = nvi;
          nk = k + 1;
          nj = 0;
          has_next = nk < a.max_iters || a.final_residual;
        }
      }
      const Op next = nj == 0 ? residual_op(nxi) : horner_op(nxi, nvi, ndst);
      if (has_next && threadIdx.x == 32) issue(next, blockIdx.x);
      // tolerance mode: the residual's ε and non-finite count now, in every CTA (a
      // non-finite Horner product always makes the next residual non-finite)
      Totals tot{0.0, 0};
      if (a.tol_mode && j == 0) {
        if (warp == 0) {
          const double* ssp = a.ss_part + (int64_t)products * tiles;
          const int* nfp = a.nf_part + (int64_t)products * tiles;
          double s2 = 0.0;
          int f = 0;
          for (int i = lane; i < tiles; i += 32) {
            s2 += __ldcg(ssp + i);
            f += __ldcg(nfp + i);
          }
          s2 = warp_sum(s2);
          f = warp_sum_i(f);
          if (lane == 0) tot_s = Totals{s2, f};
        }
        __syncthreads();
        tot = tot_s;
        __syncthreads();
      }
      ++products;
      bool stop = false;
      if (j == 0) {
        recorded = k + 1;
        if (a.tol_mode && (tot.nf != 0 || sqrt(tot.ss) * a.eps_scale < a.tol)) {
          if (tot.nf == 0) stopped = 0;
          stop = true;
        }
      }
      if (stop || !has_next) {
        if (stop && has_next) {  // drain the speculative loads
          for (int c = 0; c < chunks; ++c) mbar_wait(&full[c], phase);
          phase ^= 1;
        }
        if (!stop && !(j == 0 && k >= a.max_iters)) k = nk;  // as run_chain's ++k before its exit test
        xi = nxi;  // a completed nest's X_{k+1}
        break;
      }
      k = nk;
      j = nj;
      xi = nxi;
      vi = nvi;
      dst_i = ndst;
      cur = next;
    }
  }
  // the final iterate into the caller's buffer (every product ended in a barrier)
  if (xi != 0) {
    const double* src = a.ptr[1 + xi];
    double* dst = a.ptr[1];
    const int64_t total = (int64_t)n * n;
    for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < total; e += (int64_t)gridDim.x * kThreads) {
      const int64_t r = e / n, c = e % n;
      dst[r * ld + c] = __ldcg(src + r * ld + c);
    }
  }
  // every product's ε / non-finite slots (product q = nest·(p+1) + j), fixed order
  for (int q = blockIdx.x * kWarps + warp; q < products; q += gridDim.x * kWarps) {
    {
      const double* ssp = a.ss_part + (int64_t)q * tiles;
      const int* nfp = a.nf_part + (int64_t)q * tiles;
      double s2 = 0.0;
      int f = 0;
      for (int i = lane; i < tiles; i += 32) {
        s2 += __ldcg(ssp + i);
        f += __ldcg(nfp + i);
      }
      s2 = warp_sum(s2);
      f = warp_sum_i(f);
      if (lane == 0) {
        if (q % (p + 1) == 0) a.eps_dev[q / (p + 1)] = sqrt(s2) * a.eps_scale;
        a.nf_dev[q] = f;
      }
    }
  }
  if (lead) {
    a.status[0] = k;
    a.status[1] = products;
    a.status[2] = stopped;
    a.status[3] = recorded;
  }
}

template <int TM>
size_t smem_bytes(int n) {
  const int kp = (n + kBoxK - 1) / kBoxK * kBoxK;
  return 1024 + (size_t)TM * ((kp > 128 ? kp : 128) + kp) * 8 + (size_t)kp * 128 + (size_t)TM * 128;
}

template <int TM>
int launch(const SmallMaps& maps, SmallArgs& a, cudaStream_t s) {
  const size_t smem = smem_bytes<TM>(a.n);
  NNB_TRY(ensure_smem<small_chain_kernel<TM>>(static_cast<int>(smem)));
  int per_sm = 0, dev = 0, sms = 0;
  NNB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, small_chain_kernel<TM>, kThreads, smem));
  NNB_CUDA(cudaGetDevice(&dev));
  NNB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (per_sm < 1) return fail(1, "small chain: kernel does not fit on an SM");
  const int tiles = ((a.n + TM - 1) / TM) * ((a.n + kT - 1) / kT);
  const int grid = tiles < per_sm * sms ? tiles : per_sm * sms;
  void* params[] = {const_cast<SmallMaps*>(&maps), &a};
  NNB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(small_chain_kernel<TM>), dim3(grid), dim3(kThreads),
                                       params, smem, s));
  count_launch();
  return 0;
}

}  // namespace

int small_chain_max_n() {
  static const int v = debug_env("NNB_SMALL_CHAIN_MAX") ? std::atoi(debug_env("NNB_SMALL_CHAIN_MAX")) : 384;
  return v;
}

bool small_chain_eligible(int64_t n, int64_t ld, const ChainCfg& cfg) {
  if (n < 1 || n > 512 || n > small_chain_max_n() || (ld & 1) || cfg.max_iters < 0 || cfg.p < 0) return false;
  const int64_t tiles = ((n + 15) / 16) * ((n + 15) / 16);  // the larger (TM = 16) tiling
  return (int64_t)(cfg.max_iters + 1) * (cfg.p + 1) * tiles * 12 <= (int64_t(64) << 20);
}

static int small_tm(int64_t n) {
  static const char* force = debug_env("NNB_SMALL_TM");
  const bool fits32 = smem_bytes<32>(static_cast<int>(n)) <= 227 * 1024;
  if (force) return std::atoi(force) == 32 && fits32 ? 32 : 16;
  const int64_t t32 = ((n + 31) / 32) * ((n + 15) / 16);
  return t32 <= 148 && fits32 ? 32 : 16;  // 32-row tiles while they still fit one per SM
}

int small_chain_real(const double* A, double* X, double* R, double* w1, double* w2, int64_t n, int64_t ld,
                     const ChainCfg& cfg, double* eps_dev, int* nf_dev, int* status_dev, cudaStream_t s) {
  if (n < 1 || n > 512 || (ld & 1)) return fail(1, "small chain: unsupported size");
  const int tm = small_tm(n);
  const int tiles = static_cast<int>(((n + tm - 1) / tm) * ((n + kT - 1) / kT));
  const int64_t slots = (int64_t)(cfg.max_iters + 1) * (cfg.p + 1);  // products of the longest run
  DevBuf ws;
  NNB_TRY(ws.alloc((sizeof(double) + sizeof(int)) * slots * tiles + sizeof(int) * 8, s));
  SmallArgs a{};
  a.ptr[0] = const_cast<double*>(A);
  a.ptr[1] = X;
  a.ptr[2] = w1;
  a.ptr[3] = w2;
  a.ptr[4] = R;
  SmallMaps maps;
  for (int b = 0; b < kBufs; ++b) {
    NNB_TRY(make_tmap(&maps.row[b], a.ptr[b], n, n, ld, tm, 16, true));
    NNB_TRY(make_tmap(&maps.col[b], a.ptr[b], n, n, ld, kBoxK, 16, true));
  }
  a.n = static_cast<int>(n);
  a.ld = ld;
  a.p = cfg.p;
  a.max_iters = cfg.max_iters;
  a.final_residual = cfg.final_residual;
  a.order = cfg.order == 1 ? 1 : 0;  // SYMMETRIC runs the NORTHSTAR order with full products here
  a.tol_mode = cfg.tol > 0.0;
  a.tol = cfg.tol;
  a.eps_scale = 1.0 / std::sqrt(static_cast<double>(n));
  a.eps_dev = eps_dev;
  a.nf_dev = nf_dev;
  a.ss_part = ws.as<double>();
  a.nf_part = reinterpret_cast<int*>(a.ss_part + slots * tiles);
  a.bar = reinterpret_cast<unsigned*>(a.nf_part + slots * tiles);
  a.status = status_dev;
  NNB_CUDA(cudaMemsetAsync(a.bar, 0, sizeof(unsigned), s));
  if (tm == 32)
    NNB_TRY(launch<32>(maps, a, s));
  else
    NNB_TRY(launch<16>(maps, a, s));
  return 0;
}

}  // namespace nnb
