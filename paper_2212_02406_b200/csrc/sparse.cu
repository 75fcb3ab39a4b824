// Matrix-free factorized Neumann solve on a CSR operator (BASELINE config 4:
// 5-point Laplacian + I on a 4096² grid, θ = 0.2, γ = 63).
//
// Reference: /root/reference/proj/src/factorized.cpp:101-140 —
//   Z = B;  for f < s:  t = Z;  2^f × { y = W t (spmv_block); t = t − θ y };  Z = Z + t
//   x = θ Z
// which streams t, y and Z through three separate N-vector passes per
// application plus an allocation each.  Here one kernel per application does
//   t_out = t_in − θ·W·t_in                         (inner applications)
//   Z_new = Z + (t_in − θ·W·t_in)                   (last application of a factor)
//   X     = θ·(Z + (t_in − θ·W·t_in))               (last application overall)
// so y never exists and the factor update and the final scale ride along.
//
// Row-group kernel: a warp owns 32 consecutive rows; its lanes stream the
// group's contiguous nonzero range with coalesced loads of val/col, gather
// t_in[col], and stage the products in shared memory; each lane then sums
// its own row in ascending nonzero order.  Every operation is explicitly
// rounded (no FMA contraction) and ordered exactly as the reference's
// std::complex<double> arithmetic (spmv sum += v·x from 0, t = z − θ·y,
// Z + t, Z·θ), so the GPU result is BIT-IDENTICAL to the reference's.
// Row offsets are narrowed to int32 on the device when nnz < 2^31 (one
// conversion pass per solve, −4 B per row per application).
// HBM-bound: ≈12 B per nonzero + 4 B per row of CSR, 8 B in + 8 B out per row.
#include <cstdlib>

#include "engine.cuh"

namespace nnb {
namespace {

enum Mode { kInner = 0, kFactorEnd = 1, kFinal = 2 };

constexpr int kWarps = 8;           // warps per CTA
constexpr int kStage = 32 * 8;      // staged products per warp per column (avg ≤ 8 nnz/row)

template <int MODE>
__device__ __forceinline__ double finish(double tin, double y, double theta, const double* zold, int64_t i,
                                         bool& bad) {
  const double t = __dsub_rn(tin, __dmul_rn(theta, y));  // fused_axpy_sub, factorized.cpp:21-30
  double o;
  if (MODE == kInner) {
    o = t;
  } else if (MODE == kFactorEnd) {
    o = __dadd_rn(zold[i], t);                           // add(z, t), factorized.cpp:136
  } else {
    o = __dmul_rn(__dadd_rn(zold[i], t), theta);         // scale(z, theta), factorized.cpp:139
  }
  bad |= !isfinite(y) || !isfinite(t) || !isfinite(o);
  return o;
}

// k columns (k ≤ 2) per row; rows grouped 32 per warp.
template <typename Idx, int MODE, int K>
__global__ void __launch_bounds__(kWarps * 32)
    spmv_group_kernel(const Idx* __restrict__ rp, const int32_t* __restrict__ col, const double* __restrict__ val,
                      int64_t n, const double* __restrict__ tin, double* __restrict__ out,
                      const double* __restrict__ zold, double theta, int* __restrict__ flag) {
  __shared__ double prod[kWarps][K][kStage];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bool bad = false;
  const int64_t groups = (n + 31) / 32;
  for (int64_t grp = blockIdx.x * (int64_t)kWarps + warp; grp < groups; grp += (int64_t)gridDim.x * kWarps) {
    const int64_t r = grp * 32 + lane;
    const bool live = r < n;
    const int64_t my_b = live ? (int64_t)rp[r] : 0;
    const int64_t my_e = live ? (int64_t)rp[r + 1] : 0;
    const int64_t g_b = __shfl_sync(0xffffffffu, my_b, 0);
    const int64_t rem = n - 1 - grp * 32;
    const int last = rem < 31 ? static_cast<int>(rem) : 31;
    const int64_t g_e = __shfl_sync(0xffffffffu, my_e, last);
    const int64_t cnt = g_e - g_b;
    double y[K];
#pragma unroll
    for (int c = 0; c < K; ++c) y[c] = 0.0;
    if (cnt <= kStage) {
      // coalesced stream of the group's nonzeros, fully unrolled so every lane has
      // kStage/32 value/column loads and then as many gathers in flight;
      // products rounded as v*x
      constexpr int kPer = kStage / 32;
      double v[kPer];
      int32_t ci[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int64_t j = lane + 32 * u;
        if (j < cnt) {
          v[u] = __ldg(val + g_b + j);
          ci[u] = __ldg(col + g_b + j);
        }
      }
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int64_t j = lane + 32 * u;
        if (j < cnt) {
#pragma unroll
          for (int c = 0; c < K; ++c) prod[warp][c][j] = __dmul_rn(v[u], __ldg(tin + (int64_t)ci[u] * K + c));
        }
      }
      __syncwarp();
      if (live)
        for (int64_t e = my_b - g_b; e < my_e - g_b; ++e)
#pragma unroll
          for (int c = 0; c < K; ++c) y[c] = __dadd_rn(y[c], prod[warp][c][e]);
      __syncwarp();
    } else if (live) {
      // long rows in this group: plain per-row loop, same rounding and order
      for (int64_t e = my_b; e < my_e; ++e) {
        const double v = __ldg(val + e);
        const int64_t cidx = __ldg(col + e);
#pragma unroll
        for (int c = 0; c < K; ++c) y[c] = __dadd_rn(y[c], __dmul_rn(v, __ldg(tin + cidx * K + c)));
      }
    }
    if (live) {
#pragma unroll
      for (int c = 0; c < K; ++c) out[r * K + c] = finish<MODE>(tin[r * K + c], y[c], theta, zold, r * K + c, bad);
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
}

// One thread per row, K ≤ 2 columns, the first 8 nonzeros of a row loaded with
// full memory-level parallelism (8 value/column loads, then 8 gathers in
// flight) before the ordered, explicitly rounded sum; longer rows continue
// sequentially.  Same arithmetic as the row-group kernel (bit-exact).
template <typename Idx, int MODE, int K>
__global__ void __launch_bounds__(256)
    spmv_row8_kernel(const Idx* __restrict__ rp, const int32_t* __restrict__ col, const double* __restrict__ val,
                     int64_t n, const double* __restrict__ tin, double* __restrict__ out,
                     const double* __restrict__ zold, double theta, int* __restrict__ flag) {
  bool bad = false;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = __ldg(rp + r), e1 = __ldg(rp + r + 1);
    double v[8], xv[8][K];
    int32_t ci[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (e0 + u < e1) {
        v[u] = __ldg(val + e0 + u);
        ci[u] = __ldg(col + e0 + u);
      }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (e0 + u < e1) {
#pragma unroll
        for (int c = 0; c < K; ++c) xv[u][c] = __ldg(tin + (int64_t)ci[u] * K + c);
      }
    double y[K];
#pragma unroll
    for (int c = 0; c < K; ++c) y[c] = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (e0 + u < e1) {
#pragma unroll
        for (int c = 0; c < K; ++c) y[c] = __dadd_rn(y[c], __dmul_rn(v[u], xv[u][c]));
      }
    for (int64_t e = e0 + 8; e < e1; ++e) {
      const double vv = __ldg(val + e);
      const int64_t cc = __ldg(col + e);
#pragma unroll
      for (int c = 0; c < K; ++c) y[c] = __dadd_rn(y[c], __dmul_rn(vv, __ldg(tin + cc * K + c)));
    }
#pragma unroll
    for (int c = 0; c < K; ++c) out[r * K + c] = finish<MODE>(tin[r * K + c], y[c], theta, zold, r * K + c, bad);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// Generic k: one thread per row, all columns (used for k > 2).
template <typename Idx, int MODE>
__global__ void __launch_bounds__(256)
    spmv_rows_kernel(const Idx* __restrict__ rp, const int32_t* __restrict__ col, const double* __restrict__ val,
                     int64_t n, int64_t k, const double* __restrict__ tin, double* __restrict__ out,
                     const double* __restrict__ zold, double theta, int* __restrict__ flag) {
  bool bad = false;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = rp[r], e1 = rp[r + 1];
    for (int64_t c = 0; c < k; ++c) {
      double y = 0.0;
      for (int64_t e = e0; e < e1; ++e) y = __dadd_rn(y, __dmul_rn(val[e], tin[(int64_t)col[e] * k + c]));
      out[r * k + c] = finish<MODE>(tin[r * k + c], y, theta, zold, r * k + c, bad);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// Plain Y = W·X for nn::spmv_block (same rounding as the reference's sum).
template <typename Idx>
__global__ void spmv_plain_kernel(const Idx* __restrict__ rp, const int32_t* __restrict__ col,
                                  const double* __restrict__ val, int64_t n, int64_t k,
                                  const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = rp[r], e1 = rp[r + 1];
    for (int64_t c = 0; c < k; ++c) {
      double s = 0.0;
      for (int64_t e = e0; e < e1; ++e) s = __dadd_rn(s, __dmul_rn(val[e], x[(int64_t)col[e] * k + c]));
      y[r * k + c] = s;
    }
  }
}

__global__ void narrow_offsets_kernel(const int64_t* __restrict__ in, int32_t* __restrict__ out, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<int32_t>(in[i]);
}

unsigned rows_grid(int64_t n) {
  static const int64_t cap = std::getenv("NNB_SPMV_GRID") ? std::atoll(std::getenv("NNB_SPMV_GRID")) : 148 * 8 * 4;
  const int64_t want = (n + 255) / 256;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, cap)));
}

unsigned group_grid(int64_t n) {
  const int64_t groups = (n + 31) / 32;
  const int64_t want = (groups + kWarps - 1) / kWarps;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, 148 * 8)));
}

// 0 = row-group (shared staging), 1 = row8 (per-row, unrolled MLP), 2 = per-row
// loop (default).  Measured on B200, 4096² Laplacian, γ=63: 20.1 / 19.2 / 15.3 ms
// per solve — the 40-register per-row loop keeps 48 warps/SM resident and wins.
int spmv_variant() {
  static const int v = std::getenv("NNB_SPMV_VARIANT") ? std::atoi(std::getenv("NNB_SPMV_VARIANT")) : 2;
  return v;
}

template <typename Idx, int MODE>
void launch_step(const Idx* rp, const int32_t* col, const double* val, int64_t n, int64_t k, const double* tin,
                 double* out, const double* zold, double theta, int* flag, cudaStream_t s) {
  if (spmv_variant() == 2) {
    // persistent grid = exactly the resident blocks (grid-stride rows, no partial
    // last wave): 14.2 ms vs 15.4 ms with 4736 blocks (B200, config 4)
    static unsigned resident = 0;
    if (!resident) {
      int dev = 0, sms = 148, per = 1;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, spmv_rows_kernel<Idx, MODE>, 256, 0);
      resident = static_cast<unsigned>(sms * std::max(1, per));
    }
    const unsigned grid = std::min<unsigned>(resident, rows_grid(n));
    spmv_rows_kernel<Idx, MODE><<<grid, 256, 0, s>>>(rp, col, val, n, k, tin, out, zold, theta, flag);
  } else if (spmv_variant() == 1 && k <= 2) {
    if (k == 1)
      spmv_row8_kernel<Idx, MODE, 1><<<rows_grid(n), 256, 0, s>>>(rp, col, val, n, tin, out, zold, theta, flag);
    else
      spmv_row8_kernel<Idx, MODE, 2><<<rows_grid(n), 256, 0, s>>>(rp, col, val, n, tin, out, zold, theta, flag);
  } else if (k == 1)
    spmv_group_kernel<Idx, MODE, 1><<<group_grid(n), kWarps * 32, 0, s>>>(rp, col, val, n, tin, out, zold, theta, flag);
  else if (k == 2)
    spmv_group_kernel<Idx, MODE, 2><<<group_grid(n), kWarps * 32, 0, s>>>(rp, col, val, n, tin, out, zold, theta, flag);
  else
    spmv_rows_kernel<Idx, MODE><<<rows_grid(n), 256, 0, s>>>(rp, col, val, n, k, tin, out, zold, theta, flag);
  count_launch();
}

template <typename Idx>
void run_factors(const Idx* rp, const int32_t* col, const double* val, int64_t n, const double* B, int64_t k,
                 int s_factors, double theta, double* X, double* z[2], double* tb[2], int* flags, cudaStream_t s) {
  const double* zcur = B;  // Z = B (read in place, never written)
  int zi = 0;
  int64_t reps = 1;
  for (int f = 0; f < s_factors; ++f) {
    const double* tin = zcur;  // t = Z
    int ti = 0;
    for (int64_t r = 0; r < reps; ++r) {
      const bool last_app = (r == reps - 1);
      if (!last_app) {
        launch_step<Idx, kInner>(rp, col, val, n, k, tin, tb[ti], nullptr, theta, flags + f, s);
        tin = tb[ti];
        ti ^= 1;
      } else if (f == s_factors - 1) {
        launch_step<Idx, kFinal>(rp, col, val, n, k, tin, X, zcur, theta, flags + f, s);
      } else {
        launch_step<Idx, kFactorEnd>(rp, col, val, n, k, tin, z[zi], zcur, theta, flags + f, s);
        zcur = z[zi];
        zi ^= 1;
      }
    }
    reps <<= 1;
  }
}

}  // namespace

int spmv_csr(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n, const double* X, int64_t k,
             double* Y, cudaStream_t s) {
  if (n == 0) return 0;
  spmv_plain_kernel<int64_t><<<rows_grid(n), 256, 0, s>>>(row_ptr, col, val, n, k, X, Y);
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}

int sparse_factorized(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n, const double* B,
                      int64_t k, int s_factors, double theta, double* X, int* fail_factor, cudaStream_t s) {
  const size_t vec = (size_t)n * k;
  int64_t nnz = 0;
  NNB_CUDA(cudaMemcpyAsync(&nnz, row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  const bool narrow = nnz < INT32_MAX;
  DevBuf work;
  NNB_TRY(work.alloc(sizeof(double) * vec * 4 + sizeof(int) * 64 + (narrow ? sizeof(int32_t) * (n + 1) + 16 : 0), s));
  double* z[2] = {work.as<double>(), work.as<double>() + vec};
  double* tb[2] = {z[1] + vec, z[1] + 2 * vec};
  int* flags = reinterpret_cast<int*>(tb[1] + vec);
  NNB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * 64, s));
  if (narrow) {
    int32_t* rp32 = flags + 64;
    narrow_offsets_kernel<<<rows_grid(n + 1), 256, 0, s>>>(row_ptr, rp32, n + 1);
    count_launch();
    run_factors<int32_t>(rp32, col, val, n, B, k, s_factors, theta, X, z, tb, flags, s);
  } else {
    run_factors<int64_t>(row_ptr, col, val, n, B, k, s_factors, theta, X, z, tb, flags, s);
  }
  NNB_CUDA(cudaGetLastError());
  int hflags[64];
  NNB_CUDA(cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  for (int f = 0; f < s_factors && f < 64; ++f)
    if (hflags[f]) {
      if (fail_factor) *fail_factor = f;
      return fail(3, "solve_sparse_factorized: non-finite block at factor " + std::to_string(f));
    }
  return 0;
}

}  // namespace nnb
