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
// Every operation is explicitly rounded (no FMA contraction) and ordered as
// the reference's std::complex<double> arithmetic evaluates it for real W:
// spmv sum += v·x from 0 in ascending nonzero order, t = z − θ·y, Z + t, Z·θ.
// The GPU result is therefore BIT-IDENTICAL to the reference's, for any row
// partition (the multi-GPU path, sparse_sharded.cu, relies on this).
//
// Kernel: one thread per row, persistent grid of exactly the resident blocks.
// A row-group variant with coalesced shared staging (20.1 ms), an 8-way
// unrolled per-row variant (19.2 ms) and sliced ELL (17.0 ms; less
// memory-level parallelism than CSR order) all lost to this loop.
// One pass per solve (compact_csr) narrows the row offsets to int32 and, for
// banded operators, the columns to int16 deltas from the row.
// HBM-bound: 10 (int16) or 12 (int32 columns) B per nonzero + 4 B per row of
// CSR, 8 B in + 8 B out per row.  The register cap (32, for 64 resident warps
// per SM) buys the memory-level parallelism: 13.0 vs 13.7 ms per C5 solve at
// 48 warps; 1024-thread blocks shave another 1.6 % (12.8 ms).
#include <cstdlib>
#include <cstring>

#include "engine.cuh"
#include "sparse.cuh"

namespace nnb {

template <int MODE>
__device__ __forceinline__ double finish(double tin, double y, double theta, double zold, bool& bad) {
  const double t = __dsub_rn(tin, __dmul_rn(theta, y));  // fused_axpy_sub, factorized.cpp:21-30
  double o;
  if (MODE == kInner) {
    o = t;
  } else if (MODE == kFactorEnd) {
    o = __dadd_rn(zold, t);                              // add(z, t), factorized.cpp:136
  } else {
    o = __dmul_rn(__dadd_rn(zold, t), theta);            // scale(z, theta), factorized.cpp:139
  }
  bad |= !isfinite(y) || !isfinite(t) || !isfinite(o);
  return o;
}

// Rows [r_begin, r_end) of one application.  Gathers read t_ext through the
// (possibly halo-remapped) column indices; the diagonal term, z and the
// output are indexed by row.
// NNB_SPMV_THREADS per block; NNB_SPMV_MINB resident blocks per SM the register budget must allow.
#ifndef NNB_SPMV_THREADS
#define NNB_SPMV_THREADS 1024
#endif
#ifndef NNB_SPMV_MINB
#define NNB_SPMV_MINB (2048 / NNB_SPMV_THREADS)
#endif
template <typename Idx, typename C, int MODE>
__global__ void __launch_bounds__(NNB_SPMV_THREADS, NNB_SPMV_MINB)
    spmv_rows_kernel(const Idx* __restrict__ rp, const C* __restrict__ col, const double* __restrict__ val,
                     int64_t r_begin, int64_t r_end, int64_t diag_off, int64_t k, const double* __restrict__ t_ext,
                     const double* __restrict__ t_own, double* __restrict__ out, const double* __restrict__ zold,
                     double theta, int* __restrict__ flag) {
  bool bad = false;
  for (int64_t r = r_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r_end;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = rp[r], e1 = rp[r + 1];
    const int64_t g0 = sizeof(C) == 2 ? r + diag_off : 0;  // int16: column = row + delta
    for (int64_t c = 0; c < k; ++c) {
      double y = 0.0;
      for (int64_t e = e0; e < e1; ++e) y = __dadd_rn(y, __dmul_rn(val[e], t_ext[(g0 + col[e]) * k + c]));
      out[r * k + c] = finish<MODE>(t_own[r * k + c], y, theta, MODE == kInner ? 0.0 : zold[r * k + c], bad);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// Plain Y = W·X for nn::spmv_block (same rounding as the reference's sum).
__global__ void spmv_plain_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
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

__global__ void narrow_offsets_kernel(const int64_t* __restrict__ in, int32_t* __restrict__ out, int64_t count,
                                      int64_t base) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = static_cast<int32_t>(in[i] - base);
}

__global__ void compact_csr_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t rows,
                                   int64_t row0, int32_t* __restrict__ rp32, int16_t* __restrict__ col16,
                                   int* __restrict__ wide) {
  const int64_t base = rp[0];
  bool far = false;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= rows; r += (int64_t)gridDim.x * blockDim.x) {
    rp32[r] = static_cast<int32_t>(rp[r] - base);
    if (r == rows) continue;
    for (int64_t e = rp[r], e1 = rp[r + 1]; e < e1; ++e) {
      const int64_t d = (int64_t)col[e] - (row0 + r);
      far |= d < -32767 || d > 32767;
      col16[e - base] = static_cast<int16_t>(d);
    }
  }
  if (far) atomicOr(wide, 1);  // rare: only operators wider than the int16 band
}

namespace {

unsigned rows_grid(int64_t n) {
  const int64_t want = (n + 255) / 256;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, 148 * 8 * 4)));
}

template <typename Idx, typename C, int MODE>
unsigned resident_grid(int64_t rows) {
  static unsigned resident = 0;
  if (!resident) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, spmv_rows_kernel<Idx, C, MODE>, NNB_SPMV_THREADS, 0);
    resident = static_cast<unsigned>(sms * std::max(1, per));
  }
  const int64_t want = (rows + NNB_SPMV_THREADS - 1) / NNB_SPMV_THREADS;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(resident, want)));
}

template <typename Idx, typename C, int MODE>
void launch_rows(const SpmvOp<Idx>& op, const C* col, int64_t r_begin, int64_t r_end, cudaStream_t s) {
  spmv_rows_kernel<Idx, C, MODE><<<resident_grid<Idx, C, MODE>(r_end - r_begin), NNB_SPMV_THREADS, 0, s>>>(
      op.rp, col, op.val, r_begin, r_end, op.diag_off, op.k, op.t_ext, op.t_own, op.out, op.zold, op.theta, op.flag);
}

template <typename Idx, typename C>
void launch_mode(const SpmvOp<Idx>& op, const C* col, int mode, int64_t r_begin, int64_t r_end, cudaStream_t s) {
  switch (mode) {
    case kInner: launch_rows<Idx, C, kInner>(op, col, r_begin, r_end, s); break;
    case kFactorEnd: launch_rows<Idx, C, kFactorEnd>(op, col, r_begin, r_end, s); break;
    default: launch_rows<Idx, C, kFinal>(op, col, r_begin, r_end, s);
  }
}

}  // namespace

template <typename Idx>
void spmv_apply(const SpmvOp<Idx>& op, int mode, int64_t r_begin, int64_t r_end, cudaStream_t s) {
  if (r_end <= r_begin) return;
  if (op.col16) launch_mode(op, op.col16, mode, r_begin, r_end, s);
  else launch_mode(op, op.col, mode, r_begin, r_end, s);
  count_launch();
}
template void spmv_apply<int32_t>(const SpmvOp<int32_t>&, int, int64_t, int64_t, cudaStream_t);
template void spmv_apply<int64_t>(const SpmvOp<int64_t>&, int, int64_t, int64_t, cudaStream_t);

int narrow_offsets(const int64_t* in, int32_t* out, int64_t count, int64_t base, cudaStream_t s) {
  narrow_offsets_kernel<<<rows_grid(count), 256, 0, s>>>(in, out, count, base);
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}

int compact_csr(const int64_t* rp, const int32_t* col, int64_t rows, int64_t row0, int32_t* rp32, int16_t* col16,
                bool* fits, cudaStream_t s) {
  DevBuf flag;
  NNB_TRY(flag.alloc(sizeof(int), s));
  NNB_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
  compact_csr_kernel<<<rows_grid(rows + 1), 256, 0, s>>>(rp, col, rows, row0, rp32, col16, flag.as<int>());
  count_launch();
  NNB_CUDA(cudaGetLastError());
  int wide = 0;
  NNB_CUDA(cudaMemcpyAsync(&wide, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  *fits = !wide;
  return 0;
}

int spmv_csr(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n, const double* X, int64_t k,
             double* Y, cudaStream_t s) {
  if (n == 0) return 0;
  spmv_plain_kernel<<<rows_grid(n), 256, 0, s>>>(row_ptr, col, val, n, k, X, Y);
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}

namespace {

template <typename Idx>
void run_factors(const Idx* rp, const int32_t* col, const int16_t* col16, const double* val, int64_t n,
                 const double* B, int64_t k, int s_factors, double theta, double* X, double* z[2], double* tb[2],
                 int* flags, cudaStream_t s) {
  const double* zcur = B;  // Z = B (read in place, never written)
  int zi = 0;
  int64_t reps = 1;
  for (int f = 0; f < s_factors; ++f) {
    const double* tin = zcur;  // t = Z
    int ti = 0;
    for (int64_t r = 0; r < reps; ++r) {
      SpmvOp<Idx> op{rp, col, col16, 0, val, k, tin, tin, nullptr, zcur, theta, flags + f};
      int mode;
      if (r < reps - 1) {
        mode = kInner;
        op.out = tb[ti];
      } else if (f == s_factors - 1) {
        mode = kFinal;
        op.out = X;
      } else {
        mode = kFactorEnd;
        op.out = z[zi];
      }
      spmv_apply(op, mode, 0, n, s);
      if (mode == kInner) {
        tin = tb[ti];
        ti ^= 1;
      } else if (mode == kFactorEnd) {
        zcur = z[zi];
        zi ^= 1;
      }
    }
    reps <<= 1;
  }
}

}  // namespace

int sparse_factorized(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n, const double* B,
                      int64_t k, int s_factors, double theta, double* X, int* fail_factor, cudaStream_t s) {
  const size_t vec = (size_t)n * k;
  int64_t nnz = 0;
  NNB_CUDA(cudaMemcpyAsync(&nnz, row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  const bool narrow = nnz < INT32_MAX;
  DevBuf work;
  NNB_TRY(work.alloc(sizeof(double) * vec * 4 + sizeof(int) * 64 +
                         (narrow ? sizeof(int32_t) * (n + 1) + sizeof(int16_t) * nnz + 32 : 0),
                     s));
  double* z[2] = {work.as<double>(), work.as<double>() + vec};
  double* tb[2] = {z[1] + vec, z[1] + 2 * vec};
  int* flags = reinterpret_cast<int*>(tb[1] + vec);
  NNB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * 64, s));
  if (narrow) {
    // int32 offsets, and int16 column deltas when the operator's band allows
    int32_t* rp32 = flags + 64;
    int16_t* col16 = reinterpret_cast<int16_t*>(rp32 + n + 2);
    bool fits = false;
    NNB_TRY(compact_csr(row_ptr, col, n, 0, rp32, col16, &fits, s));
    static const bool force32 = [] {  // NNB_SPARSE_COL=32: int32 columns (A/B measurement)
      const char* e = std::getenv("NNB_SPARSE_COL");
      return e && std::strcmp(e, "32") == 0;
    }();
    fits = fits && !force32;
    run_factors<int32_t>(rp32, col, fits ? col16 : nullptr, val, n, B, k, s_factors, theta, X, z, tb, flags, s);
  } else {
    run_factors<int64_t>(row_ptr, col, nullptr, val, n, B, k, s_factors, theta, X, z, tb, flags, s);
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
