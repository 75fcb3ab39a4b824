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
// Measured on B200 (config 4): 14.2 ms per solve = 91 % of HBM; a row-group
// variant with coalesced shared staging (20.1 ms) and an 8-way unrolled
// per-row variant (19.2 ms) lost to the occupancy of this 40-register loop.
// Row offsets are narrowed to int32 on the device when nnz < 2^31.
// HBM-bound: 12 B per nonzero + 4 B per row of CSR, 8 B in + 8 B out per row.
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
template <typename Idx, int MODE>
__global__ void __launch_bounds__(256)
    spmv_rows_kernel(const Idx* __restrict__ rp, const int32_t* __restrict__ col, const double* __restrict__ val,
                     int64_t r_begin, int64_t r_end, int64_t k, const double* __restrict__ t_ext,
                     const double* __restrict__ t_own, double* __restrict__ out, const double* __restrict__ zold,
                     double theta, int* __restrict__ flag) {
  bool bad = false;
  for (int64_t r = r_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r_end;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = rp[r], e1 = rp[r + 1];
    for (int64_t c = 0; c < k; ++c) {
      double y = 0.0;
      for (int64_t e = e0; e < e1; ++e) y = __dadd_rn(y, __dmul_rn(val[e], t_ext[(int64_t)col[e] * k + c]));
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

namespace {

unsigned rows_grid(int64_t n) {
  const int64_t want = (n + 255) / 256;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, 148 * 8 * 4)));
}

template <typename Idx, int MODE>
unsigned resident_grid(int64_t rows) {
  static unsigned resident = 0;
  if (!resident) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, spmv_rows_kernel<Idx, MODE>, 256, 0);
    resident = static_cast<unsigned>(sms * std::max(1, per));
  }
  return std::min<unsigned>(resident, rows_grid(rows));
}

}  // namespace

template <typename Idx>
void spmv_apply(const SpmvOp<Idx>& op, int mode, int64_t r_begin, int64_t r_end, cudaStream_t s) {
  if (r_end <= r_begin) return;
  const int64_t rows = r_end - r_begin;
  switch (mode) {
    case kInner:
      spmv_rows_kernel<Idx, kInner><<<resident_grid<Idx, kInner>(rows), 256, 0, s>>>(
          op.rp, op.col, op.val, r_begin, r_end, op.k, op.t_ext, op.t_own, op.out, op.zold, op.theta, op.flag);
      break;
    case kFactorEnd:
      spmv_rows_kernel<Idx, kFactorEnd><<<resident_grid<Idx, kFactorEnd>(rows), 256, 0, s>>>(
          op.rp, op.col, op.val, r_begin, r_end, op.k, op.t_ext, op.t_own, op.out, op.zold, op.theta, op.flag);
      break;
    default:
      spmv_rows_kernel<Idx, kFinal><<<resident_grid<Idx, kFinal>(rows), 256, 0, s>>>(
          op.rp, op.col, op.val, r_begin, r_end, op.k, op.t_ext, op.t_own, op.out, op.zold, op.theta, op.flag);
  }
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
void run_factors(const Idx* rp, const int32_t* col, const double* val, int64_t n, const double* B, int64_t k,
                 int s_factors, double theta, double* X, double* z[2], double* tb[2], int* flags, cudaStream_t s) {
  const double* zcur = B;  // Z = B (read in place, never written)
  int zi = 0;
  int64_t reps = 1;
  for (int f = 0; f < s_factors; ++f) {
    const double* tin = zcur;  // t = Z
    int ti = 0;
    for (int64_t r = 0; r < reps; ++r) {
      SpmvOp<Idx> op{rp, col, val, k, tin, tin, nullptr, zcur, theta, flags + f};
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
  NNB_TRY(work.alloc(sizeof(double) * vec * 4 + sizeof(int) * 64 + (narrow ? sizeof(int32_t) * (n + 1) + 16 : 0), s));
  double* z[2] = {work.as<double>(), work.as<double>() + vec};
  double* tb[2] = {z[1] + vec, z[1] + 2 * vec};
  int* flags = reinterpret_cast<int*>(tb[1] + vec);
  NNB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * 64, s));
  if (narrow) {
    int32_t* rp32 = flags + 64;
    NNB_TRY(narrow_offsets(row_ptr, rp32, n + 1, 0, s));
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
