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
// so y never exists, the factor update and the final scale ride along with the
// last application, and each application is one HBM pass over the CSR arrays
// (HBM-bound: ≈12 B per nonzero + 8 B per row in, 8 B per row out).
// Non-finite results raise a per-factor flag (integer atomics only).
#include "engine.cuh"

namespace nnb {
namespace {

enum Mode { kInner = 0, kFactorEnd = 1, kFinal = 2 };

template <typename Idx, int MODE>
__global__ void __launch_bounds__(256)
    spmv_step_kernel(const Idx* __restrict__ row_ptr, const int32_t* __restrict__ col,
                     const double* __restrict__ val, int64_t n, int64_t k,
                     const double* __restrict__ tin, double* __restrict__ out,
                     const double* __restrict__ zold, double theta, int* __restrict__ flag) {
  bool bad = false;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const Idx e0 = __ldg(row_ptr + r), e1 = __ldg(row_ptr + r + 1);
    for (int64_t c = 0; c < k; ++c) {
      double y = 0.0;  // ascending-nonzero order, like spmv_block (kernels.cpp:459-467)
      for (Idx e = e0; e < e1; ++e) y = fma(__ldg(val + e), __ldg(tin + (int64_t)__ldg(col + e) * k + c), y);
      const double t = tin[r * k + c] - theta * y;
      double o;
      if (MODE == kInner) {
        o = t;
      } else if (MODE == kFactorEnd) {
        o = zold[r * k + c] + t;
      } else {
        o = (zold[r * k + c] + t) * theta;
      }
      bad |= !isfinite(t) || !isfinite(o);
      out[r * k + c] = o;
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

template <typename Idx>
__global__ void spmv_plain_kernel(const Idx* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                  const double* __restrict__ val, int64_t n, int64_t k,
                                  const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const Idx e0 = row_ptr[r], e1 = row_ptr[r + 1];
    for (int64_t c = 0; c < k; ++c) {
      double s = 0.0;
      for (Idx e = e0; e < e1; ++e) s = fma(val[e], x[(int64_t)col[e] * k + c], s);
      y[r * k + c] = s;
    }
  }
}

unsigned rows_grid(int64_t n) {
  const int64_t want = (n + 255) / 256;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, 148 * 8 * 4)));
}

template <int MODE>
void launch_step(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n,
                 int64_t k, const double* tin, double* out, const double* zold, double theta,
                 int* flag, cudaStream_t s) {
  spmv_step_kernel<int64_t, MODE><<<rows_grid(n), 256, 0, s>>>(row_ptr, col, val, n, k, tin, out,
                                                                zold, theta, flag);
  count_launch();
}

}  // namespace

int spmv_csr(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n,
             const double* X, int64_t k, double* Y, cudaStream_t s) {
  if (n == 0) return 0;
  spmv_plain_kernel<int64_t><<<rows_grid(n), 256, 0, s>>>(row_ptr, col, val, n, k, X, Y);
  count_launch();
  NNB_CUDA(cudaGetLastError());
  return 0;
}

int sparse_factorized(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n,
                      const double* B, int64_t k, int s_factors, double theta, double* X,
                      int* fail_factor, cudaStream_t s) {
  const size_t vec = (size_t)n * k;
  DevBuf work;
  NNB_TRY(work.alloc(sizeof(double) * vec * 4 + sizeof(int) * 64, s));
  double* z[2] = {work.as<double>(), work.as<double>() + vec};
  double* tb[2] = {z[1] + vec, z[1] + 2 * vec};
  int* flags = reinterpret_cast<int*>(tb[1] + vec);
  NNB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * 64, s));

  const double* zcur = B;  // Z = B (read in place, never written)
  int zi = 0;
  int64_t reps = 1;
  for (int f = 0; f < s_factors; ++f) {
    const double* tin = zcur;  // t = Z
    int ti = 0;
    for (int64_t r = 0; r < reps; ++r) {
      const bool last_app = (r == reps - 1);
      if (!last_app) {
        launch_step<kInner>(row_ptr, col, val, n, k, tin, tb[ti], nullptr, theta, flags + f, s);
        tin = tb[ti];
        ti ^= 1;
      } else if (f == s_factors - 1) {
        launch_step<kFinal>(row_ptr, col, val, n, k, tin, X, zcur, theta, flags + f, s);
      } else {
        launch_step<kFactorEnd>(row_ptr, col, val, n, k, tin, z[zi], zcur, theta, flags + f, s);
        zcur = z[zi];
        zi ^= 1;
      }
    }
    reps <<= 1;
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
