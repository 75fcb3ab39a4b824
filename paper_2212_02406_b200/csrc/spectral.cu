// Spectral-norm power iteration on the device — the contraction measurement
// behind theta_trace:
//   dense:  nn::spectral_norm_estimate        (proj/src/kernels.cpp:244-269)
//   sparse: nn::spectral_norm_estimate_shifted (proj/src/kernels.cpp:271-305)
// Same recurrence as the reference: w = M v, next = ‖w‖², u = Mᴴ w,
// v = u/‖u‖, converged when |next − λ| ≤ tol·max(next, 1e-300).  The matrix
// stays resident; every reduction is fixed-order (bit-reproducible).
#include <cmath>
#include <vector>

#include "../../include/nnb.h"
#include "engine.cuh"

namespace nnb {
namespace {

// w = M v (complex, row-major): one warp per row, fixed lane/shuffle order.
__global__ void zgemv_kernel(const double2* __restrict__ M, int64_t n,
                             const double2* __restrict__ v, double2* __restrict__ w) {
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double re = 0.0, im = 0.0;
  for (int64_t c = lane; c < n; c += 32) {
    const double2 m = M[row * n + c], x = v[c];
    re = fma(m.x, x.x, fma(-m.y, x.y, re));
    im = fma(m.x, x.y, fma(m.y, x.x, im));
  }
  re = warp_sum(re);
  im = warp_sum(im);
  if (lane == 0) w[row] = make_double2(re, im);
}

// u = Mᴴ w: thread per column, rows in ascending order (coalesced across the warp).
__global__ void zgemv_h_kernel(const double2* __restrict__ M, int64_t n,
                               const double2* __restrict__ w, double2* __restrict__ u) {
  const int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (col >= n) return;
  double re = 0.0, im = 0.0;
  for (int64_t r = 0; r < n; ++r) {
    const double2 m = M[r * n + col], x = w[r];
    // conj(m) * x
    re = fma(m.x, x.x, fma(m.y, x.y, re));
    im = fma(m.x, x.y, fma(-m.y, x.x, im));
  }
  u[col] = make_double2(re, im);
}

// out = x − θ·W x for real CSR W and complex x (the shifted operator I − θW).
__global__ void shifted_csr_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                   const double* __restrict__ val, int64_t n, double theta,
                                   const double2* __restrict__ x, double2* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
      const double2 xv = x[ci[e]];
      re = fma(val[e], xv.x, re);
      im = fma(val[e], xv.y, im);
    }
    out[r] = make_double2(x[r].x - theta * re, x[r].y - theta * im);
  }
}

__global__ void scale_by_inv_norm_kernel(const double2* __restrict__ u, int64_t n,
                                         const double* __restrict__ ss, double2* __restrict__ v) {
  const double inv = 1.0 / sqrt(*ss);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = make_double2(u[i].x * inv, u[i].y * inv);
}

template <class ApplyFwd, class ApplyAdj>
int power_iteration(int64_t n, double* v /*device, complex n*/, double tol, int max_iters,
                    ApplyFwd fwd, ApplyAdj adj, double* value, int* converged, int* iters,
                    cudaStream_t s) {
  DevBuf work;
  NNB_TRY(work.alloc(sizeof(double) * (4 * n + 8), s));
  double* w = work.as<double>();
  double* u = w + 2 * n;
  double* ss = u + 2 * n;  // [0] = ‖w‖², [1] = ‖u‖²
  double lambda = 0.0;
  double h[2];
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(1184, (n + 255) / 256));
  for (int it = 1; it <= max_iters; ++it) {
    NNB_TRY(fwd(v, w));
    NNB_TRY(sumsq(w, 2 * n, ss, s));
    NNB_TRY(adj(w, u));
    NNB_TRY(sumsq(u, 2 * n, ss + 1, s));
    NNB_CUDA(cudaMemcpyAsync(h, ss, sizeof(h), cudaMemcpyDeviceToHost, s));
    NNB_CUDA(cudaStreamSynchronize(s));
    const double next = h[0];
    if (h[1] == 0.0) {
      *value = std::sqrt(next);
      *converged = 1;
      *iters = it;
      return 0;
    }
    scale_by_inv_norm_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const double2*>(u), n, ss + 1,
                                                  reinterpret_cast<double2*>(v));
    count_launch();
    if (it > 1 && std::fabs(next - lambda) <= tol * std::max(next, 1e-300)) {
      *value = std::sqrt(next);
      *converged = 1;
      *iters = it;
      return 0;
    }
    lambda = next;
  }
  *value = std::sqrt(lambda);
  *converged = 0;
  *iters = max_iters;
  return 0;
}

}  // namespace
}  // namespace nnb

using namespace nnb;

extern "C" {

int nnb_spectral_norm_z(const double* M, int64_t n, const double* v0, double tol,
                        int32_t max_iters, double* value, int32_t* converged, int32_t* iterations,
                        void* stream) {
  NNB_TRY(require_device());
  if (tol <= 0.0) return fail(NNB_ERR_DOMAIN, "spectral_norm_estimate: tol must be positive");
  if (n == 0) {
    *value = 0.0;
    *converged = 1;
    *iterations = 0;
    return 0;
  }
  cudaStream_t s = resolve(stream);
  In m;
  NNB_TRY(m.stage(M, (size_t)(2 * n * n), s));
  DevBuf vb;
  NNB_TRY(vb.alloc(sizeof(double) * 2 * n, s));
  NNB_CUDA(cudaMemcpyAsync(vb.p, v0, sizeof(double) * 2 * n, cudaMemcpyDefault, s));
  const double2* md = reinterpret_cast<const double2*>(m.d);
  auto fwd = [&](const double* x, double* y) {
    zgemv_kernel<<<static_cast<unsigned>((n + 7) / 8), 256, 0, s>>>(
        md, n, reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y));
    count_launch();
    NNB_CUDA(cudaGetLastError());
    return 0;
  };
  auto adj = [&](const double* x, double* y) {
    zgemv_h_kernel<<<static_cast<unsigned>((n + 127) / 128), 128, 0, s>>>(
        md, n, reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y));
    count_launch();
    NNB_CUDA(cudaGetLastError());
    return 0;
  };
  int conv = 0, its = 0;
  NNB_TRY(power_iteration(n, vb.as<double>(), tol, max_iters, fwd, adj, value, &conv, &its, s));
  *converged = conv;
  *iterations = its;
  return 0;
}

int nnb_spectral_norm_shifted_csr(const int64_t* row_ptr, const int32_t* col, const double* val,
                                  int64_t n, int64_t nnz, double theta, const double* v0,
                                  double tol, int32_t max_iters, double* value,
                                  int32_t* converged, int32_t* iterations, void* stream) {
  NNB_TRY(require_device());
  if (n == 0) {
    *value = 0.0;
    *converged = 1;
    *iterations = 0;
    return 0;
  }
  cudaStream_t s = resolve(stream);
  DevBuf csr;
  const size_t b_rp = sizeof(int64_t) * (n + 1), b_v = sizeof(double) * nnz,
               b_c = sizeof(int32_t) * nnz;
  NNB_TRY(csr.alloc(b_rp + b_v + b_c + 64, s));
  char* base = csr.as<char>();
  NNB_CUDA(cudaMemcpyAsync(base, row_ptr, b_rp, cudaMemcpyDefault, s));
  NNB_CUDA(cudaMemcpyAsync(base + b_rp, val, b_v, cudaMemcpyDefault, s));
  NNB_CUDA(cudaMemcpyAsync(base + b_rp + b_v, col, b_c, cudaMemcpyDefault, s));
  const int64_t* rp = reinterpret_cast<const int64_t*>(base);
  const double* vv = reinterpret_cast<const double*>(base + b_rp);
  const int32_t* ci = reinterpret_cast<const int32_t*>(base + b_rp + b_v);
  DevBuf vb;
  NNB_TRY(vb.alloc(sizeof(double) * 2 * n, s));
  NNB_CUDA(cudaMemcpyAsync(vb.p, v0, sizeof(double) * 2 * n, cudaMemcpyDefault, s));
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(148 * 16, (n + 255) / 256));
  // the shifted operator is Hermitian (W symmetric): S^H = S
  auto apply = [&](const double* x, double* y) {
    shifted_csr_kernel<<<grid, 256, 0, s>>>(rp, ci, vv, n, theta,
                                            reinterpret_cast<const double2*>(x),
                                            reinterpret_cast<double2*>(y));
    count_launch();
    NNB_CUDA(cudaGetLastError());
    return 0;
  };
  int conv = 0, its = 0;
  NNB_TRY(power_iteration(n, vb.as<double>(), tol, max_iters, apply, apply, value, &conv, &its, s));
  *converged = conv;
  *iterations = its;
  return 0;
}

}  // extern "C"
