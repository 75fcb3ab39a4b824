// Seeded test-matrix generators on the device.
//
// Reference: proj/src/kernels.cpp:64-105 (householder_q), :116-124
// (log_uniform_spectrum), :352-381 (random_spd), :383-407
// (random_conditioned_complex).  The reference runs these as naive
// single-threaded O(n^3) loops — minutes at the C3 size (N = 4096).  Here:
//   * the Gaussian matrix comes from the host-side GaussianStream (a
//     sequential mt19937_64 stream; the caller draws it) and λ from the
//     host's std::pow, so both are the reference's bits;
//   * Householder QR and the backward accumulation of Q run one reflector at
//     a time: a block stages the strided column in shared memory and one
//     thread forms v and β with the reference's sequential sums (≈10 µs at
//     n = 4096 instead of ≈1 ms of dependent global loads), then one thread
//     per column computes its dot product
//     (ascending i) and applies the rank-1 update to its own column
//     (coalesced across the warp);
//   * W = (Q·diag λ)·Qᵀ goes through the reference-exact GEMM (ascending k,
//     one rounded multiply and add per term) and the averaging
//     symmetrisation.
// Real data: every operation is explicitly rounded (no contraction) in the
// reference's order, so random_spd is BIT-IDENTICAL to the reference's.
// Complex data (random_conditioned_complex): the reference's std::norm and
// std::abs go through hypot; here |z|² = re² + im², so results agree to a
// few ulps rather than bit for bit.
#include "engine.cuh"

namespace nnb {
namespace {

// ---- real --------------------------------------------------------------------
// Reflector k of A (n×n, row-major, in place): v (row k of V, zero left of k) and β
// (0 marks a skipped reflector: zero column or zero v, as the reference's `continue`).
// The block stages the strided column in shared memory (`col`, n − k doubles;
// null: read it from global), then thread 0 runs the sums in the reference's order.
__global__ void reflector_d_kernel(const double* __restrict__ a, int64_t n, int64_t k, double* __restrict__ v,
                                   double* __restrict__ beta, int staged) {
  extern __shared__ double col[];
  const int64_t m = n - k;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double x = i >= k ? a[i * n + k] : 0.0;
    if (staged && i >= k) col[i - k] = x;
    v[i] = x;  // a's column; v[k] is fixed up below
  }
  __syncthreads();
  if (threadIdx.x) return;
  const double* c = staged ? col : v + k;
  double xnorm2 = 0.0;
  for (int64_t i = 0; i < m; ++i) xnorm2 = __dadd_rn(xnorm2, __dmul_rn(c[i], c[i]));
  *beta = 0.0;
  const double xnorm = __dsqrt_rn(xnorm2);
  if (xnorm == 0.0) {
    for (int64_t i = k; i < n; ++i) v[i] = 0.0;  // the reference keeps a zero reflector
    return;
  }
  const double x0 = c[0];
  const double x0abs = fabs(x0);
  const double phase = x0abs > 0.0 ? __ddiv_rn(x0, x0abs) : 1.0;
  const double alpha = __dmul_rn(-phase, xnorm);
  const double vk = __dsub_rn(x0, alpha);
  v[k] = vk;
  double vnorm2 = __dmul_rn(vk, vk);
  for (int64_t i = 1; i < m; ++i) vnorm2 = __dadd_rn(vnorm2, __dmul_rn(c[i], c[i]));
  if (vnorm2 == 0.0) return;
  *beta = __ddiv_rn(2.0, vnorm2);
}

// M ← (I − β v vᵀ) M on rows [k, n) of columns [j0, n).  A block owns 32
// columns: its 256 threads stage row tiles of those columns in shared memory
// (coalesced, many loads in flight), one thread per column runs its dot
// product over the tile in ascending i (the reference's order), and the
// rank-1 update is then spread over all threads.
constexpr int kRcCols = 32, kRcRows = 128, kRcThreads = 256;
__global__ void __launch_bounds__(kRcThreads)
    reflect_columns_d_kernel(double* __restrict__ m, int64_t n, int64_t k, int64_t j0, const double* __restrict__ v,
                             const double* __restrict__ beta) {
  __shared__ double tile[kRcRows][kRcCols + 1];
  __shared__ double vs[kRcRows];
  __shared__ double dots[kRcCols];
  const double b = *beta;
  if (b == 0.0) return;
  const int64_t jb = j0 + blockIdx.x * (int64_t)kRcCols;
  const int lane = threadIdx.x % kRcCols, row = threadIdx.x / kRcCols;  // 8 rows of 32 columns per pass
  const int64_t j = jb + lane;
  double dot = 0.0;
  for (int64_t i0 = k; i0 < n; i0 += kRcRows) {
    const int rows = (int)std::min<int64_t>(kRcRows, n - i0);
    for (int r = row; r < rows; r += kRcThreads / kRcCols) tile[r][lane] = j < n ? m[(i0 + r) * n + j] : 0.0;
    for (int r = threadIdx.x; r < rows; r += kRcThreads) vs[r] = v[i0 + r];
    __syncthreads();
    if (threadIdx.x < kRcCols)
      for (int r = 0; r < rows; ++r) dot = __dadd_rn(dot, __dmul_rn(vs[r], tile[r][threadIdx.x]));
    __syncthreads();
  }
  if (threadIdx.x < kRcCols) dots[threadIdx.x] = __dmul_rn(dot, b);
  __syncthreads();
  if (j >= n) return;
  const double d = dots[lane];
  for (int64_t i = k + row; i < n; i += kRcThreads / kRcCols) m[i * n + j] = __dsub_rn(m[i * n + j], __dmul_rn(v[i], d));
}

__global__ void identity_d_kernel(double* q, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x)
    q[e] = (e / n == e % n) ? 1.0 : 0.0;
}

__global__ void scale_columns_d_kernel(const double* __restrict__ q, const double* __restrict__ lam, int64_t n,
                                       double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = __dmul_rn(q[e], lam[e % n]);
}

// w(i,j) = w(j,i) = (w(i,j) + w(j,i))·0.5 for i < j; counts non-finite entries.
__global__ void symmetrize_d_kernel(double* w, int64_t n, int* nonfinite) {
  int bad = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    if (i < j) {
      const double avg = __dmul_rn(__dadd_rn(w[i * n + j], w[j * n + i]), 0.5);
      w[i * n + j] = avg;
      w[j * n + i] = avg;
      bad += !isfinite(avg);
    } else if (i == j) {
      bad += !isfinite(w[e]);
    }
  }
  if (bad) atomicAdd(nonfinite, bad);
}

// ---- complex (interleaved double2) ----------------------------------------------
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {  // (ac − bd) + i(ad + bc), each op rounded
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double cnorm(double2 a) { return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y)); }

__global__ void reflector_z_kernel(const double2* __restrict__ a, int64_t n, int64_t k, double2* __restrict__ v,
                                   double* __restrict__ beta) {
  if (threadIdx.x | blockIdx.x) return;
  double xnorm2 = 0.0;
  for (int64_t i = k; i < n; ++i) xnorm2 = __dadd_rn(xnorm2, cnorm(a[i * n + k]));
  for (int64_t i = 0; i < n; ++i) v[i] = make_double2(0.0, 0.0);
  *beta = 0.0;
  const double xnorm = __dsqrt_rn(xnorm2);
  if (xnorm == 0.0) return;
  const double2 x0 = a[k * n + k];
  const double x0abs = hypot(x0.x, x0.y);
  const double2 phase = x0abs > 0.0 ? make_double2(__ddiv_rn(x0.x, x0abs), __ddiv_rn(x0.y, x0abs))
                                    : make_double2(1.0, 0.0);
  const double2 alpha = make_double2(__dmul_rn(-phase.x, xnorm), __dmul_rn(-phase.y, xnorm));
  for (int64_t i = k; i < n; ++i) v[i] = a[i * n + k];
  v[k] = make_double2(__dsub_rn(v[k].x, alpha.x), __dsub_rn(v[k].y, alpha.y));
  double vnorm2 = 0.0;
  for (int64_t i = k; i < n; ++i) vnorm2 = __dadd_rn(vnorm2, cnorm(v[i]));
  if (vnorm2 == 0.0) return;
  *beta = __ddiv_rn(2.0, vnorm2);
}

__global__ void reflect_columns_z_kernel(double2* __restrict__ m, int64_t n, int64_t k, int64_t j0,
                                         const double2* __restrict__ v, const double* __restrict__ beta) {
  const double b = *beta;
  const int64_t j = j0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b == 0.0 || j >= n) return;
  double2 dot = make_double2(0.0, 0.0);
  for (int64_t i = k; i < n; ++i) {
    const double2 t = cmul(cconj(v[i]), m[i * n + j]);
    dot = make_double2(__dadd_rn(dot.x, t.x), __dadd_rn(dot.y, t.y));
  }
  dot = make_double2(__dmul_rn(dot.x, b), __dmul_rn(dot.y, b));
  for (int64_t i = k; i < n; ++i) {
    const double2 t = cmul(v[i], dot);
    m[i * n + j] = make_double2(__dsub_rn(m[i * n + j].x, t.x), __dsub_rn(m[i * n + j].y, t.y));
  }
}

__global__ void identity_z_kernel(double2* q, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x)
    q[e] = make_double2((e / n == e % n) ? 1.0 : 0.0, 0.0);
}

// a(i,j) = Σ_k u(i,k)·σ_k·conj(v(j,k)), ascending k (random_conditioned_complex's product).
__global__ void usvh_z_kernel(const double2* __restrict__ u, const double2* __restrict__ v,
                              const double* __restrict__ sigma, int64_t n, double2* __restrict__ a, int* nonfinite) {
  int bad = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    double2 sum = make_double2(0.0, 0.0);
    for (int64_t k = 0; k < n; ++k) {
      const double2 us = make_double2(__dmul_rn(u[i * n + k].x, sigma[k]), __dmul_rn(u[i * n + k].y, sigma[k]));
      const double2 t = cmul(us, cconj(v[j * n + k]));
      sum = make_double2(__dadd_rn(sum.x, t.x), __dadd_rn(sum.y, t.y));
    }
    a[e] = sum;
    bad += !(isfinite(sum.x) && isfinite(sum.y));
  }
  if (bad) atomicAdd(nonfinite, bad);
}

unsigned grid_n2(int64_t n) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n * n + 255) / 256, 148 * 16)));
}

// Q of A's Householder QR in `q` (A is consumed).  V holds one reflector per row.
template <typename T, bool CPLX>
int householder_q_dev(T* a, int64_t n, T* q, T* vmat, double* betas, cudaStream_t s) {
  constexpr int kCols = 128;
  constexpr int64_t kMaxStaged = 220 * 1024 / sizeof(double);  // the column fits one SM's shared memory
  const bool staged = !CPLX && n <= kMaxStaged;
  if (staged && n * (int64_t)sizeof(double) > 48 * 1024)
    NNB_TRY(ensure_smem<reflector_d_kernel>((int)(n * sizeof(double))));
  for (int64_t k = 0; k + 1 < n; ++k) {
    T* v = vmat + k * n;
    if constexpr (CPLX) {
      reflector_z_kernel<<<1, 32, 0, s>>>(a, n, k, v, betas + k);
      reflect_columns_z_kernel<<<(unsigned)((n - k + kCols - 1) / kCols), kCols, 0, s>>>(a, n, k, k, v, betas + k);
    } else {
      const size_t smem = staged ? sizeof(double) * (n - k) : 0;
      reflector_d_kernel<<<1, 1024, smem, s>>>(a, n, k, v, betas + k, staged ? 1 : 0);
      reflect_columns_d_kernel<<<(unsigned)((n - k + kRcCols - 1) / kRcCols), kRcThreads, 0, s>>>(a, n, k, k, v,
                                                                                                   betas + k);
    }
  }
  if constexpr (CPLX) identity_z_kernel<<<grid_n2(n), 256, 0, s>>>(q, n);
  else identity_d_kernel<<<grid_n2(n), 256, 0, s>>>(q, n);
  // Q = H_0 H_1 … H_{n−2}: apply the reflectors to I from the last to the first
  for (int64_t r = n - 2; r >= 0; --r) {
    const unsigned blocks = (unsigned)((n + kCols - 1) / kCols);
    if constexpr (CPLX)
      reflect_columns_z_kernel<<<blocks, kCols, 0, s>>>(q, n, r, 0, vmat + r * n, betas + r);
    else
      reflect_columns_d_kernel<<<(unsigned)((n + kRcCols - 1) / kRcCols), kRcThreads, 0, s>>>(q, n, r, 0,
                                                                                              vmat + r * n, betas + r);
  }
  count_launch(n > 1 ? 3 * (n - 1) + 1 : 1);
  NNB_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace

int householder_q(const double* A, int64_t n, int cplx, double* Q, cudaStream_t s) {
  const size_t el = cplx ? 2 : 1, mat = (size_t)(n * n) * el;
  DevBuf work;
  NNB_TRY(work.alloc(sizeof(double) * (2 * mat + n), s));
  double* a = work.as<double>();
  double* vmat = a + mat;
  double* betas = vmat + mat;
  NNB_CUDA(cudaMemcpyAsync(a, A, sizeof(double) * mat, cudaMemcpyDeviceToDevice, s));
  if (cplx)
    return householder_q_dev<double2, true>(reinterpret_cast<double2*>(a), n, reinterpret_cast<double2*>(Q),
                                            reinterpret_cast<double2*>(vmat), betas, s);
  return householder_q_dev<double, false>(a, n, Q, vmat, betas, s);
}

int random_spd_dev(const double* G, const double* lam, int64_t n, double* W, cudaStream_t s) {
  const size_t mat = (size_t)(n * n);
  DevBuf work;
  NNB_TRY(work.alloc(sizeof(double) * 3 * mat + 64, s));
  double* q = work.as<double>();
  double* ql = q + mat;
  double* qt = ql + mat;
  int* nonfinite = reinterpret_cast<int*>(qt + mat);
  NNB_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(int), s));
  NNB_TRY(householder_q(G, n, 0, q, s));
  scale_columns_d_kernel<<<grid_n2(n), 256, 0, s>>>(q, lam, n, ql);  // Q·diag(λ)
  NNB_TRY(transpose(q, n, n, 0, qt, s));
  GemmOp op;  // W = (Q·diag λ)·Qᵀ in the reference's ascending-k rounding
  op.A = ql;
  op.lda = n;
  op.B = qt;
  op.ldb = n;
  op.M = op.N = op.K = n;
  op.ep.C = W;
  op.ep.ldc = n;
  NNB_TRY(gemm_exact(op, s));
  symmetrize_d_kernel<<<grid_n2(n), 256, 0, s>>>(W, n, nonfinite);
  count_launch(2);
  NNB_CUDA(cudaGetLastError());
  int bad = 0;
  NNB_CUDA(cudaMemcpyAsync(&bad, nonfinite, sizeof(int), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  if (bad) return fail(2, "random_spd: non-finite entry");
  return 0;
}

int random_conditioned_dev(const double* GU, const double* GV, const double* sigma, int64_t n, double* A,
                           cudaStream_t s) {
  const size_t mat = (size_t)(2 * n * n);
  DevBuf work;
  NNB_TRY(work.alloc(sizeof(double) * 2 * mat + 64, s));
  double* u = work.as<double>();
  double* v = u + mat;
  int* nonfinite = reinterpret_cast<int*>(v + mat);
  NNB_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(int), s));
  NNB_TRY(householder_q(GU, n, 1, u, s));
  NNB_TRY(householder_q(GV, n, 1, v, s));
  usvh_z_kernel<<<grid_n2(n), 256, 0, s>>>(reinterpret_cast<const double2*>(u), reinterpret_cast<const double2*>(v),
                                           sigma, n, reinterpret_cast<double2*>(A), nonfinite);
  count_launch();
  NNB_CUDA(cudaGetLastError());
  int bad = 0;
  NNB_CUDA(cudaMemcpyAsync(&bad, nonfinite, sizeof(int), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  if (bad) return fail(2, "random_conditioned_complex: non-finite entry");
  return 0;
}


// ---------------------------------------------------------------------------
// Gauss–Jordan inverse with partial pivoting (nn::direct_inverse_oracle,
// proj/src/kernels.cpp:317-350): the small-scale ground truth.  Columns run in
// order; per column one block finds the pivot (largest |a(r,col)|, the first
// on ties as the reference's strict `>`), then row swap + pivot-row scaling and
// the elimination run element-parallel — each element still sees the
// reference's single rounded operation, so real inputs give BIT-IDENTICAL
// inverses.  Complex |z| and division follow hypot / Smith (a few ulps).
namespace {

template <typename T>
__device__ __forceinline__ double mag(T v) {
  if constexpr (sizeof(T) == 16) return hypot(v.x, v.y);
  else return fabs(v);
}

// pivot search over rows [col, n) of column col; state[0] = pivot row, scal[0] = d (as doubles)
template <typename T>
__global__ void gj_pivot_kernel(const T* __restrict__ a, int64_t n, int64_t col, double floor_,
                                long long* __restrict__ piv, T* __restrict__ d, int* __restrict__ singular) {
  __shared__ double best[1024];
  __shared__ long long who[1024];
  double b = -1.0;
  long long w = col;
  for (int64_t r = col + threadIdx.x; r < n; r += blockDim.x) {
    const double c = mag(a[r * n + col]);
    if (c > b) {  // strided scan: the first (smallest r) maximum of this thread's rows
      b = c;
      w = r;
    }
  }
  best[threadIdx.x] = b;
  who[threadIdx.x] = w;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double ob = best[threadIdx.x + s];
      const long long ow = who[threadIdx.x + s];
      if (ob > best[threadIdx.x] || (ob == best[threadIdx.x] && ow < who[threadIdx.x])) {
        best[threadIdx.x] = ob;
        who[threadIdx.x] = ow;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *piv = who[0];
    *d = a[who[0] * n + col];
    if (!(best[0] > floor_) && *singular < 0) *singular = static_cast<int>(col);
  }
}

__device__ __forceinline__ double gj_div(double x, double d) { return __ddiv_rn(x, d); }
__device__ __forceinline__ double2 gj_div(double2 x, double2 d) {  // Smith, as libgcc's __divdc3
  if (fabs(d.x) >= fabs(d.y)) {
    const double r = __ddiv_rn(d.y, d.x), den = __dadd_rn(__dmul_rn(d.y, r), d.x);
    return make_double2(__ddiv_rn(__dadd_rn(__dmul_rn(x.y, r), x.x), den),
                        __ddiv_rn(__dsub_rn(x.y, __dmul_rn(x.x, r)), den));
  }
  const double r = __ddiv_rn(d.x, d.y), den = __dadd_rn(__dmul_rn(d.x, r), d.y);
  return make_double2(__ddiv_rn(__dadd_rn(__dmul_rn(x.x, r), x.y), den),
                      __ddiv_rn(__dsub_rn(__dmul_rn(x.y, r), x.x), den));
}
__device__ __forceinline__ double gj_fms(double a, double f, double x) { return __dsub_rn(a, __dmul_rn(f, x)); }
__device__ __forceinline__ double2 gj_fms(double2 a, double2 f, double2 x) {
  const double2 p = cmul(f, x);
  return make_double2(__dsub_rn(a.x, p.x), __dsub_rn(a.y, p.y));
}
template <typename T>
__device__ __forceinline__ bool is_zero(T v) {
  if constexpr (sizeof(T) == 16) return v.x == 0.0 && v.y == 0.0;
  else return v == 0.0;
}

// swap rows col and piv, scale the pivot row by 1/d
template <typename T>
__global__ void gj_swap_scale_kernel(T* __restrict__ a, T* __restrict__ inv, int64_t n, int64_t col,
                                     const long long* __restrict__ piv, const T* __restrict__ d,
                                     const int* __restrict__ singular) {
  if (*singular >= 0) return;
  const long long p = *piv;
  const T dv = *d;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const T pa = a[p * n + j], pi = inv[p * n + j];
    if (p != col) {
      a[p * n + j] = a[col * n + j];
      inv[p * n + j] = inv[col * n + j];
    }
    a[col * n + j] = gj_div(pa, dv);
    inv[col * n + j] = gj_div(pi, dv);
  }
}

template <typename T>
__global__ void gj_save_column_kernel(const T* __restrict__ a, int64_t n, int64_t col, const int* __restrict__ singular,
                                      T* __restrict__ fcol) {
  if (*singular >= 0) return;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    fcol[r] = a[r * n + col];
}

template <typename T>
__global__ void gj_eliminate_kernel(T* __restrict__ a, T* __restrict__ inv, int64_t n, int64_t col,
                                    const T* __restrict__ fcol, const int* __restrict__ singular) {
  if (*singular >= 0) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / n, j = e % n;
    if (r == col) continue;
    const T f = fcol[r];
    if (is_zero(f)) continue;  // the reference skips zero multipliers
    a[e] = gj_fms(a[e], f, a[col * n + j]);
    inv[e] = gj_fms(inv[e], f, inv[col * n + j]);
  }
}

template <typename T>
__global__ void gj_identity_kernel(T* q, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    if constexpr (sizeof(T) == 16) q[e] = make_double2((e / n == e % n) ? 1.0 : 0.0, 0.0);
    else q[e] = (e / n == e % n) ? 1.0 : 0.0;
  }
}

template <typename T>
__global__ void gj_nonfinite_kernel(const T* __restrict__ q, int64_t n, int* __restrict__ count) {
  int bad = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
    if constexpr (sizeof(T) == 16) bad += !(isfinite(q[e].x) && isfinite(q[e].y));
    else bad += !isfinite(q[e]);
  }
  if (bad) atomicAdd(count, bad);
}

template <typename T>
int direct_inverse_dev(const T* m, int64_t n, double pivot_floor, T* inv, int* singular_col, cudaStream_t s) {
  DevBuf work;
  NNB_TRY(work.alloc(sizeof(T) * (size_t)(n * n + n + 2) + 64, s));
  T* a = work.as<T>();
  T* fcol = a + n * n;
  T* d = fcol + n;
  long long* piv = reinterpret_cast<long long*>(d + 1);
  int* singular = reinterpret_cast<int*>(piv + 1);
  int* nonfinite = singular + 1;
  NNB_CUDA(cudaMemcpyAsync(a, m, sizeof(T) * n * n, cudaMemcpyDeviceToDevice, s));
  NNB_CUDA(cudaMemsetAsync(singular, 0xff, sizeof(int), s));  // -1
  NNB_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(int), s));
  gj_identity_kernel<T><<<grid_n2(n), 256, 0, s>>>(inv, n);
  const unsigned rows_grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 4)));
  for (int64_t col = 0; col < n; ++col) {
    gj_pivot_kernel<T><<<1, 1024, 0, s>>>(a, n, col, pivot_floor, piv, d, singular);
    gj_swap_scale_kernel<T><<<rows_grid, 256, 0, s>>>(a, inv, n, col, piv, d, singular);
    gj_save_column_kernel<T><<<rows_grid, 256, 0, s>>>(a, n, col, singular, fcol);
    gj_eliminate_kernel<T><<<grid_n2(n), 256, 0, s>>>(a, inv, n, col, fcol, singular);
  }
  gj_nonfinite_kernel<T><<<grid_n2(n), 256, 0, s>>>(inv, n, nonfinite);
  count_launch(4 * n + 2);
  NNB_CUDA(cudaGetLastError());
  int h[2];
  NNB_CUDA(cudaMemcpyAsync(h, singular, sizeof(h), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  *singular_col = h[0];
  if (h[0] < 0 && h[1]) return fail(2, "direct_inverse_oracle: produced a non-finite entry");
  return 0;
}

}  // namespace

int direct_inverse(const double* M, int64_t n, int cplx, double pivot_floor, double* inv, int* singular_col,
                   cudaStream_t s) {
  if (cplx)
    return direct_inverse_dev<double2>(reinterpret_cast<const double2*>(M), n, pivot_floor,
                                       reinterpret_cast<double2*>(inv), singular_col, s);
  return direct_inverse_dev<double>(M, n, pivot_floor, inv, singular_col, s);
}

}  // namespace nnb
