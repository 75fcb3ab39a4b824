/* ORACLE — test infrastructure only.  See nn_oracle.h.
 *
 * Each function restates one reference routine; the file:line it follows is
 * cited beside it.  Complex arithmetic is written out by hand as the
 * reference's std::complex<double> evaluates it for finite operands:
 *   (a*b).re = a.re*b.re - a.im*b.im,  (a*b).im = a.re*b.im + a.im*b.re,
 * compiled with -ffp-contract=off so no FMA changes the rounding (the
 * reference's Release build targets baseline x86-64, which has no FMA).
 */
#include "nn_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double re, im; } cplx;

static int g_threads = 1;
void nno_set_threads(int threads) { g_threads = threads < 1 ? 1 : threads; }

static int all_finite(const double* p, int64_t count2) {
  for (int64_t i = 0; i < count2; ++i)
    if (!isfinite(p[i])) return 0;
  return 1;
}

/* ---- matmul: proj/src/kernels.cpp:137-162 (ascending-k inner sum, row
 * partition that never changes an element's reduction order, :19-40). ---- */
typedef struct {
  const cplx *a, *b;
  cplx* c;
  int64_t k, n, lo, hi;
} mm_job;

static void* mm_rows(void* arg) {
  const mm_job* j = (const mm_job*)arg;
  for (int64_t i = j->lo; i < j->hi; ++i) {
    const cplx* arow = j->a + i * j->k;
    for (int64_t col = 0; col < j->n; ++col) {
      double sre = 0.0, sim = 0.0;
      for (int64_t kk = 0; kk < j->k; ++kk) {
        const cplx x = arow[kk], y = j->b[kk * j->n + col];
        const double pre = x.re * y.re - x.im * y.im;
        const double pim = x.re * y.im + x.im * y.re;
        sre += pre;
        sim += pim;
      }
      j->c[i * j->n + col].re = sre;
      j->c[i * j->n + col].im = sim;
    }
  }
  return NULL;
}

/* Real-data fast path.  When both operands have all-zero imaginary parts
 * (every real chain: C1, C3, C4), std::complex's (a*b).re = a.re*b.re - (±0)
 * is a.re*b.re exactly and every imaginary sum stays +0, so the reference's
 * element C[i][j] = (((0 + a_i0 b_0j) + a_i1 b_1j) + ...) is reproduced by
 * any loop nest that keeps each element's products rounded separately and
 * added in ascending k.  This one holds a 4x16 block of C in vector
 * registers across the whole k loop (mul and add as separate instructions:
 * -ffp-contract=off), over a packed 16-column panel of B.  Pinned
 * bit-for-bit against oracle/_ref like the general loop
 * (tests/test_oracle_pins.py::test_matmul_real_fast_path). */
typedef double v8d __attribute__((vector_size(64)));
typedef struct {
  const double *ar, *br; /* ar m x k, br k x n (real parts) */
  double* cr;            /* m x n */
  int64_t m, k, n, p0, p1; /* panel range [p0, p1) of 16-column panels; p == n/16 is the tail */
} mmr_job;

#define MMR_BODY                                                                         \
  const mmr_job* j = (const mmr_job*)arg;                                                \
  const int64_t m = j->m, k = j->k, n = j->n;                                            \
  v8d* pan = (v8d*)aligned_alloc(64, sizeof(v8d) * 2 * (size_t)(k > 0 ? k : 1));         \
  for (int64_t p = j->p0; p < j->p1; ++p) {                                              \
    const int64_t c0 = p * 16;                                                           \
    if (c0 + 16 <= n) {                                                                  \
      for (int64_t kk = 0; kk < k; ++kk) memcpy(&pan[2 * kk], j->br + kk * n + c0, 128); \
      int64_t i = 0;                                                                     \
      for (; i + 4 <= m; i += 4) {                                                       \
        v8d s00 = {0}, s01 = {0}, s10 = {0}, s11 = {0}, s20 = {0}, s21 = {0}, s30 = {0}, s31 = {0}; \
        const double *a0 = j->ar + i * k, *a1 = a0 + k, *a2 = a1 + k, *a3 = a2 + k;      \
        for (int64_t kk = 0; kk < k; ++kk) {                                             \
          const v8d b0 = pan[2 * kk], b1 = pan[2 * kk + 1];                              \
          v8d t;                                                                         \
          t = a0[kk] * b0; s00 += t; t = a0[kk] * b1; s01 += t;                         \
          t = a1[kk] * b0; s10 += t; t = a1[kk] * b1; s11 += t;                         \
          t = a2[kk] * b0; s20 += t; t = a2[kk] * b1; s21 += t;                         \
          t = a3[kk] * b0; s30 += t; t = a3[kk] * b1; s31 += t;                         \
        }                                                                                \
        memcpy(j->cr + (i + 0) * n + c0, &s00, 64); memcpy(j->cr + (i + 0) * n + c0 + 8, &s01, 64); \
        memcpy(j->cr + (i + 1) * n + c0, &s10, 64); memcpy(j->cr + (i + 1) * n + c0 + 8, &s11, 64); \
        memcpy(j->cr + (i + 2) * n + c0, &s20, 64); memcpy(j->cr + (i + 2) * n + c0 + 8, &s21, 64); \
        memcpy(j->cr + (i + 3) * n + c0, &s30, 64); memcpy(j->cr + (i + 3) * n + c0 + 8, &s31, 64); \
      }                                                                                  \
      for (; i < m; ++i) {                                                               \
        v8d s0 = {0}, s1 = {0};                                                          \
        const double* a0 = j->ar + i * k;                                                \
        for (int64_t kk = 0; kk < k; ++kk) {                                             \
          v8d t = a0[kk] * pan[2 * kk]; s0 += t; t = a0[kk] * pan[2 * kk + 1]; s1 += t;  \
        }                                                                                \
        memcpy(j->cr + i * n + c0, &s0, 64); memcpy(j->cr + i * n + c0 + 8, &s1, 64);    \
      }                                                                                  \
    } else {                                                                             \
      for (int64_t i = 0; i < m; ++i)                                                    \
        for (int64_t col = c0; col < n; ++col) {                                         \
          double s = 0.0;                                                                \
          for (int64_t kk = 0; kk < k; ++kk) { const double t = j->ar[i * k + kk] * j->br[kk * n + col]; s += t; } \
          j->cr[i * n + col] = s;                                                        \
        }                                                                                \
    }                                                                                    \
  }                                                                                      \
  free(pan);                                                                             \
  return NULL;

__attribute__((target("avx512f"))) static void* mmr_panels_avx512(void* arg) { MMR_BODY }
static void* mmr_panels_generic(void* arg) { MMR_BODY }

static int imag_all_zero(const double* p, int64_t count) {
  for (int64_t i = 0; i < count; ++i)
    if (p[2 * i + 1] != 0.0) return 0;
  return 1;
}

/* real row-major ar (m x k) times br (k x n) into cr, ascending k per element */
static void matmul_real_raw(const double* ar, const double* br, int64_t m, int64_t k, int64_t n, double* cr) {
  void* (*fn)(void*) = __builtin_cpu_supports("avx512f") ? mmr_panels_avx512 : mmr_panels_generic;
  const int64_t panels = (n + 15) / 16;
  int workers = g_threads < panels ? g_threads : (int)panels;
  if (workers < 1) workers = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * workers);
  mmr_job* jobs = (mmr_job*)malloc(sizeof(mmr_job) * workers);
  for (int w = 0; w < workers; ++w) {
    jobs[w] = (mmr_job){ar, br, cr, m, k, n, panels * w / workers, panels * (w + 1) / workers};
    if (workers > 1) pthread_create(&th[w], NULL, fn, &jobs[w]);
  }
  if (workers > 1) for (int w = 0; w < workers; ++w) pthread_join(th[w], NULL);
  else fn(&jobs[0]);
  free(th); free(jobs);
}

static void matmul_real(const double* a, const double* b, int64_t m, int64_t k, int64_t n, double* c) {
  double* ar = (double*)malloc(sizeof(double) * (size_t)(m * k + 1));
  double* br = (double*)malloc(sizeof(double) * (size_t)(k * n + 1));
  double* cr = (double*)malloc(sizeof(double) * (size_t)(m * n + 1));
  for (int64_t i = 0; i < m * k; ++i) ar[i] = a[2 * i];
  for (int64_t i = 0; i < k * n; ++i) br[i] = b[2 * i];
  matmul_real_raw(ar, br, m, k, n, cr);
  for (int64_t i = 0; i < m * n; ++i) { c[2 * i] = cr[i]; c[2 * i + 1] = 0.0; }
  free(ar); free(br); free(cr);
}

int nno_matmul_z(const double* a, const double* b, int64_t m, int64_t k, int64_t n, double* c) {
  if (m * n >= 4096 && imag_all_zero(a, m * k) && imag_all_zero(b, k * n)) {
    matmul_real(a, b, m, k, n, c);
    return all_finite(c, 2 * m * n) ? 0 : 2;
  }
  int workers = g_threads;
  if (workers <= 1 || m < 64) {
    mm_job j = {(const cplx*)a, (const cplx*)b, (cplx*)c, k, n, 0, m};
    mm_rows(&j);
  } else {
    if (workers > m) workers = (int)m;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * workers);
    mm_job* jobs = (mm_job*)malloc(sizeof(mm_job) * workers);
    const int64_t chunk = (m + workers - 1) / workers;
    int started = 0;
    for (int w = 0; w < workers; ++w) {
      const int64_t lo = w * chunk, hi = lo + chunk < m ? lo + chunk : m;
      if (lo >= hi) break;
      jobs[w] = (mm_job){(const cplx*)a, (const cplx*)b, (cplx*)c, k, n, lo, hi};
      pthread_create(&th[w], NULL, mm_rows, &jobs[w]);
      ++started;
    }
    for (int w = 0; w < started; ++w) pthread_join(th[w], NULL);
    free(th);
    free(jobs);
  }
  return all_finite(c, 2 * m * n) ? 0 : 2; /* check_finite, kernels.cpp:14-17 */
}

/* frobenius_norm: proj/src/kernels.cpp:238-242 (serial sum of std::norm). */
double nno_frobenius_z(const double* m, int64_t count) {
  double s = 0.0;
  for (int64_t i = 0; i < count; ++i) s += m[2 * i] * m[2 * i] + m[2 * i + 1] * m[2 * i + 1];
  return sqrt(s);
}

/* identity_minus: proj/src/kernels.cpp:203-212 (in place). */
static void identity_minus_inplace(cplx* m, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      cplx* v = &m[i * n + j];
      v->re = (i == j ? 1.0 : 0.0) - v->re;
      v->im = 0.0 - v->im;
    }
}

/* plus_identity: proj/src/kernels.cpp:214-221 (in place). */
static void plus_identity_inplace(cplx* m, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    m[i * n + i].re += 1.0;
    m[i * n + i].im += 0.0;
  }
}

/* residual_epsilon: proj/src/solver.cpp:72-75. */
int nno_residual_eps_z(const double* x, const double* a, int64_t n, double* eps) {
  double* p = (double*)malloc(sizeof(double) * 2 * n * n);
  int st = nno_matmul_z(x, a, n, n, n, p);
  if (st == 0) {
    identity_minus_inplace((cplx*)p, n);
    *eps = nno_frobenius_z(p, n * n) / sqrt((double)n);
  }
  free(p);
  return st;
}

/* nn_step: proj/src/solver.cpp:93-103 with horner_power_sum :27-36.
 * P = I - phi W~; S = I + P; S = I + P S (L-1 times); out = S phi. */
int nno_nn_step_z(const double* x, const double* a, int64_t n, int64_t depth_l, double* out) {
  const size_t bytes = sizeof(double) * 2 * n * n;
  if (depth_l == 0) { memmove(out, x, bytes); return 0; }
  double* p = (double*)malloc(bytes);
  double* s = (double*)malloc(bytes);
  double* t = (double*)malloc(bytes);
  int st = nno_matmul_z(x, a, n, n, n, p);
  if (st == 0) {
    identity_minus_inplace((cplx*)p, n);
    memcpy(s, p, bytes);
    plus_identity_inplace((cplx*)s, n);
    for (int64_t j = 2; j <= depth_l && st == 0; ++j) {
      st = nno_matmul_z(p, s, n, n, n, t);
      if (st == 0) {
        plus_identity_inplace((cplx*)t, n);
        double* sw = s; s = t; t = sw;
      }
    }
    if (st == 0) st = nno_matmul_z(s, x, n, n, n, t);
    if (st == 0) memcpy(out, t, bytes);
  }
  free(p); free(s); free(t);
  return st;
}

static int is_identity(const cplx* m, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      const cplx v = m[i * n + j];
      if (v.re != (i == j ? 1.0 : 0.0) || v.im != 0.0) return 0;
    }
  return 1;
}

/* ns_sum: proj/src/solver.cpp:77-91.  P = I - phi0 W~ (product skipped when
 * phi0 == I), t = I + P, t = t P + I (order-1 times), return t phi0. */
int nno_ns_sum_z(const double* x0, const double* a, int64_t n, int64_t order, double* out) {
  const size_t bytes = sizeof(double) * 2 * n * n;
  if (order == 0) { memmove(out, x0, bytes); return 0; }
  const int identity_start = is_identity((const cplx*)x0, n);
  double* p = (double*)malloc(bytes);
  double* t = (double*)malloc(bytes);
  double* u = (double*)malloc(bytes);
  int st = 0;
  if (identity_start) memcpy(p, a, bytes);
  else st = nno_matmul_z(x0, a, n, n, n, p);
  if (st == 0) {
    identity_minus_inplace((cplx*)p, n);
    memcpy(t, p, bytes);
    plus_identity_inplace((cplx*)t, n);
    for (int64_t step = 2; step <= order && st == 0; ++step) {
      st = nno_matmul_z(t, p, n, n, n, u);
      if (st == 0) {
        plus_identity_inplace((cplx*)u, n);
        double* sw = t; t = u; u = sw;
      }
    }
    if (st == 0) {
      if (identity_start) memcpy(out, t, bytes);
      else st = nno_matmul_z(t, x0, n, n, n, out);
    }
  }
  free(p); free(t); free(u);
  return st;
}

/* SURVEY §8(c) explicit-X0 driver over residual_epsilon + nn_step, the loop
 * body of nn_invert (proj/src/solver.cpp:138-159). */
int nno_chain_z(const double* a, int64_t n, const double* x0, int p, int max_iters, double tol,
                double* x_out, double* eps_hist, int* iters_out, int* fail_iter) {
  const size_t bytes = sizeof(double) * 2 * n * n;
  double* x = (double*)malloc(bytes);
  memcpy(x, x0, bytes);
  int it = 0, st = 0;
  for (;;) {
    double eps = 0.0;
    st = nno_residual_eps_z(x, a, n, &eps);
    if (st) break;
    if (eps_hist) eps_hist[it] = eps;
    if (tol > 0.0 && eps < tol) break;
    if (it >= max_iters) break;
    st = nno_nn_step_z(x, a, n, p, x);
    if (st) { st = 3; if (fail_iter) *fail_iter = it + 1; break; }
    ++it;
  }
  if (iters_out) *iters_out = it;
  memcpy(x_out, x, bytes);
  free(x);
  return st;
}

/* Batched C2 leg: Jacobi X0 = diag(A)^-1 then the chain (mode 0, eps after
 * the last nest in eps_last) or ns_sum of order `iters` (mode 1). */
typedef struct {
  int mode, p, iters, stride, t;
  const double* a;
  int64_t batch, n;
  double *x, *eps;
  int status;
} batch_job;

static void* batch_worker(void* arg) {
  batch_job* j = (batch_job*)arg;
  const int64_t n = j->n, nn = n * n;
  double* x0 = (double*)calloc(2 * nn, sizeof(double));
  double* hist = (double*)malloc(sizeof(double) * (j->iters + 1));
  for (int64_t s = j->t; s < j->batch; s += j->stride) {
    const double* a = j->a + 2 * s * nn;
    memset(x0, 0, sizeof(double) * 2 * nn);
    for (int64_t i = 0; i < n; ++i) {
      /* Scalar{1,0} / a(i,i) as libgcc's __divdc3 evaluates it (Smith's
       * ratio form); for the Hermitian diagonal (im == 0) this is 1/re. */
      const double c = a[2 * (i * n + i)], d = a[2 * (i * n + i) + 1];
      double xr, xi;
      if (fabs(c) >= fabs(d)) {
        const double r = d / c, den = c + d * r;
        xr = (1.0 + 0.0 * r) / den;
        xi = (0.0 - 1.0 * r) / den;
      } else {
        const double r = c / d, den = c * r + d;
        xr = (1.0 * r + 0.0) / den;
        xi = (0.0 * r - 1.0) / den;
      }
      x0[2 * (i * n + i)] = xr;
      x0[2 * (i * n + i) + 1] = xi;
    }
    int st;
    if (j->mode == 0)
      st = nno_chain_z(a, n, x0, j->p, j->iters, 0.0, j->x + 2 * s * nn, hist, NULL, NULL);
    else
      st = nno_ns_sum_z(x0, a, n, j->iters, j->x + 2 * s * nn);
    if (st) j->status = st;
    if (j->mode == 0 && j->eps) j->eps[s] = hist[j->iters];
  }
  free(x0);
  free(hist);
  return NULL;
}

int nno_batched_z(int mode, const double* a, int64_t batch, int64_t n, int p, int iters,
                  double* x_out, double* eps_last, int threads) {
  const int saved = g_threads;
  g_threads = 1; /* parallel across systems, serial inside (n < 64 anyway) */
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  batch_job* jobs = (batch_job*)malloc(sizeof(batch_job) * threads);
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (batch_job){mode, p, iters, threads, t, a, batch, n, x_out, eps_last, 0};
    pthread_create(&th[t], NULL, batch_worker, &jobs[t]);
  }
  int st = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(th[t], NULL);
    if (jobs[t].status) st = jobs[t].status;
  }
  free(th);
  free(jobs);
  g_threads = saved;
  return st;
}

/* spmv_block: proj/src/kernels.cpp:454-471 (real CSR values, complex block). */
int nno_spmv_block_z(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n,
                     const double* x, int64_t k, double* out) {
  for (int64_t r = 0; r < n; ++r)
    for (int64_t c = 0; c < k; ++c) {
      double sre = 0.0, sim = 0.0;
      for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
        const double v = val[e];
        const double xr = x[2 * (col[e] * k + c)], xi = x[2 * (col[e] * k + c) + 1];
        const double pre = v * xr - 0.0 * xi;
        const double pim = v * xi + 0.0 * xr;
        sre += pre;
        sim += pim;
      }
      out[2 * (r * k + c)] = sre;
      out[2 * (r * k + c) + 1] = sim;
    }
  return all_finite(out, 2 * n * k) ? 0 : 2;
}

/* solve_sparse_factorized: proj/src/factorized.cpp:101-140 with
 * fused_axpy_sub :21-30.  Z = B; for n < s: t = Z, 2^n x (t = t - theta W t),
 * Z = Z + t; return theta Z.  gamma + 1 must be a power of two. */
int nno_sparse_factorized_z(const int64_t* row_ptr, const int32_t* col, const double* val,
                            int64_t n, const double* b, int64_t k, int64_t gamma, double theta,
                            double* x_out, int64_t* spmv_count, int* fail_index) {
  if (gamma < 1 || ((gamma + 1) & gamma) != 0) return 5; /* PlanError */
  int s = 0;
  for (int64_t g = gamma + 1; g > 1; g >>= 1) ++s;
  const int64_t cnt = 2 * n * k;
  double* z = (double*)malloc(sizeof(double) * cnt);
  double* t = (double*)malloc(sizeof(double) * cnt);
  double* y = (double*)malloc(sizeof(double) * cnt);
  memcpy(z, b, sizeof(double) * cnt);
  int64_t reps = 1, applied = 0;
  int st = 0;
  for (int f = 0; f < s && st == 0; ++f) {
    memcpy(t, z, sizeof(double) * cnt);
    for (int64_t r = 0; r < reps; ++r) {
      if (nno_spmv_block_z(row_ptr, col, val, n, t, k, y)) { st = 3; break; }
      applied += k;
      for (int64_t i = 0; i < cnt; ++i) t[i] = t[i] - theta * y[i];
      if (!all_finite(t, cnt)) { st = 3; break; }
    }
    if (st) { if (fail_index) *fail_index = f; break; }
    for (int64_t i = 0; i < cnt; ++i) z[i] = z[i] + t[i];
    reps <<= 1;
  }
  if (st == 0)
    for (int64_t i = 0; i < cnt; ++i) x_out[i] = z[i] * theta;
  if (spmv_count) *spmv_count = applied;
  free(z); free(t); free(y);
  return st;
}

/* ---- GaussianStream: proj/include/nn/rng.hpp:15-52 (mt19937_64 + Box-Muller,
 * libm log/sqrt/sin/cos), restated with the standard mt19937_64 recurrence. ---- */
typedef struct {
  uint64_t mt[312];
  int mti;
  double spare;
  int have_spare;
} gauss_stream;

static void gs_init(gauss_stream* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i) g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->mti = 312;
  g->have_spare = 0;
  g->spare = 0.0;
}

static uint64_t gs_u64(gauss_stream* g) {
  static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t um = 0xFFFFFFFF80000000ULL, lm = 0x7FFFFFFFULL;
  if (g->mti >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (g->mt[i] & um) | (g->mt[i + 1] & lm);
      g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ mag[x & 1];
    }
    for (; i < 311; ++i) {
      x = (g->mt[i] & um) | (g->mt[i + 1] & lm);
      g->mt[i] = g->mt[i + (156 - 312)] ^ (x >> 1) ^ mag[x & 1];
    }
    x = (g->mt[311] & um) | (g->mt[0] & lm);
    g->mt[311] = g->mt[155] ^ (x >> 1) ^ mag[x & 1];
    g->mti = 0;
  }
  uint64_t x = g->mt[g->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

static double gs_uniform01(gauss_stream* g) { return (double)(gs_u64(g) >> 11) * 0x1.0p-53; }

static double gs_next(gauss_stream* g) {
  if (g->have_spare) {
    g->have_spare = 0;
    return g->spare;
  }
  double u1 = 0.0;
  do {
    u1 = gs_uniform01(g);
  } while (u1 <= 0.0);
  const double u2 = gs_uniform01(g);
  const double radius = sqrt(-2.0 * log(u1));
  const double angle = 2.0 * 3.14159265358979323846 * u2;
  g->spare = radius * sin(angle);
  g->have_spare = 1;
  return radius * cos(angle);
}

void nno_gaussian(uint64_t seed, int64_t count, double* out) {
  gauss_stream g;
  gs_init(&g, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = gs_next(&g);
}

/* ---- random_spd: proj/src/kernels.cpp:64-124,352-381 for real data.
 * householder_q's column loops (for j: dot_j = Σ_i conj(v_i) a(i,j); a(i,j) -= v_i dot_j)
 * are run row-wise here -- every dot_j still accumulates in ascending i and every
 * a(i,j) sees the same single update -- so the result is the reference's bit for bit
 * (std::complex on zero imaginary parts is real arithmetic: conj(v)*a has real part
 * v*a - (-0)*0 = v*a).  Pinned against oracle/_ref (tests/test_oracle_pins.py). ---- */
#define HH_APPLY_BODY                                                                   \
  for (int64_t j = j0; j < n; ++j) dot[j] = 0.0;                                        \
  for (int64_t i = r0; i < n; ++i) {                                                    \
    const double vi = v[i];                                                             \
    const double* row = m + i * n;                                                      \
    for (int64_t j = j0; j < n; ++j) { const double t = vi * row[j]; dot[j] += t; }     \
  }                                                                                     \
  for (int64_t j = j0; j < n; ++j) dot[j] *= beta;                                      \
  for (int64_t i = r0; i < n; ++i) {                                                    \
    const double vi = v[i];                                                             \
    double* row = m + i * n;                                                            \
    for (int64_t j = j0; j < n; ++j) { const double t = vi * dot[j]; row[j] -= t; }     \
  }

/* m <- (I - beta v v^T) m on rows r0.., columns j0.. */
__attribute__((target("avx512f"))) static void hh_apply_avx512(double* m, const double* v, double* dot, int64_t n,
                                                                int64_t r0, int64_t j0, double beta) {
  HH_APPLY_BODY
}
static void hh_apply_generic(double* m, const double* v, double* dot, int64_t n, int64_t r0, int64_t j0,
                             double beta) {
  HH_APPLY_BODY
}

int nno_random_spd(int64_t n, double cond, uint64_t seed, double* out) {
  if (n < 1 || cond < 1.0) return 2;
  void (*apply)(double*, const double*, double*, int64_t, int64_t, int64_t, double) =
      __builtin_cpu_supports("avx512f") ? hh_apply_avx512 : hh_apply_generic;
  double* a = (double*)malloc(sizeof(double) * n * n);
  double* refl = (double*)calloc((size_t)n * n, sizeof(double));
  double* dot = (double*)malloc(sizeof(double) * n);
  nno_gaussian(seed, n * n, a);
  /* householder_q: kernels.cpp:64-103 */
  for (int64_t k = 0; k + 1 < n; ++k) {
    double* v = refl + k * n;
    double xnorm2 = 0.0;
    for (int64_t i = k; i < n; ++i) { const double t = a[i * n + k] * a[i * n + k]; xnorm2 += t; }
    const double xnorm = sqrt(xnorm2);
    if (xnorm == 0.0) continue;
    const double x0 = a[k * n + k];
    const double x0abs = fabs(x0);
    const double phase = x0abs > 0.0 ? x0 / x0abs : 1.0;
    const double alpha = -phase * xnorm;
    for (int64_t i = k; i < n; ++i) v[i] = a[i * n + k];
    v[k] -= alpha;
    double vnorm2 = 0.0;
    for (int64_t i = k; i < n; ++i) { const double t = v[i] * v[i]; vnorm2 += t; }
    if (vnorm2 == 0.0) continue;
    apply(a, v, dot, n, k, k, 2.0 / vnorm2);
  }
  /* Q = H_0 ... H_{n-2}, applied to I from the last reflector (kernels.cpp:91-102) */
  double* q = (double*)calloc((size_t)n * n, sizeof(double));
  for (int64_t i = 0; i < n; ++i) q[i * n + i] = 1.0;
  for (int64_t r = n - 1; r-- > 0;) {
    const double* v = refl + r * n;
    double vnorm2 = 0.0;
    for (int64_t i = r; i < n; ++i) { const double t = v[i] * v[i]; vnorm2 += t; }
    if (vnorm2 == 0.0) continue;
    apply(q, v, dot, n, r, 0, 2.0 / vnorm2);
  }
  /* lambda (kernels.cpp:116-124), ql = Q diag(lambda), w = ql Q^T, symmetrised (:359-379) */
  double* ql = (double*)malloc(sizeof(double) * n * n);
  for (int64_t j = 0; j < n; ++j) {
    const double lam = n == 1 ? 1.0 : pow(cond, -((double)(n - 1 - j) / (double)(n - 1)));
    for (int64_t i = 0; i < n; ++i) ql[i * n + j] = q[i * n + j] * lam;
  }
  double* qt = (double*)malloc(sizeof(double) * n * n);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) qt[j * n + i] = q[i * n + j];
  matmul_real_raw(ql, qt, n, n, n, out);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) {
      const double avg = (out[i * n + j] + out[j * n + i]) * 0.5;
      out[i * n + j] = avg;
      out[j * n + i] = avg;
    }
  free(a); free(refl); free(dot); free(q); free(ql); free(qt);
  return all_finite(out, n * n) ? 0 : 2;
}
