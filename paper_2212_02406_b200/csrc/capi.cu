// extern "C" entry points of libnnb.so (declared in include/nnb.h).
//
// Each entry point validates its arguments the way the reference routine it
// replaces does, stages host operands through device buffers (padded to an
// even leading dimension so the TMA descriptors and 16-byte epilogue stores
// are legal), runs the device path, and copies results back.  No entry
// point computes anything on the host.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../../include/nnb.h"
#include "engine.cuh"
#include "sparse.cuh"

using namespace nnb;

void nnb::trace_dump() {
  if (!trace_on()) return;
  int* n;
  TraceMark* m = trace_marks(&n);
  cudaDeviceSynchronize();
  for (int i = 0; i < *n; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, m[0].ev, m[i].ev);
    std::fprintf(stderr, "trace %9.2f ms  host %9.2f ms  %s\n", ms, m[i].host_ms - m[0].host_ms, m[i].label);
  }
  for (int i = 0; i < *n; ++i) cudaEventDestroy(m[i].ev);
  *n = 0;
}

namespace {

int64_t pad8(int64_t c) { return (c + 7) / 8 * 8; }

// Device view of a row-major rows×cols FP64 matrix with an even leading
// dimension and 16B-aligned base: borrows a suitable device pointer, else
// stages a padded copy.
struct DMat {
  double* d = nullptr;
  int64_t ld = 0, rows = 0, cols = 0;
  DevBuf own;
  int alloc(int64_t r, int64_t c, cudaStream_t s) {
    rows = r;
    cols = c;
    ld = pad8(c);
    NNB_TRY(own.alloc(sizeof(double) * std::max<int64_t>(1, r * ld), s));
    d = own.as<double>();
    return 0;
  }
  int load(const double* src, int64_t r, int64_t c, int64_t ld_src, cudaStream_t s,
           bool allow_borrow = true) {
    if (allow_borrow && is_device_ptr(src) && !(reinterpret_cast<uintptr_t>(src) & 15) &&
        !(ld_src & 1)) {
      d = const_cast<double*>(src);
      ld = ld_src;
      rows = r;
      cols = c;
      return 0;
    }
    NNB_TRY(alloc(r, c, s));
    if (r * c)
      NNB_CUDA(cudaMemcpy2DAsync(d, ld * 8, src, ld_src * 8, c * 8, r, cudaMemcpyDefault, s));
    return 0;
  }
  int store(double* dst, int64_t ld_dst, cudaStream_t s) const {
    if (dst != d && rows * cols)
      NNB_CUDA(cudaMemcpy2DAsync(dst, ld_dst * 8, d, ld * 8, cols * 8, rows, cudaMemcpyDefault, s));
    return 0;
  }
};

// Planar (re, im) padded device copy of an interleaved complex matrix.
struct ZMat {
  DevBuf own;
  double *re = nullptr, *im = nullptr;
  int64_t ld = 0, rows = 0, cols = 0;
  int alloc(int64_t r, int64_t c, cudaStream_t s) {
    rows = r;
    cols = c;
    ld = pad8(c);
    NNB_TRY(own.alloc(sizeof(double) * std::max<int64_t>(1, 2 * r * ld), s));
    re = own.as<double>();
    im = re + r * ld;
    NNB_CUDA(cudaMemsetAsync(own.p, 0, own.bytes, s));
    return 0;
  }
  int load(const double* z, int64_t r, int64_t c, cudaStream_t s) {
    NNB_TRY(alloc(r, c, s));
    In in;
    NNB_TRY(in.stage(z, (size_t)(2 * r * c), s));
    return deinterleave2d(in.d, r, c, re, im, ld, s);
  }
  int store(double* z, cudaStream_t s) const {
    Out out;
    NNB_TRY(out.prepare(z, (size_t)(2 * rows * cols), s));
    NNB_TRY(interleave2d(re, im, rows, cols, ld, out.d, s));
    return out.finish(s);
  }
};

int sync(cudaStream_t s) {
  NNB_CUDA(cudaStreamSynchronize(s));
  return 0;
}

int chain_cfg(const nnb_chain_config* cfg, ChainCfg* c) {
  if (!cfg) return fail(NNB_ERR_DOMAIN, "nn chain: config is NULL");
  if (cfg->depth_p < 0) return fail(NNB_ERR_DOMAIN, "nn chain: depth must be >= 0");
  if (cfg->max_iters < 0) return fail(NNB_ERR_DOMAIN, "nn chain: max_iters must be >= 0");
  if (cfg->order != NNB_ORDER_NORTHSTAR && cfg->order != NNB_ORDER_REFERENCE && cfg->order != NNB_ORDER_SYMMETRIC)
    return fail(NNB_ERR_DOMAIN, "nn chain: unknown operand order");
  c->p = cfg->depth_p;
  c->max_iters = cfg->max_iters;
  c->tol = cfg->tol;
  c->order = cfg->order;
  c->final_residual = cfg->final_residual;
  return 0;
}

// NNB_ORDER_SYMMETRIC preconditions: A and X0 exactly symmetric (X0 built
// here is: Aᵀ/(‖A‖₁‖A‖∞), diag(A)⁻¹ or θI of a symmetric A).  Then every
// Horner product X·S(R)·R is symmetric and may compute its upper tile
// triangle only (chain.cu).
int symmetric_check(const nnb_chain_config* cfg, const double* A, const double* X0, int64_t n, int64_t ld,
                    cudaStream_t s) {
  if (cfg->order != NNB_ORDER_SYMMETRIC) return 0;
  bool sym = false;
  NNB_TRY(is_symmetric_dev(A, n, ld, &sym, s));
  if (!sym) return fail(NNB_ERR_DOMAIN, "nn chain: the symmetric order needs A == A^T");
  if (cfg->x0_kind == NNB_X0_GIVEN) {
    NNB_TRY(is_symmetric_dev(X0, n, ld, &sym, s));
    if (!sym) return fail(NNB_ERR_DOMAIN, "nn chain: the symmetric order needs X0 == X0^T");
  }
  return 0;
}

void fill_result(nnb_chain_result* r, const ChainOut& o) {
  if (!r) return;
  r->iters = o.iters;
  r->fail_iter = o.fail_iter;
  r->stopped = o.stopped;
  r->products = o.products;
  r->last_eps = o.last_eps;
  r->device_ms = o.device_ms;
}

// nnb_nn_chain_d with host A and/or host X_out, n >= kStreamMinN, fast
// arithmetic.  X0, then A's row chunks, go host→device on a copy stream with
// an event per chunk, so the first residual product starts once X0 and A's
// first chunk have landed rather than after all 2·8·n² bytes.  The final X
// leaves per chunk of the last Horner product (ChainIo).  NNB_STREAM_CHUNKS
// sets the chunk count (default 16, 1..64: 8 and 32 measured 5-10 % slower e2e at N=32768).
constexpr int64_t kStreamMinN = 8192;

struct CopyLane {
  cudaStream_t cs = nullptr;
  std::vector<cudaEvent_t> ev;
  CopyLane() = default;
  CopyLane(const CopyLane&) = delete;
  CopyLane& operator=(const CopyLane&) = delete;
  ~CopyLane() {
    if (cs) cudaStreamSynchronize(cs);
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    if (cs) cudaStreamDestroy(cs);
  }
  int init(int events) {
    NNB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    ev.assign(events, nullptr);
    for (cudaEvent_t& e : ev) NNB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return 0;
  }
};

int chain_d_streamed(const double* A, int64_t n, const double* X0, const nnb_chain_config* cfg,
                     const ChainCfg& c, double* X_out, double* eps_hist, nnb_chain_result* result,
                     cudaStream_t s) {
  static const int chunks = [] {
    const char* e = debug_env("NNB_STREAM_CHUNKS");
    return std::min(64, std::max(1, e ? std::atoi(e) : 16));
  }();
  const bool host_a = !is_device_ptr(A), host_out = X_out && !is_device_ptr(X_out);
  const bool x0_given = cfg->x0_kind == NNB_X0_GIVEN;
  if (x0_given && !X0) return fail(NNB_ERR_DOMAIN, "nn chain: X0 required for NNB_X0_GIVEN");
  if (trace_on()) trace_reset();
  trace_mark(s, "start");
  DMat a, x;
  if (host_a) NNB_TRY(a.alloc(n, n, s));
  else NNB_TRY(a.load(A, n, n, n, s));
  x.rows = x.cols = n;
  x.ld = a.ld;
  NNB_TRY(x.own.alloc(sizeof(double) * n * a.ld, s));
  x.d = x.own.as<double>();
  CopyLane lane;  // declared after the buffers: its destructor drains the copies before they are freed
  NNB_TRY(lane.init(3 * chunks + 3));
  cudaEvent_t* a_ready = lane.ev.data();
  cudaEvent_t* out_done = a_ready + chunks;
  cudaEvent_t alloc_ev = out_done[chunks], copy_done = out_done[chunks + 1], in_done = out_done[chunks + 2];
  cudaEvent_t* x_cols = out_done + chunks + 3;  // [chunks]
  // the copy stream may touch the stream-ordered allocations only once they exist
  NNB_CUDA(cudaEventRecord(alloc_ev, s));
  NNB_CUDA(cudaStreamWaitEvent(lane.cs, alloc_ev, 0));
  const int64_t rows_per = ((n + chunks - 1) / chunks + 127) / 128 * 128;
  const int used = static_cast<int>((n + rows_per - 1) / rows_per);
  // block q of the first product's inner dimension: X0's rows and A's columns of q
  // the K-split first product resumes DMMA accumulators (acc_in): DMMA-only
  const bool ksplit = host_a && x0_given && cfg->order == NNB_ORDER_NORTHSTAR && arith() == 3;
  // int8 emulation: A by row chunks and X0 by column chunks, interleaved, so block (0, 0)
  // starts after two chunks; the first product R = I − A·X0 runs block by block behind them
  const bool rows_stream = host_a && x0_given && cfg->order == NNB_ORDER_NORTHSTAR && !ksplit && arith() != 1 &&
                           (arith() == 2 || ozaki_pays(n, n, n));
  if (rows_stream) {
    auto copy_a = [&](int q) -> int {
      const int64_t r0 = q * rows_per, rq = std::min<int64_t>(rows_per, n - r0);
      NNB_CUDA(cudaMemcpy2DAsync(a.d + r0 * a.ld, a.ld * 8, A + r0 * n, n * 8, n * 8, rq, cudaMemcpyHostToDevice,
                                 lane.cs));
      NNB_CUDA(cudaEventRecord(a_ready[q], lane.cs));
      trace_mark(lane.cs, "h2d A rows ", q);
      return 0;
    };
    for (int q = 0; q < used; ++q) {  // A_0, X_0, A_1, X_1, ... (chain.cu product_2d's order)
      NNB_TRY(copy_a(q));
      const int64_t c0 = q * rows_per, cq = std::min<int64_t>(rows_per, n - c0);
      NNB_CUDA(cudaMemcpy2DAsync(x.d + c0, x.ld * 8, X0 + c0, n * 8, cq * 8, n, cudaMemcpyDefault, lane.cs));
      NNB_CUDA(cudaEventRecord(x_cols[q], lane.cs));
      trace_mark(lane.cs, "h2d X0 cols ", q);
    }
  } else if (ksplit) {
    for (int q = 0; q < used; ++q) {
      const int64_t k0 = q * rows_per, kq = std::min<int64_t>(rows_per, n - k0);
      NNB_CUDA(cudaMemcpy2DAsync(x.d + k0 * x.ld, x.ld * 8, X0 + k0 * n, n * 8, n * 8, kq, cudaMemcpyDefault,
                                 lane.cs));
      NNB_CUDA(cudaMemcpy2DAsync(a.d + k0, a.ld * 8, A + k0, n * 8, kq * 8, n, cudaMemcpyHostToDevice, lane.cs));
      NNB_CUDA(cudaEventRecord(a_ready[q], lane.cs));
    }
  } else {
    if (x0_given)
      NNB_CUDA(cudaMemcpy2DAsync(x.d, x.ld * 8, X0, n * 8, n * 8, n, cudaMemcpyDefault, lane.cs));
    if (host_a)
      NNB_CUDA(cudaMemcpy2DAsync(a.d, a.ld * 8, A, n * 8, n * 8, n, cudaMemcpyHostToDevice, lane.cs));
  }
  NNB_CUDA(cudaEventRecord(in_done, lane.cs));
  ChainIo io;
  io.chunks = used;
  io.chunk_rows = rows_per;
  io.copy = lane.cs;
  io.out_done = out_done;
  io.copy_done = copy_done;
  io.host_out = host_out ? X_out : nullptr;
  if (ksplit) {
    io.a_ready = a_ready;  // the first product consumes A and X0 block by block
  } else if (rows_stream) {
    io.a_rows_ready = a_ready;
    io.x_cols_ready = x_cols;
  } else {
    NNB_CUDA(cudaStreamWaitEvent(s, in_done, 0));
    if (!x0_given) NNB_TRY(x0_build(a.d, a.ld, n, cfg->x0_kind, cfg->x0_scale, x.d, x.ld, s));
    NNB_TRY(symmetric_check(cfg, a.d, x.d, n, a.ld, s));
  }
  ChainOut o;
  const int st = chain_real(a.d, n, a.ld, x.d, c, eps_hist, &o, s, &io);
  trace_mark(s, "chain done");
  fill_result(result, o);
  if (st != 0 && st != NNB_ERR_DIVERGENCE && st != NNB_ERR_DOMAIN) return st;
  // with zero products (max_iters = 0, no final residual) nothing on s has waited
  // for X0's copy yet; the store must not read x ahead of it
  NNB_CUDA(cudaStreamWaitEvent(s, in_done, 0));
  if (X_out && !io.out_streamed) NNB_TRY(x.store(X_out, n, s));
  NNB_TRY(sync(s));
  NNB_CUDA(cudaStreamSynchronize(lane.cs));
  trace_mark(s, "end");
  trace_dump();
  return st;
}

}  // namespace

extern "C" {

int nnb_abi_version(void) { return NNB_ABI_VERSION; }
const char* nnb_last_error(void) { return last_error(); }
int nnb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}
uint64_t nnb_kernel_launches(void) { return launches(); }

int nnb_release_cached_memory(void) {
  NNB_TRY(require_device());
  int dev = 0;
  NNB_CUDA(cudaGetDevice(&dev));
  NNB_CUDA(cudaDeviceSynchronize());
  cudaMemPool_t pool;
  NNB_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  NNB_CUDA(cudaMemPoolTrimTo(pool, 0));
  return 0;
}

int nnb_set_arithmetic(int32_t mode) {
  if (mode < NNB_ARITH_FAST || mode > NNB_ARITH_DMMA)
    return fail(NNB_ERR_DOMAIN, "nnb_set_arithmetic: unknown mode");
  set_arith(mode);
  return 0;
}
int32_t nnb_get_arithmetic(void) { return arith(); }
int32_t nnb_ozaki_moduli(int64_t k) { return ozaki_moduli_for(k); }
int nnb_chain_capture_residual(double* R_out, int64_t ldr) {
  if (R_out && !is_device_ptr(R_out)) return fail(NNB_ERR_DOMAIN, "residual capture needs a device buffer");
  set_chain_capture(R_out, ldr);
  return 0;
}
void nnb_ozaki_profile(int32_t on) { ozaki_profile(on); }
void nnb_ozaki_stats(double* ms, double* work, int64_t* launches, int32_t reset) {
  ozaki_stats(ms, work, launches, reset);
}

// ---------------------------------------------------------------- dense kernels
int nnb_gemm_d(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
               int64_t m, int64_t k, int64_t n, void* stream) {
  NNB_TRY(require_device());
  if (m < 0 || k < 0 || n < 0 || lda < k || ldb < n || ldc < n)
    return fail(NNB_ERR_SHAPE, "matmul: inner dimensions disagree or bad leading dimension");
  cudaStream_t s = resolve(stream);
  DMat a, b, c;
  NNB_TRY(a.load(A, m, k, lda, s));
  NNB_TRY(b.load(B, k, n, ldb, s));
  const bool direct = is_device_ptr(C) && !(reinterpret_cast<uintptr_t>(C) & 15) && !(ldc & 1);
  if (direct) {
    c.d = C; c.ld = ldc; c.rows = m; c.cols = n;
  } else {
    NNB_TRY(c.alloc(m, n, s));
  }
  RedWs red;
  NNB_TRY(red.init(max_tiles_for(m, n), s));
  DevBuf nf;
  NNB_TRY(nf.alloc(sizeof(int), s));
  NNB_CUDA(cudaMemsetAsync(nf.p, 0, sizeof(int), s));
  GemmOp op;
  op.A = a.d; op.lda = a.ld; op.B = b.d; op.ldb = b.ld;
  op.M = m; op.N = n; op.K = k;
  op.ep.C = c.d; op.ep.ldc = c.ld;
  op.ep.nf_out = nf.as<int>();
  NNB_TRY(gemm(op, &red, s));
  if (!direct) NNB_TRY(c.store(C, ldc, s));
  int h = 0;
  NNB_CUDA(cudaMemcpyAsync(&h, nf.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  NNB_TRY(sync(s));
  if (h) return fail(NNB_ERR_DOMAIN, "matmul: produced a non-finite entry");
  return 0;
}

int nnb_gemm_nt_d(const double* A, int64_t lda, const double* Bt, int64_t ldbt, double* C, int64_t ldc,
                  int64_t m, int64_t k, int64_t n, void* stream) {
  NNB_TRY(require_device());
  if (m < 0 || k < 0 || n < 0 || lda < k || ldbt < k || ldc < n)
    return fail(NNB_ERR_SHAPE, "matmul: inner dimensions disagree or bad leading dimension");
  cudaStream_t s = resolve(stream);
  DMat a, b, c;
  NNB_TRY(a.load(A, m, k, lda, s));
  NNB_TRY(b.load(Bt, n, k, ldbt, s));
  const bool direct = is_device_ptr(C) && !(reinterpret_cast<uintptr_t>(C) & 15) && !(ldc & 1);
  if (direct) {
    c.d = C; c.ld = ldc; c.rows = m; c.cols = n;
  } else {
    NNB_TRY(c.alloc(m, n, s));
  }
  RedWs red;
  NNB_TRY(red.init(max_tiles_for(m, n), s));
  DevBuf nf;
  NNB_TRY(nf.alloc(sizeof(int), s));
  GemmOp op;
  op.A = a.d; op.lda = a.ld; op.B = b.d; op.ldb = b.ld; op.b_kmajor = true;
  op.M = m; op.N = n; op.K = k;
  op.ep.C = c.d; op.ep.ldc = c.ld;
  op.ep.nf_out = nf.as<int>();
  NNB_TRY(gemm(op, &red, s));
  if (!direct) NNB_TRY(c.store(C, ldc, s));
  int h = 0;
  NNB_CUDA(cudaMemcpyAsync(&h, nf.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  NNB_TRY(sync(s));
  if (h) return fail(NNB_ERR_DOMAIN, "matmul: produced a non-finite entry");
  return 0;
}

int nnb_gemm_z(const double* A, const double* B, double* C, int64_t m, int64_t k, int64_t n,
               void* stream) {
  NNB_TRY(require_device());
  if (m < 0 || k < 0 || n < 0) return fail(NNB_ERR_SHAPE, "matmul: bad shape");
  cudaStream_t s = resolve(stream);
  ZMat a, b, c;
  NNB_TRY(a.load(A, m, k, s));
  NNB_TRY(b.load(B, k, n, s));
  NNB_TRY(c.alloc(m, n, s));
  RedWs red;
  NNB_TRY(red.init(max_tiles_for(m, n), s));
  DevBuf nf;
  NNB_TRY(nf.alloc(2 * sizeof(int), s));
  NNB_CUDA(cudaMemsetAsync(nf.p, 0, 2 * sizeof(int), s));
  if (arith() != 1 && k > 0) {  // 3M on DMMA (zgemm3m); the exact mode keeps the 4M form
    ZGemm z;
    z.M = m;
    z.N = n;
    z.K = k;
    z.Ar = a.re;
    z.Ai = a.im;
    z.lda = a.ld;
    z.Br = b.re;
    z.Bi = b.im;
    z.ldb = b.ld;
    z.Cr = c.re;
    z.Ci = c.im;
    z.ldc = c.ld;
    z.ss_out = nullptr;
    z.nf_out = nf.as<int>();
    NNB_TRY(zgemm3m(z, &red, s));
    NNB_TRY(c.store(C, s));
    int h = 0;
    NNB_CUDA(cudaMemcpyAsync(&h, nf.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    NNB_TRY(sync(s));
    if (h) return fail(NNB_ERR_DOMAIN, "matmul: produced a non-finite entry");
    return 0;
  }
  auto run = [&](const double* x, int64_t ldx, const double* y, int64_t ldy, double alpha,
                 const double* d, double* out, int* nfo) {
    GemmOp op;
    op.A = x; op.lda = ldx; op.B = y; op.ldb = ldy;
    op.M = m; op.N = n; op.K = k;
    op.ep.alpha = alpha; op.ep.D = d; op.ep.ldd = c.ld; op.ep.beta = 1.0;
    op.ep.C = out; op.ep.ldc = c.ld; op.ep.nf_out = nfo;
    return gemm(op, nfo ? &red : nullptr, s);
  };
  NNB_TRY(run(a.re, a.ld, b.re, b.ld, 1.0, nullptr, c.re, nullptr));
  NNB_TRY(run(a.im, a.ld, b.im, b.ld, -1.0, c.re, c.re, nf.as<int>()));
  NNB_TRY(run(a.re, a.ld, b.im, b.ld, 1.0, nullptr, c.im, nullptr));
  NNB_TRY(run(a.im, a.ld, b.re, b.ld, 1.0, c.im, c.im, nf.as<int>() + 1));
  NNB_TRY(c.store(C, s));
  int h[2] = {0, 0};
  NNB_CUDA(cudaMemcpyAsync(h, nf.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  NNB_TRY(sync(s));
  if (h[0] || h[1]) return fail(NNB_ERR_DOMAIN, "matmul: produced a non-finite entry");
  return 0;
}

int nnb_axpby_d(double alpha, const double* A, double beta, const double* B, double gamma,
                double* out, int64_t rows, int64_t cols, void* stream) {
  NNB_TRY(require_device());
  if (gamma != 0.0 && rows != cols)
    return fail(NNB_ERR_SHAPE, "identity_minus/plus_identity: matrix must be square");
  cudaStream_t s = resolve(stream);
  const size_t cnt = (size_t)(rows * cols);
  In a, b;
  NNB_TRY(a.stage(A, cnt, s));
  if (B) NNB_TRY(b.stage(B, cnt, s));
  Out o;
  NNB_TRY(o.prepare(out, cnt, s));
  NNB_TRY(axpby(alpha, a.d, cols, beta, B ? b.d : nullptr, cols, gamma, 0, o.d, cols, rows, cols, s));
  NNB_TRY(o.finish(s));
  return sync(s);
}

int nnb_axpby_z(const double* alpha2, const double* A, const double* beta2, const double* B,
                const double* gamma2, double* out, int64_t rows, int64_t cols, void* stream) {
  NNB_TRY(require_device());
  const double g0 = gamma2 ? gamma2[0] : 0.0, g1 = gamma2 ? gamma2[1] : 0.0;
  if ((g0 != 0.0 || g1 != 0.0) && rows != cols)
    return fail(NNB_ERR_SHAPE, "identity_minus/plus_identity: matrix must be square");
  cudaStream_t s = resolve(stream);
  const size_t cnt = (size_t)(2 * rows * cols);
  In a, b;
  NNB_TRY(a.stage(A, cnt, s));
  if (B) NNB_TRY(b.stage(B, cnt, s));
  Out o;
  NNB_TRY(o.prepare(out, cnt, s));
  NNB_TRY(axpby_z(alpha2[0], alpha2[1], a.d, beta2 ? beta2[0] : 0.0, beta2 ? beta2[1] : 0.0,
                  B ? b.d : nullptr, g0, g1, o.d, rows, cols, s));
  NNB_TRY(o.finish(s));
  return sync(s);
}

int nnb_gaussian_stream(uint64_t seed, int64_t count, double* out) {
  // mt19937_64, 53-bit uniforms in (0, 1] for the radius, Box–Muller pairs
  // with the cosine returned first and the sine kept as the spare
  if (count < 0 || (count && !out)) return fail(NNB_ERR_DOMAIN, "gaussian_stream: bad output");
  std::mt19937_64 eng(seed);
  auto unit = [&eng] { return static_cast<double>(eng() >> 11) * 0x1.0p-53; };
  for (int64_t i = 0; i < count; i += 2) {
    double u1 = unit();
    while (u1 <= 0.0) u1 = unit();
    const double u2 = unit();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double ang = 2.0 * 3.14159265358979323846 * u2;
    out[i] = rad * std::cos(ang);
    if (i + 1 < count) out[i + 1] = rad * std::sin(ang);
  }
  return 0;
}

int nnb_householder_q_d(const double* A, int64_t n, double* Q, void* stream) {
  NNB_TRY(require_device());
  if (n < 1) return fail(NNB_ERR_DOMAIN, "householder_q: n must be >= 1");
  cudaStream_t s = resolve(stream);
  In a;
  NNB_TRY(a.stage(A, (size_t)(n * n), s));
  Out q;
  NNB_TRY(q.prepare(Q, (size_t)(n * n), s));
  NNB_TRY(householder_q(a.d, n, 0, q.d, s));
  NNB_TRY(q.finish(s));
  return sync(s);
}

int nnb_householder_q_z(const double* A, int64_t n, double* Q, void* stream) {
  NNB_TRY(require_device());
  if (n < 1) return fail(NNB_ERR_DOMAIN, "householder_q: n must be >= 1");
  cudaStream_t s = resolve(stream);
  In a;
  NNB_TRY(a.stage(A, (size_t)(2 * n * n), s));
  Out q;
  NNB_TRY(q.prepare(Q, (size_t)(2 * n * n), s));
  NNB_TRY(householder_q(a.d, n, 1, q.d, s));
  NNB_TRY(q.finish(s));
  return sync(s);
}

int nnb_random_spd_d(const double* G, const double* lam, int64_t n, double* W, void* stream) {
  NNB_TRY(require_device());
  if (n < 1) return fail(NNB_ERR_DOMAIN, "random_spd: n must be >= 1");
  cudaStream_t s = resolve(stream);
  In g, l;
  NNB_TRY(g.stage(G, (size_t)(n * n), s));
  NNB_TRY(l.stage(lam, (size_t)n, s));
  Out w;
  NNB_TRY(w.prepare(W, (size_t)(n * n), s));
  NNB_TRY(random_spd_dev(g.d, l.d, n, w.d, s));
  NNB_TRY(w.finish(s));
  return sync(s);
}

int nnb_random_conditioned_z(const double* GU, const double* GV, const double* sigma, int64_t n, double* A,
                             void* stream) {
  NNB_TRY(require_device());
  if (n < 1) return fail(NNB_ERR_DOMAIN, "random_conditioned_complex: n must be >= 1");
  cudaStream_t s = resolve(stream);
  In gu, gv, sg;
  NNB_TRY(gu.stage(GU, (size_t)(2 * n * n), s));
  NNB_TRY(gv.stage(GV, (size_t)(2 * n * n), s));
  NNB_TRY(sg.stage(sigma, (size_t)n, s));
  Out a;
  NNB_TRY(a.prepare(A, (size_t)(2 * n * n), s));
  NNB_TRY(random_conditioned_dev(gu.d, gv.d, sg.d, n, a.d, s));
  NNB_TRY(a.finish(s));
  return sync(s);
}

static int direct_inverse_call(const double* M, int64_t n, int cplx, double* out, int32_t* pivot_index,
                               void* stream) {
  NNB_TRY(require_device());
  if (n < 0) return fail(NNB_ERR_SHAPE, "direct_inverse_oracle: matrix must be square");
  if (n == 0) return 0;
  cudaStream_t s = resolve(stream);
  const size_t cnt = (size_t)((cplx ? 2 : 1) * n * n);
  In m;
  NNB_TRY(m.stage(M, cnt, s));
  DevBuf fro;
  NNB_TRY(fro.alloc(sizeof(double), s));
  NNB_TRY(sumsq(m.d, (int64_t)cnt, fro.as<double>(), s));
  double ss = 0.0;
  NNB_CUDA(cudaMemcpyAsync(&ss, fro.p, sizeof(double), cudaMemcpyDeviceToHost, s));
  NNB_CUDA(cudaStreamSynchronize(s));
  Out o;
  NNB_TRY(o.prepare(out, cnt, s));
  int singular = -1;
  NNB_TRY(direct_inverse(m.d, n, cplx, 1e-13 * std::sqrt(ss), o.d, &singular, s));
  if (singular >= 0) {
    if (pivot_index) *pivot_index = singular;
    return fail(NNB_ERR_SINGULAR, "direct_inverse_oracle: singular pivot at index " + std::to_string(singular));
  }
  NNB_TRY(o.finish(s));
  return sync(s);
}

int nnb_direct_inverse_d(const double* M, int64_t n, double* out, int32_t* pivot_index, void* stream) {
  return direct_inverse_call(M, n, 0, out, pivot_index, stream);
}

int nnb_direct_inverse_z(const double* M, int64_t n, double* out, int32_t* pivot_index, void* stream) {
  return direct_inverse_call(M, n, 1, out, pivot_index, stream);
}

static int transpose_call(const double* M, int64_t rows, int64_t cols, int cplx, double* out, void* stream) {
  NNB_TRY(require_device());
  if (rows < 0 || cols < 0) return fail(NNB_ERR_SHAPE, "conjugate_transpose: negative shape");
  if (M == out && rows * cols) return fail(NNB_ERR_DOMAIN, "conjugate_transpose: out must not alias M");
  cudaStream_t s = resolve(stream);
  const size_t cnt = (size_t)((cplx ? 2 : 1) * rows * cols);
  In m;
  NNB_TRY(m.stage(M, cnt, s));
  Out o;
  NNB_TRY(o.prepare(out, cnt, s));
  NNB_TRY(transpose(m.d, rows, cols, cplx, o.d, s));
  NNB_TRY(o.finish(s));
  return sync(s);
}

int nnb_transpose_d(const double* M, int64_t rows, int64_t cols, double* out, void* stream) {
  return transpose_call(M, rows, cols, 0, out, stream);
}

int nnb_conj_transpose_z(const double* M, int64_t rows, int64_t cols, double* out, void* stream) {
  return transpose_call(M, rows, cols, 1, out, stream);
}

static int frob(const double* M, int64_t count, double* out, cudaStream_t s) {
  In m;
  NNB_TRY(m.stage(M, (size_t)count, s));
  DevBuf r;
  NNB_TRY(r.alloc(sizeof(double), s));
  NNB_TRY(sumsq(m.d, count, r.as<double>(), s));
  double h = 0;
  NNB_CUDA(cudaMemcpyAsync(&h, r.p, sizeof(double), cudaMemcpyDeviceToHost, s));
  NNB_TRY(sync(s));
  *out = std::sqrt(h);
  return 0;
}

int nnb_frobenius_d(const double* M, int64_t count, double* out, void* stream) {
  NNB_TRY(require_device());
  return frob(M, count, out, resolve(stream));
}
int nnb_frobenius_z(const double* M, int64_t count, double* out, void* stream) {
  NNB_TRY(require_device());
  return frob(M, 2 * count, out, resolve(stream));
}

int nnb_trace_z(const double* M, int64_t n, double* out2, void* stream) {
  NNB_TRY(require_device());
  cudaStream_t s = resolve(stream);
  In m;
  NNB_TRY(m.stage(M, (size_t)(2 * n * n), s));
  DevBuf r;
  NNB_TRY(r.alloc(2 * sizeof(double), s));
  NNB_TRY(trace_dev(m.d, n, n, 2, r.as<double>(), s));
  NNB_CUDA(cudaMemcpyAsync(out2, r.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  return sync(s);
}

int nnb_x0_d(const double* A, int64_t n, int32_t x0_kind, double x0_scale, double* X0,
             void* stream) {
  NNB_TRY(require_device());
  cudaStream_t s = resolve(stream);
  DMat a, x;
  NNB_TRY(a.load(A, n, n, n, s));
  NNB_TRY(x.alloc(n, n, s));
  NNB_TRY(x0_build(a.d, a.ld, n, x0_kind, x0_scale, x.d, x.ld, s));
  NNB_TRY(x.store(X0, n, s));
  return sync(s);
}

// ---------------------------------------------------------------- the chain
int nnb_nn_chain_d(const double* A, int64_t n, const double* X0, const nnb_chain_config* cfg,
                   double* X_out, double* eps_hist, nnb_chain_result* result, void* stream) {
  NNB_TRY(require_device());
  if (n < 1) return fail(NNB_ERR_SHAPE, "nn chain: matrix must be square and non-empty");
  ChainCfg c;
  NNB_TRY(chain_cfg(cfg, &c));
  cudaStream_t s = resolve(stream);
  const bool host_a = !is_device_ptr(A), host_out = X_out && !is_device_ptr(X_out);
  if ((host_a || host_out) && n >= kStreamMinN && arith() != 1)
    return chain_d_streamed(A, n, X0, cfg, c, X_out, eps_hist, result, s);
  DMat a;
  NNB_TRY(a.load(A, n, n, n, s));
  DMat x;  // working X with A's leading dimension: the caller's device X_out when it fits
  x.rows = x.cols = n;
  x.ld = a.ld;
  const bool direct = X_out && !host_out && a.ld == n && !(reinterpret_cast<uintptr_t>(X_out) & 15) &&
                      X_out != A && X_out != X0;
  if (direct) {
    x.d = X_out;
  } else {
    NNB_TRY(x.own.alloc(sizeof(double) * n * a.ld, s));
    x.d = x.own.as<double>();
  }
  if (cfg->x0_kind == NNB_X0_GIVEN) {
    if (!X0) return fail(NNB_ERR_DOMAIN, "nn chain: X0 required for NNB_X0_GIVEN");
    NNB_CUDA(cudaMemcpy2DAsync(x.d, x.ld * 8, X0, n * 8, n * 8, n, cudaMemcpyDefault, s));
  } else {
    NNB_TRY(x0_build(a.d, a.ld, n, cfg->x0_kind, cfg->x0_scale, x.d, x.ld, s));
  }
  NNB_TRY(symmetric_check(cfg, a.d, x.d, n, a.ld, s));
  ChainOut o;
  const int st = chain_real(a.d, n, a.ld, x.d, c, eps_hist, &o, s);
  fill_result(result, o);
  if (st != 0 && st != NNB_ERR_DIVERGENCE && st != NNB_ERR_DOMAIN) return st;
  if (!direct) {
    NNB_TRY(x.store(X_out, n, s));
    NNB_TRY(sync(s));
  }
  return st;
}

int nnb_nn_chain_z(const double* A, int64_t n, const double* X0, const nnb_chain_config* cfg,
                   double* X_out, double* eps_hist, nnb_chain_result* result, void* stream) {
  NNB_TRY(require_device());
  if (n < 1) return fail(NNB_ERR_SHAPE, "nn chain: matrix must be square and non-empty");
  ChainCfg c;
  NNB_TRY(chain_cfg(cfg, &c));
  if (cfg->order == NNB_ORDER_SYMMETRIC)
    return fail(NNB_ERR_DOMAIN, "nn chain (complex): the symmetric order is real-only");
  cudaStream_t s = resolve(stream);
  ZMat a, x;
  NNB_TRY(a.load(A, n, n, s));
  if (cfg->x0_kind == NNB_X0_GIVEN) {
    if (!X0) return fail(NNB_ERR_DOMAIN, "nn chain: X0 required for NNB_X0_GIVEN");
    NNB_TRY(x.load(X0, n, n, s));
  } else if (cfg->x0_kind == NNB_X0_SCALED_IDENTITY) {
    NNB_TRY(x.alloc(n, n, s));
    NNB_TRY(fill_identity(x.re, n, x.ld, cfg->x0_scale, s));
  } else {
    return fail(NNB_ERR_DOMAIN, "nn chain (complex): X0 must be given or a scaled identity");
  }
  ChainOut o;
  const int st = chain_complex(a.re, a.im, n, a.ld, x.re, x.im, c, eps_hist, &o, s);
  fill_result(result, o);
  if (st != 0 && st != NNB_ERR_DIVERGENCE && st != NNB_ERR_DOMAIN) return st;
  NNB_TRY(x.store(X_out, s));
  return st;
}

int nnb_residual_eps_d(const double* X, const double* A, int64_t n, double* eps, void* stream) {
  nnb_chain_config cfg{0, 0, 0.0, NNB_ORDER_REFERENCE, NNB_X0_GIVEN, 0.0, 1};
  nnb_chain_result r{};
  double h[1] = {0.0};
  // X_out must be distinct from the inputs; a residual-only chain leaves X unchanged
  NNB_TRY(require_device());
  cudaStream_t s = resolve(stream);
  DevBuf xo;
  NNB_TRY(xo.alloc(sizeof(double) * std::max<int64_t>(1, n * n), s));
  const int st = nnb_nn_chain_d(A, n, X, &cfg, xo.as<double>(), h, &r, stream);
  if (st == 0) *eps = h[0];
  return st;
}

int nnb_residual_eps_z(const double* X, const double* A, int64_t n, double* eps, void* stream) {
  nnb_chain_config cfg{0, 0, 0.0, NNB_ORDER_REFERENCE, NNB_X0_GIVEN, 0.0, 1};
  nnb_chain_result r{};
  double h[1] = {0.0};
  NNB_TRY(require_device());
  cudaStream_t s = resolve(stream);
  DevBuf xo;
  NNB_TRY(xo.alloc(sizeof(double) * std::max<int64_t>(1, 2 * n * n), s));
  const int st = nnb_nn_chain_z(A, n, X, &cfg, xo.as<double>(), h, &r, stream);
  if (st == 0) *eps = h[0];
  return st;
}

int nnb_nn_step_d(const double* phi, const double* w, int64_t n, int32_t depth, double* out,
                  void* stream) {
  NNB_TRY(require_device());
  cudaStream_t s = resolve(stream);
  if (depth == 0) {
    NNB_CUDA(cudaMemcpyAsync(out, phi, sizeof(double) * n * n, cudaMemcpyDefault, s));
    return sync(s);
  }
  nnb_chain_config cfg{depth, 1, 0.0, NNB_ORDER_REFERENCE, NNB_X0_GIVEN, 0.0, 0};
  nnb_chain_result r{};
  const int st = nnb_nn_chain_d(w, n, phi, &cfg, out, nullptr, &r, stream);
  if (st == NNB_ERR_DIVERGENCE || st == NNB_ERR_DOMAIN)
    return fail(NNB_ERR_DOMAIN, "nn_step: matmul produced a non-finite entry");
  return st;
}

int nnb_nn_step_z(const double* phi, const double* w, int64_t n, int32_t depth, double* out,
                  void* stream) {
  NNB_TRY(require_device());
  cudaStream_t s = resolve(stream);
  if (depth == 0) {
    NNB_CUDA(cudaMemcpyAsync(out, phi, sizeof(double) * 2 * n * n, cudaMemcpyDefault, s));
    return sync(s);
  }
  nnb_chain_config cfg{depth, 1, 0.0, NNB_ORDER_REFERENCE, NNB_X0_GIVEN, 0.0, 0};
  nnb_chain_result r{};
  const int st = nnb_nn_chain_z(w, n, phi, &cfg, out, nullptr, &r, stream);
  if (st == NNB_ERR_DIVERGENCE || st == NNB_ERR_DOMAIN)
    return fail(NNB_ERR_DOMAIN, "nn_step: matmul produced a non-finite entry");
  return st;
}

int nnb_ns_sum_d(const double* phi0, const double* w, int64_t n, int64_t order, double* out,
                 double* products_out, void* stream) {
  NNB_TRY(require_device());
  cudaStream_t s = resolve(stream);
  if (products_out) *products_out = 0;
  if (order == 0) {
    NNB_CUDA(cudaMemcpyAsync(out, phi0, sizeof(double) * n * n, cudaMemcpyDefault, s));
    return sync(s);
  }
  DMat p, wm, o;
  NNB_TRY(p.load(phi0, n, n, n, s, false));
  NNB_TRY(wm.load(w, n, n, n, s, false));
  NNB_TRY(o.alloc(n, n, s));
  bool ident = false;
  NNB_TRY(is_identity_dev(p.d, nullptr, n, p.ld, &ident, s));
  NNB_TRY(ns_sum_dev(p.d, nullptr, wm.d, nullptr, n, p.ld, order, ident, o.d, nullptr,
                     products_out, s));
  NNB_TRY(o.store(out, n, s));
  return sync(s);
}

int nnb_ns_sum_z(const double* phi0, const double* w, int64_t n, int64_t order, double* out,
                 double* products_out, void* stream) {
  NNB_TRY(require_device());
  cudaStream_t s = resolve(stream);
  if (products_out) *products_out = 0;
  if (order == 0) {
    NNB_CUDA(cudaMemcpyAsync(out, phi0, sizeof(double) * 2 * n * n, cudaMemcpyDefault, s));
    return sync(s);
  }
  ZMat p, wm, o;
  NNB_TRY(p.load(phi0, n, n, s));
  NNB_TRY(wm.load(w, n, n, s));
  NNB_TRY(o.alloc(n, n, s));
  bool ident = false;
  NNB_TRY(is_identity_dev(p.re, p.im, n, p.ld, &ident, s));
  NNB_TRY(ns_sum_dev(p.re, p.im, wm.re, wm.im, n, p.ld, order, ident, o.re, o.im, products_out, s));
  return o.store(out, s);
}

// ---------------------------------------------------------------- product-form schedules
// (the same fused GEMM, different schedules)
namespace {
enum class Sched { Factorized, Ladder, Explicit };

int sched_d(Sched which, const double* phi0, const double* w, int64_t n, int64_t a, int64_t b, double* out,
            double* products, void* stream) {
  NNB_TRY(require_device());
  cudaStream_t s = resolve(stream);
  DMat p, wm, o;
  NNB_TRY(p.load(phi0, n, n, n, s, false));
  if (w) NNB_TRY(wm.load(w, n, n, n, s, false));
  NNB_TRY(o.alloc(n, n, s));
  bool ident = false;
  if (which != Sched::Ladder) NNB_TRY(is_identity_dev(p.d, nullptr, n, p.ld, &ident, s));
  switch (which) {
    case Sched::Factorized:
      NNB_TRY(ns_factorized_dev(p.d, nullptr, wm.d, nullptr, n, p.ld, (int)a, ident, o.d, nullptr, products, s));
      break;
    case Sched::Ladder:
      NNB_TRY(power_ladder_dev(p.d, nullptr, n, p.ld, (uint64_t)a, o.d, nullptr, products, s));
      break;
    default:
      NNB_TRY(nn_explicit_dev(p.d, nullptr, wm.d, nullptr, n, p.ld, (int)a, (int)b, ident, o.d, nullptr, products, s));
  }
  NNB_TRY(o.store(out, n, s));
  return sync(s);
}

int sched_z(Sched which, const double* phi0, const double* w, int64_t n, int64_t a, int64_t b, double* out,
            double* products, void* stream) {
  NNB_TRY(require_device());
  cudaStream_t s = resolve(stream);
  ZMat p, wm, o;
  NNB_TRY(p.load(phi0, n, n, s));
  if (w) NNB_TRY(wm.load(w, n, n, s));
  NNB_TRY(o.alloc(n, n, s));
  bool ident = false;
  if (which != Sched::Ladder) NNB_TRY(is_identity_dev(p.re, p.im, n, p.ld, &ident, s));
  switch (which) {
    case Sched::Factorized:
      NNB_TRY(ns_factorized_dev(p.re, p.im, wm.re, wm.im, n, p.ld, (int)a, ident, o.re, o.im, products, s));
      break;
    case Sched::Ladder:
      NNB_TRY(power_ladder_dev(p.re, p.im, n, p.ld, (uint64_t)a, o.re, o.im, products, s));
      break;
    default:
      NNB_TRY(nn_explicit_dev(p.re, p.im, wm.re, wm.im, n, p.ld, (int)a, (int)b, ident, o.re, o.im, products, s));
  }
  return o.store(out, s);
}

int factor_count(int64_t gamma, int64_t* s_factors) {
  if (gamma < 1 || ((gamma + 1) & gamma) != 0)
    return fail(NNB_ERR_PLAN, "FactorizedPlan: order + 1 must be a power of two");
  *s_factors = 0;
  for (int64_t g = gamma + 1; g > 1; g >>= 1) ++*s_factors;
  return 0;
}

int explicit_budget(int64_t nests_i, int64_t depth_L) {
  // (L+1)^i must stay below 2^62 (proj/src/solver.cpp:182-185)
  long double v = 1.0L;
  for (int64_t i = 0; i < nests_i; ++i) {
    v *= static_cast<long double>(depth_L + 1);
    if (v > 4611686018427387904.0L) return fail(NNB_ERR_BUDGET, "nn_explicit: inner power (L+1)^i is not representable");
  }
  return 0;
}
}  // namespace

int nnb_ns_factorized_d(const double* phi0, const double* w, int64_t n, int64_t gamma, double* out,
                        double* products_out, void* stream) {
  int64_t sf = 0;
  NNB_TRY(factor_count(gamma, &sf));
  return sched_d(Sched::Factorized, phi0, w, n, sf, 0, out, products_out, stream);
}
int nnb_ns_factorized_z(const double* phi0, const double* w, int64_t n, int64_t gamma, double* out,
                        double* products_out, void* stream) {
  int64_t sf = 0;
  NNB_TRY(factor_count(gamma, &sf));
  return sched_z(Sched::Factorized, phi0, w, n, sf, 0, out, products_out, stream);
}
int nnb_power_ladder_d(const double* p, int64_t n, uint64_t exponent, double* out, double* products_out,
                       void* stream) {
  return sched_d(Sched::Ladder, p, nullptr, n, (int64_t)exponent, 0, out, products_out, stream);
}
int nnb_power_ladder_z(const double* p, int64_t n, uint64_t exponent, double* out, double* products_out,
                       void* stream) {
  return sched_z(Sched::Ladder, p, nullptr, n, (int64_t)exponent, 0, out, products_out, stream);
}
int nnb_nn_explicit_d(const double* phi0, const double* w, int64_t n, int64_t nests_i, int64_t depth_L,
                      double* out, double* products_out, void* stream) {
  NNB_TRY(explicit_budget(nests_i, depth_L));
  return sched_d(Sched::Explicit, phi0, w, n, nests_i, depth_L, out, products_out, stream);
}
int nnb_nn_explicit_z(const double* phi0, const double* w, int64_t n, int64_t nests_i, int64_t depth_L,
                      double* out, double* products_out, void* stream) {
  NNB_TRY(explicit_budget(nests_i, depth_L));
  return sched_z(Sched::Explicit, phi0, w, n, nests_i, depth_L, out, products_out, stream);
}

// ---------------------------------------------------------------- batched
// Host-to-host calls stream the batch through the device in chunks on three
// rotating lanes (stream per lane): H2D of chunk i+1, the kernel on chunk i
// and D2H of chunk i-1 overlap, so the PCIe traffic in both directions (full
// duplex) hides behind itself and the compute instead of adding up.
// 32 MB in + 32 MB out per chunk on 4 lanes: PCIe in and out overlap the DMMA
// work and each other; smaller chunks shorten the pipeline's fill and drain.
static constexpr int64_t kChunkSystems = 8192;

static int batched_pipelined(const double* A, int64_t batch, int p, int iters, int ns_order, double* X_out,
                             double* eps_last, cudaStream_t s) {
  constexpr int kLanes = 4;
  const size_t sys_doubles = 2 * 256;
  static thread_local cudaStream_t lanes[kLanes] = {};
  for (auto& l : lanes)
    if (!l) NNB_CUDA(cudaStreamCreateWithFlags(&l, cudaStreamNonBlocking));
  DevBuf buf;
  const size_t per_lane = kChunkSystems * sys_doubles * 2 + kChunkSystems;  // A, X, eps
  NNB_TRY(buf.alloc(sizeof(double) * per_lane * kLanes, s));
  cudaEvent_t start, done[kLanes];
  NNB_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  for (auto& d : done) NNB_CUDA(cudaEventCreateWithFlags(&d, cudaEventDisableTiming));
  NNB_CUDA(cudaEventRecord(start, s));  // buffers are allocated in stream order on s
  for (auto& l : lanes) NNB_CUDA(cudaStreamWaitEvent(l, start, 0));
  int st = 0;
  for (int64_t c0 = 0, i = 0; c0 < batch && st == 0; c0 += kChunkSystems, ++i) {
    const int64_t nb = std::min<int64_t>(kChunkSystems, batch - c0);
    const int lane = static_cast<int>(i % kLanes);
    cudaStream_t ls = lanes[lane];
    double* da = buf.as<double>() + lane * per_lane;
    double* dx = da + kChunkSystems * sys_doubles;
    double* de = dx + kChunkSystems * sys_doubles;
    NNB_CUDA(cudaMemcpyAsync(da, A + c0 * sys_doubles, sizeof(double) * nb * sys_doubles,
                             cudaMemcpyHostToDevice, ls));
    st = batched_nn_z16(da, nb, p, iters, ns_order, dx, eps_last ? de : nullptr, ls);
    NNB_CUDA(cudaMemcpyAsync(X_out + c0 * sys_doubles, dx, sizeof(double) * nb * sys_doubles,
                             cudaMemcpyDeviceToHost, ls));
    if (eps_last)
      NNB_CUDA(cudaMemcpyAsync(eps_last + c0, de, sizeof(double) * nb, cudaMemcpyDeviceToHost, ls));
  }
  for (int l = 0; l < kLanes; ++l) {
    NNB_CUDA(cudaEventRecord(done[l], lanes[l]));
    NNB_CUDA(cudaStreamWaitEvent(s, done[l], 0));  // buffer release is ordered after every lane
  }
  buf.release();
  NNB_CUDA(cudaStreamSynchronize(s));
  cudaEventDestroy(start);
  for (auto& d : done) cudaEventDestroy(d);
  return st;
}

static int batched(const double* A, int64_t batch, int32_t n, int p, int iters, int ns_order,
                   double* X_out, double* eps_last, void* stream) {
  NNB_TRY(require_device());
  if (n != 8 && n != 16 && n != 24 && n != 32)
    return fail(NNB_ERR_SHAPE, "batched: n must be 8, 16, 24 or 32 (users of a massive-MIMO uplink)");
  if (batch < 0) return fail(NNB_ERR_SHAPE, "batched: negative batch");
  cudaStream_t s = resolve(stream);
  if (n != 16) {  // batched_generic.cu
    const size_t cnt = (size_t)batch * 2 * n * n;
    In a;
    NNB_TRY(a.stage(A, cnt, s));
    Out x, e;
    NNB_TRY(x.prepare(X_out, cnt, s));
    if (eps_last) NNB_TRY(e.prepare(eps_last, (size_t)batch, s));
    NNB_TRY(batched_nn_gen(a.d, batch, n, p, iters, ns_order, x.d, eps_last ? e.d : nullptr, s));
    NNB_TRY(x.finish(s));
    if (eps_last) NNB_TRY(e.finish(s));
    return 0;
  }
  const size_t cnt = (size_t)batch * 2 * 256;
  const bool host_in = !is_device_ptr(A), host_out = !is_device_ptr(X_out) ||
                                                     (eps_last && !is_device_ptr(eps_last));
  if (host_in && host_out && batch > 2 * kChunkSystems)
    return batched_pipelined(A, batch, p, iters, ns_order, X_out, eps_last, s);
  In a;
  NNB_TRY(a.stage(A, cnt, s));
  Out x, e;
  NNB_TRY(x.prepare(X_out, cnt, s));
  if (eps_last) NNB_TRY(e.prepare(eps_last, (size_t)batch, s));
  NNB_TRY(batched_nn_z16(a.d, batch, p, iters, ns_order, x.d, eps_last ? e.d : nullptr, s));
  NNB_TRY(x.finish(s));
  if (eps_last) NNB_TRY(e.finish(s));
  return 0;
}

int nnb_nn_batched_z(const double* A, int64_t batch, int32_t n, int32_t p, int32_t iters,
                     double* X_out, double* eps_last, void* stream) {
  if (p < 1 || p > 4) return fail(NNB_ERR_DOMAIN, "batched: depth p must be in 1..4");
  if (iters < 0) return fail(NNB_ERR_DOMAIN, "batched: iters must be >= 0");
  return batched(A, batch, n, p, iters, -1, X_out, eps_last, stream);
}

int nnb_mimo_detect_z(const double* H, const double* y, int64_t batch, int32_t antennas, int32_t users,
                      double sigma2, int32_t p, int32_t iters, double* xhat_out, double* X_out, double* eps_last,
                      void* stream) {
  NNB_TRY(require_device());
  if (users != 8 && users != 16 && users != 24 && users != 32)
    return fail(NNB_ERR_SHAPE, "mimo detect: users must be 8, 16, 24 or 32");
  if (antennas < 4 || antennas % 4) return fail(NNB_ERR_SHAPE, "mimo detect: antennas must be a positive multiple of 4");
  if (p < 1 || p > 4 || iters < 0) return fail(NNB_ERR_DOMAIN, "mimo detect: depth p in 1..4, iters >= 0");
  if (batch < 0) return fail(NNB_ERR_SHAPE, "mimo detect: negative batch");
  cudaStream_t s = resolve(stream);
  In h, yy;
  NNB_TRY(h.stage(H, (size_t)batch * antennas * users * 2, s));
  NNB_TRY(yy.stage(y, (size_t)batch * antennas * 2, s));
  Out xh, x, e;
  NNB_TRY(xh.prepare(xhat_out, (size_t)batch * users * 2, s));
  if (X_out) NNB_TRY(x.prepare(X_out, (size_t)batch * 2 * users * users, s));
  if (eps_last) NNB_TRY(e.prepare(eps_last, (size_t)batch, s));
  if (users == 16)
    NNB_TRY(mimo_detect_z16(h.d, yy.d, batch, antennas, sigma2, p, iters, xh.d, X_out ? x.d : nullptr,
                            eps_last ? e.d : nullptr, s));
  else
    NNB_TRY(mimo_detect_gen(h.d, yy.d, batch, antennas, users, sigma2, p, iters, xh.d, X_out ? x.d : nullptr,
                            eps_last ? e.d : nullptr, s));
  NNB_TRY(xh.finish(s));
  if (X_out) NNB_TRY(x.finish(s));
  if (eps_last) NNB_TRY(e.finish(s));
  return 0;
}

int nnb_ns_batched_z(const double* A, int64_t batch, int32_t n, int32_t order, double* X_out,
                     void* stream) {
  if (order < 0) return fail(NNB_ERR_DOMAIN, "batched ns: order must be >= 0");
  return batched(A, batch, n, 1, 0, order, X_out, nullptr, stream);
}

// ---------------------------------------------------------------- sparse
static int stage_csr(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n,
                     int64_t nnz, cudaStream_t s, DevBuf& own, const int64_t** rp,
                     const int32_t** ci, const double** v) {
  const bool dev = is_device_ptr(row_ptr) && is_device_ptr(col) && is_device_ptr(val);
  if (dev) {
    *rp = row_ptr; *ci = col; *v = val;
    return 0;
  }
  const size_t b_rp = sizeof(int64_t) * (n + 1), b_v = sizeof(double) * nnz,
               b_c = sizeof(int32_t) * nnz;
  NNB_TRY(own.alloc(b_rp + b_v + b_c + 64, s));
  char* base = own.as<char>();
  NNB_CUDA(cudaMemcpyAsync(base, row_ptr, b_rp, cudaMemcpyDefault, s));
  NNB_CUDA(cudaMemcpyAsync(base + b_rp, val, b_v, cudaMemcpyDefault, s));
  NNB_CUDA(cudaMemcpyAsync(base + b_rp + b_v, col, b_c, cudaMemcpyDefault, s));
  *rp = reinterpret_cast<const int64_t*>(base);
  *v = reinterpret_cast<const double*>(base + b_rp);
  *ci = reinterpret_cast<const int32_t*>(base + b_rp + b_v);
  return 0;
}

int nnb_spmv_block_d(const int64_t* row_ptr, const int32_t* col, const double* val, int64_t n,
                     int64_t nnz, const double* X, int64_t k, double* Y, void* stream) {
  NNB_TRY(require_device());
  cudaStream_t s = resolve(stream);
  DevBuf csr;
  const int64_t* rp; const int32_t* ci; const double* v;
  NNB_TRY(stage_csr(row_ptr, col, val, n, nnz, s, csr, &rp, &ci, &v));
  In x;
  NNB_TRY(x.stage(X, (size_t)(n * k), s));
  Out y;
  NNB_TRY(y.prepare(Y, (size_t)(n * k), s));
  NNB_TRY(spmv_csr(rp, ci, v, n, x.d, k, y.d, s));
  NNB_TRY(y.finish(s));
  return sync(s);
}

int nnb_sparse_last_bytes_per_nnz(void) { return sparse_bytes_per_nnz(); }
int64_t nnb_sparse_last_matrix_bytes(void) { return sparse_matrix_bytes(); }
const char* nnb_sparse_last_format(void) { return sparse_format(); }

int nnb_sparse_factorized_d(const int64_t* row_ptr, const int32_t* col, const double* val,
                            int64_t n, int64_t nnz, const double* B, int64_t k, int64_t gamma,
                            double theta, double* X_out, int64_t* spmv_count_out,
                            int32_t* fail_factor_out, void* stream) {
  NNB_TRY(require_device());
  // validation order of proj/src/factorized.cpp:104-115
  if (gamma < 1 || ((gamma + 1) & gamma) != 0)
    return fail(NNB_ERR_PLAN, "solve_sparse_factorized: order + 1 must be a power of two");
  if (gamma > (int64_t(1) << 30))
    return fail(NNB_ERR_BUDGET, "solve_sparse_factorized: order too large to apply");
  int s_factors = 0;
  for (int64_t g = gamma + 1; g > 1; g >>= 1) ++s_factors;
  cudaStream_t s = resolve(stream);
  DevBuf csr;
  const int64_t* rp; const int32_t* ci; const double* v;
  NNB_TRY(stage_csr(row_ptr, col, val, n, nnz, s, csr, &rp, &ci, &v));
  In b;
  NNB_TRY(b.stage(B, (size_t)(n * k), s));
  Out x;
  NNB_TRY(x.prepare(X_out, (size_t)(n * k), s));
  int ff = -1;
  const int st = sparse_factorized(rp, ci, v, n, b.d, k, s_factors, theta, x.d, &ff, s);
  if (fail_factor_out) *fail_factor_out = ff;
  if (st) return st;
  if (spmv_count_out) *spmv_count_out = gamma * k;
  return x.finish(s);
}

}  // extern "C"
