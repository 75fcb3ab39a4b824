// Shared device helpers for the sm_100a Nested Neumann kernels:
// mbarrier / TMA (cp.async.bulk.tensor) wrappers and the FP64 tensor-core
// MMA (mma.sync m8n8k4 .f64, SASS DMMA.8x8x4).  sm_100a has no tcgen05 f64
// kind (ptxas: "Unknown modifier '.kind::f64'"), so DMMA is the FP64 tensor
// path on B200; measured chip peak 37.2 TFLOP/s (profiles/r01_fp64_peak.txt).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <ctime>

namespace nnb {

// A/B measurement knobs (NNB_GEMM_CFG, NNB_SPARSE_*, NNB_SMALL_CHAIN_MAX, ...).
// The product path reads no environment variable unless NNB_DEBUG=1 is set, so
// a stray variable cannot change the benchmarked path; with NNB_DEBUG=1 the
// named variable overrides the built-in choice.  (NNB_ARITHMETIC is not a
// knob: it is the documented switch of nnb_set_arithmetic.)
inline const char* debug_env(const char* name) {
  static const bool on = [] {
    const char* e = std::getenv("NNB_DEBUG");
    return e && e[0] == '1';
  }();
  return on ? std::getenv(name) : nullptr;
}

// NNB_DEBUG=1 NNB_TRACE=1: timing events at labelled points on any stream; trace_dump()
// synchronizes and prints each point's time since the first one to stderr (the e2e
// copy/compute timeline: tools/e2e_timeline.py)
struct TraceMark {
  char label[24];
  cudaEvent_t ev;
  double host_ms;  // host clock at the mark (a device time below it = the GPU waited for the host)
};
inline double trace_host_ms() {
  timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec * 1e3 + t.tv_nsec * 1e-6;
}
inline TraceMark* trace_marks(int** count) {
  static TraceMark marks[512];
  static int n = 0;
  *count = &n;
  return marks;
}
inline bool trace_on() {
  static const bool on = debug_env("NNB_TRACE") != nullptr;
  return on;
}
inline void trace_mark(cudaStream_t s, const char* label, int idx = -1) {
  if (!trace_on()) return;
  int* n;
  TraceMark* m = trace_marks(&n);
  if (*n >= 512) return;
  TraceMark& t = m[*n];
  if (cudaEventCreate(&t.ev) != cudaSuccess) return;
  int i = 0;
  for (; label[i] && i < 16; ++i) t.label[i] = label[i];
  if (idx >= 0) {
    t.label[i++] = static_cast<char>('0' + idx / 10 % 10);
    t.label[i++] = static_cast<char>('0' + idx % 10);
  }
  t.label[i] = 0;
  t.host_ms = trace_host_ms();
  cudaEventRecord(t.ev, s);
  ++*n;
}
inline void trace_reset() {
  int* n;
  TraceMark* m = trace_marks(&n);
  for (int i = 0; i < *n; ++i) cudaEventDestroy(m[i].ev);
  *n = 0;
}
void trace_dump();  // capi.cu

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier -------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// Orders this thread's prior generic-proxy shared-memory accesses before
// later async-proxy (TMA) accesses.  Consumers that read a stage with plain
// ld.shared must execute it before releasing the slot to the TMA producer:
// without it ptxas schedules the release above the last fragment loads and
// the next TMA fill races them (seen as corrupted rows with >=2 CTAs/SM).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---- TMA ------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// 2D tile load global -> shared, completion signalled on `bar` (complete_tx).
// c0 = innermost (column) coordinate, c1 = row coordinate, in elements.
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// ---- FP64 tensor core -----------------------------------------------------
// D(8x8) += A(8x4, row) * B(4x8, col).  Fragment ownership (lane = l):
//   a = A[l>>2][l&3], b = B[l&3][l>>2], {d0,d1} = D[l>>2][2*(l&3) + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace nnb
