// FP64 pipe peak microbenchmark for B200 (sm_100a).
// Measures: DFMA (CUDA-core FP64) throughput and DMMA (mma.sync f64 m8n8k4,
// the FP64 tensor path) throughput, full chip, CUDA-event timed.
// These numbers are the roofline denominators for the dense NN chain.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int ILP>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

template <int ILP>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
  double c[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* d; CK(cudaMalloc(&d, 64));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int threads : {256, 512, 1024}) {
    for (int bps : {1, 2}) {
      int blocks = sms * bps;
      dfma_loop<8><<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dfma_loop<8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * (double)iters * threads * blocks;
      printf("DFMA threads=%d blocks=%d: %.2f TFLOP/s (%.3f ms)\n", threads, blocks, flops / ms / 1e9, ms);
    }
  }
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps;
      dmma_loop<8><<<blocks, threads>>>(d, 100);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_loop<8><<<blocks, threads>>>(d, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 8 * (double)iters * (threads / 32) * blocks;
      printf("DMMA threads=%d blocks=%d: %.2f TFLOP/s (%.3f ms)\n", threads, blocks, flops / ms / 1e9, ms);
    }
  }
  return 0;
}
