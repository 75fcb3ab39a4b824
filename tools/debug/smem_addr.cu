// Where does each co-resident CTA's dynamic shared window start?
#include <cstdio>
#include <cstdint>
__global__ void probe(int* out) {
  extern __shared__ uint8_t sm[];
  unsigned smid; asm("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = smid;
    out[blockIdx.x * 2 + 1] = (int)__cvta_generic_to_shared(sm);
  }
  // keep CTAs resident together
  long long t0 = clock64(); while (clock64() - t0 < 2000000) {}
}
int main() {
  for (int bytes : {66816, 86816, 40000}) {
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    int* d; cudaMalloc(&d, 148 * 8 * 8);
    probe<<<148 * 3, 160, bytes>>>(d);
    int h[148 * 3 * 2]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("bytes=%d:", bytes);
    int shown = 0;
    for (int b = 0; b < 148 * 3 && shown < 12; ++b) if (h[2*b] == 0) { printf(" cta%d@%d(mod1024=%d)", b, h[2*b+1], h[2*b+1] % 1024); ++shown; }
    printf("\n");
    cudaFree(d);
  }
}
