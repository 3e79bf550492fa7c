// Kernel-boundary gap probe: empty kernels bracketing a sleep kernel, timed with globaltimer.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void stamp(unsigned long long* t, int i) {
  if (threadIdx.x == 0 && blockIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t[i]));
}
__global__ void work(unsigned long long* t, int i, int ns, size_t) {
  extern __shared__ char smem[];
  unsigned long long a;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a));
  if (threadIdx.x == 0) { atomicMin(&t[i], a); smem[0] = 1; }
  __nanosleep(ns);
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a));
  if (threadIdx.x == 0) atomicMax(&t[i + 1], a);
}
int main() {
  unsigned long long* t;
  cudaMalloc(&t, 64 * 8);
  for (size_t smem : {0ul, 100000ul, 200000ul}) {
    cudaFuncSetAttribute(work, cudaFuncAttributeMaxDynamicSharedMemorySize, 220000);
    unsigned long long h[8] = {0, ~0ull, 0, 0, 0, 0, 0, 0};
    cudaMemcpy(t, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    stamp<<<1, 32>>>(t, 0);
    cudaEventRecord(a);
    work<<<296, 160, smem>>>(t, 1, 50000, smem);
    cudaEventRecord(b);
    stamp<<<1, 32>>>(t, 3);
    cudaDeviceSynchronize();
    cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("smem %zu: stamp->first CTA %.1f us, CTA span %.1f us, last CTA->stamp %.1f us, event %.1f us\\n", smem,
           (h[1] - h[0]) / 1e3, (h[2] - h[1]) / 1e3, (h[3] - h[2]) / 1e3, ms * 1e3);
  }
  return 0;
}
