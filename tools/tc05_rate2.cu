// tcgen05.mma rate with NACC independent accumulators (round-robin D addresses): is the small-N
// ~51-cycle cost a dependent-accumulation latency or a per-instruction floor?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc05_rate2 tools/tc05_rate2.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t make_idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <int N, bool TS, int NACC>
__global__ void rate(long long* out, int iters) {
  __shared__ __align__(1024) uint8_t sB[256 * 16 * 2];
  __shared__ __align__(1024) uint8_t sA[128 * 16 * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t taddr_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (int)sizeof(sB) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sB)[i] = 0x3c003c00u;
  for (int i = tid; i < (int)sizeof(sA) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sA)[i] = 0x3c003c00u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&taddr_s)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = taddr_s;
  if (tid == 0) {
    const uint32_t idesc = make_idesc(N);
    const uint64_t bd = make_desc(smem_u32(sB), 128, 256);
    const uint64_t ad = make_desc(smem_u32(sA), 128, 256);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (TS)
        asm volatile("{.reg .pred p; setp.ne.b32 p, %3, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %4, p;}"
                     ::"r"(t + (uint32_t)((i % NACC) * N)), "r"(t + 256), "l"(bd), "r"((int)(i >= NACC)), "r"(idesc));
      else
        asm volatile("{.reg .pred p; setp.ne.b32 p, %3, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;}"
                     ::"r"(t + (uint32_t)((i % NACC) * N)), "l"(ad), "l"(bd), "r"((int)(i >= NACC)), "r"(idesc));
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(smem_u32(&bar)));
    long long t2 = clock64();
    out[2 * blockIdx.x] = t1 - t0;
    out[2 * blockIdx.x + 1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(512));
}

template <int N, bool TS, int NACC>
void run() {
  long long* d;
  cudaMalloc(&d, 2 * 148 * sizeof(long long));
  const int iters = 4096;
  rate<N, TS, NACC><<<148, 128>>>(d, iters);
  rate<N, TS, NACC><<<148, 128>>>(d, iters);
  cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%s N=%3d NACC=%d: issue %.1f cyc/MMA, complete %.1f cyc/MMA (floor 128*N/256 = %d) err=%s\n", TS ? "TS" : "SS",
         N, NACC, (double)h[0] / iters, (double)h[1] / iters, 128 * N / 256, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64, true, 1>(); run<64, true, 2>(); run<64, true, 4>();
  run<64, false, 1>(); run<64, false, 2>(); run<64, false, 4>();
  run<128, true, 1>(); run<128, true, 2>(); run<128, false, 1>(); run<128, false, 2>();
  run<32, false, 4>(); run<96, false, 2>();
  return 0;
}
