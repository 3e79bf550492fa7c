// tcgen05 primitive probe (sm_100a): TMEM alloc / st / ld, tcgen05.mma kind::f16 (bf16 in,
// fp32 accumulate) with A from TMEM (TS) or shared memory (SS), B from shared memory in the
// K-major and MN-major no-swizzle canonical layouts, commit to an mbarrier.  Checks
// D[128][N] = A[128][K] . B[K][N] against a host reference and prints the max error per case.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc05_probe tools/tc05_probe.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int M = 128, K = 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // sm_100 shared-memory matrix descriptor: start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46),
  // version 1 [46,48), base offset 0, lbo mode 0, layout type SWIZZLE_NONE (0) [61,64)
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t make_idesc(int n, int a_mn_major, int b_mn_major) {
  // kind::f16: c_format F32 (1) [4,6), a_format BF16 (1) [7,10), b_format BF16 (1) [10,13),
  // a_major [15], b_major [16], N >> 3 [17,23), M >> 4 [24,29)
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn_major << 15) | ((uint32_t)b_mn_major << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// element (n, k) of B in the K-major SWIZZLE_NONE layout: core matrices of 8 rows (n) x 16 B (8 k);
// K-chunks at LBO, 8-row groups at SBO
__device__ __forceinline__ uint32_t b_kmaj_off(int n, int k, uint32_t lbo, uint32_t sbo) {
  return (uint32_t)(n / 8) * sbo + (uint32_t)(k / 8) * lbo + (uint32_t)(n % 8) * 16 + (uint32_t)(k % 8) * 2;
}
// element (k, n) of B in the MN-major SWIZZLE_NONE layout: core matrices of 8 k-rows x 16 B (8 n);
// 8-element n groups at SBO, 8-row k groups at LBO
__device__ __forceinline__ uint32_t b_mnmaj_off(int n, int k, uint32_t lbo, uint32_t sbo) {
  return (uint32_t)(n / 8) * sbo + (uint32_t)(k / 8) * lbo + (uint32_t)(k % 8) * 16 + (uint32_t)(n % 8) * 2;
}

template <int N>
__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int mode) {
  // mode 0: TS, B K-major; 1: TS, B MN-major; 2: SS (A K-major), B K-major
  __shared__ __align__(1024) uint8_t sB[N * K * 2];
  __shared__ __align__(1024) uint8_t sA[M * K * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t taddr_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr uint32_t LBO_K = 128, SBO_K = (K / 8) * 128;            // B K-major: K chunks adjacent
  constexpr uint32_t LBO_MN = 128, SBO_MN = (K / 8) * 128;          // B MN-major: k groups adjacent
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    const uint32_t off = mode == 1 ? b_mnmaj_off(n, k, LBO_MN, SBO_MN) : b_kmaj_off(n, k, LBO_K, SBO_K);
    *reinterpret_cast<__nv_bfloat16*>(sB + off) = B[k * N + n];
  }
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sA + b_kmaj_off(m, k, 128, (K / 8) * 128)) = A[m * K + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&taddr_s)), "r"(256));
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
  const uint32_t tbase = taddr_s;
  const uint32_t tA = tbase + 128;   // A operand columns [128, 128 + K/2)
  // A into TMEM: thread = lane m (warps 0..3), columns k/2, element k in half (k & 1)
  if (warp < 4) {
    const int m = 32 * warp + lane;
    uint32_t r[K / 2];
    for (int c = 0; c < K / 2; ++c) {
      const __nv_bfloat16 lo = A[m * K + 2 * c], hi = A[m * K + 2 * c + 1];
      r[c] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
    }
    const uint32_t ta = tA + ((uint32_t)(32 * warp) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                 "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t idesc = make_idesc(N, 0, mode == 1 ? 1 : 0);
    for (int s = 0; s < K / 16; ++s) {
      const uint32_t boff = mode == 1 ? (uint32_t)(2 * s) * LBO_MN : (uint32_t)(2 * s) * LBO_K;
      const uint64_t bdesc = make_desc(smem_u32(sB) + boff, mode == 1 ? LBO_MN : LBO_K, mode == 1 ? SBO_MN : SBO_K);
      const uint32_t acc = s > 0;
      if (mode == 2) {
        const uint64_t adesc = make_desc(smem_u32(sA) + (uint32_t)(2 * s) * 128, 128, (K / 8) * 128);
        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                     ::"r"(tbase), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
      } else {
        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}"
                     ::"r"(tbase), "r"(tA + (uint32_t)(8 * s)), "l"(bdesc), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  // wait for the MMAs
  asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    const int m = 32 * warp + lane;
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tbase + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 8; ++j) D[m * N + c0 + j] = __uint_as_float(r[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(256));
}

template <int N>
void run(int mode) {
  __nv_bfloat16 *hA = (__nv_bfloat16*)malloc(M * K * 2), *hB = (__nv_bfloat16*)malloc(K * N * 2);
  float *fA = (float*)malloc(M * K * 4), *fB = (float*)malloc(K * N * 4), *hD = (float*)malloc(M * N * 4);
  srand(7 + mode);
  for (int i = 0; i < M * K; ++i) { hA[i] = __float2bfloat16((rand() % 2001 - 1000) / 1000.f); fA[i] = __bfloat162float(hA[i]); }
  for (int i = 0; i < K * N; ++i) { hB[i] = __float2bfloat16((rand() % 2001 - 1000) / 1000.f); fB[i] = __bfloat162float(hB[i]); }
  __nv_bfloat16 *dA, *dB; float* dD;
  CK(cudaMalloc(&dA, M * K * 2)); CK(cudaMalloc(&dB, K * N * 2)); CK(cudaMalloc(&dD, M * N * 4));
  CK(cudaMemcpy(dA, hA, M * K * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB, K * N * 2, cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, M * N * 4));
  probe<N><<<1, 128>>>(dA, dB, dD, mode);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost));
  double err = 0; int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)fA[m * K + k] * fB[k * N + n];
      const double e = fabs(ref - hD[m * N + n]);
      if (e > err) err = e;
      if (e > 1e-3 && bad < 4) { printf("  mode %d N %d: D[%d][%d] = %g, ref %g\n", mode, N, m, n, hD[m * N + n], ref); ++bad; }
    }
  printf("mode %d (%s) N=%d: max abs err %.3e %s\n", mode, mode == 0 ? "TS, B K-major" : mode == 1 ? "TS, B MN-major" : "SS",
         N, err, err < 1e-4 ? "OK" : "FAIL");
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
}

int main() {
  for (int mode = 0; mode < 3; ++mode) { run<64>(mode); run<32>(mode); }
  return 0;
}
