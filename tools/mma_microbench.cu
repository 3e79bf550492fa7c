// Legacy warp-level tensor-core (mma.sync -> HMMA) throughput on sm_100a, full chip:
// m16n8k8 tf32 and m16n8k16 bf16 with fp32 accumulators.  Decides whether the
// banded (Toeplitz) formulation of the spatial Gaussian can leave the FP32 pipe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_microbench tools/mma_microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 2048;
constexpr int kAcc = 8;  // independent accumulator tiles per warp

// bf16 with NACC independent accumulator chains (latency / per-warp issue probe)
template <int NACC>
__global__ void mma_bf16_chain(float* out, unsigned seed) {
  unsigned a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = (seed + threadIdx.x * 7 + i) & 0x3f803f80u;
#pragma unroll
  for (int i = 0; i < 2; ++i) b[i] = (seed ^ (threadIdx.x * 13 + i)) & 0x3f803f80u;
  float d[NACC][4];
#pragma unroll
  for (int j = 0; j < NACC; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[j][i] = 0.f;
  for (int it = 0; it < kIters * kAcc / NACC; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < NACC; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void mma_tf32(float* out, unsigned seed) {
  unsigned a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = seed + threadIdx.x * 7 + i;
#pragma unroll
  for (int i = 0; i < 2; ++i) b[i] = seed ^ (threadIdx.x * 13 + i);
  float d[kAcc][4];
#pragma unroll
  for (int j = 0; j < kAcc; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[j][i] = 0.f;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int j = 0; j < kAcc; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < kAcc; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void mma_bf16(float* out, unsigned seed) {
  unsigned a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = (seed + threadIdx.x * 7 + i) & 0x3f803f80u;
#pragma unroll
  for (int i = 0; i < 2; ++i) b[i] = (seed ^ (threadIdx.x * 13 + i)) & 0x3f803f80u;
  float d[kAcc][4];
#pragma unroll
  for (int j = 0; j < kAcc; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[j][i] = 0.f;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int j = 0; j < kAcc; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < kAcc; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

template <typename K>
void run(const char* name, K kern, double flop_per_mma, int threads, int blocks_per_sm) {
  float* out;
  cudaMalloc(&out, 4096 * sizeof(float));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * blocks_per_sm;
  kern<<<blocks, threads>>>(out, 1u);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(out, 1u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = (double)blocks * threads / 32;
  const double flop = 5.0 * warps * kIters * kAcc * flop_per_mma;
  printf("%-10s threads=%4d blocks/SM=%d  %.1f TFLOP/s  (%s)\n", name, threads, blocks_per_sm,
         flop / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  for (int bps : {1, 2, 4}) {
    run("tf32", mma_tf32, 2.0 * 16 * 8 * 8, 256, bps);
    run("bf16", mma_bf16, 2.0 * 16 * 8 * 16, 256, bps);
  }
  run("tf32", mma_tf32, 2.0 * 16 * 8 * 8, 128, 4);
  run("bf16", mma_bf16, 2.0 * 16 * 8 * 16, 128, 4);
  // chains x warps per SM sub-partition (128 threads per block = 1 warp per SMSP)
  for (int wps : {1, 2, 3, 4}) {
    run("bf16 acc1", mma_bf16_chain<1>, 2.0 * 16 * 8 * 16, 128, wps);
    run("bf16 acc2", mma_bf16_chain<2>, 2.0 * 16 * 8 * 16, 128, wps);
    run("bf16 acc4", mma_bf16_chain<4>, 2.0 * 16 * 8 * 16, 128, wps);
    run("bf16 acc8", mma_bf16_chain<8>, 2.0 * 16 * 8 * 16, 128, wps);
  }
  return 0;
}
