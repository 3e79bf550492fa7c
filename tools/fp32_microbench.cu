// FP32 FMA-pipe microbenchmark for the ALU roofline of the spatial pass
// (SURVEY.md B16): throughput of FFMA with a uniform/constant operand, FFMA with
// three vector registers, and packed fma.rn.f32x2 (sm_100+), full chip.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_microbench tools/fp32_microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 16;

__global__ void ffma_const(float* out, float a, float b) {
  float acc[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) acc[i] = threadIdx.x * 1e-7f + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) acc[i] = fmaf(acc[i], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += acc[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void ffma_reg(float* out, float a0, float b0) {
  float acc[kChains], x[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    acc[i] = threadIdx.x * 1e-7f + i;
    x[i] = a0 + i * 1e-3f + threadIdx.x * 1e-9f;
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) acc[i] = fmaf(x[i], x[(i + 1) % kChains], acc[i]);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += acc[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

// stencil-like: acc[j] += g * v[j] with g uniform, v per-thread (the spass inner loop shape)
__global__ void ffma_stencil(float* out, float g0) {
  float acc[kChains], v[kChains];
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    acc[i] = 0.f;
    v[i] = threadIdx.x * 1e-7f + i;
  }
  for (int it = 0; it < kIters; ++it) {
    const float g = g0 + it * 1e-9f;  // uniform across the warp
#pragma unroll
    for (int i = 0; i < kChains; ++i) acc[i] = fmaf(g, v[i], acc[i]);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += acc[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void ffma2_stencil(float* out, float g0) {
  unsigned long long acc[kChains / 2], v[kChains / 2];
#pragma unroll
  for (int i = 0; i < kChains / 2; ++i) {
    float lo = threadIdx.x * 1e-7f + 2 * i, hi = lo + 1.f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(v[i]) : "f"(lo), "f"(hi));
    acc[i] = 0ull;
  }
  for (int it = 0; it < kIters; ++it) {
    const float g = g0 + it * 1e-9f;
    unsigned long long gg;
    asm("mov.b64 %0, {%1, %1};" : "=l"(gg) : "f"(g));
#pragma unroll
    for (int i = 0; i < kChains / 2; ++i)
      asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc[i]) : "l"(gg), "l"(v[i]));
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < kChains / 2; ++i) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[i]));
    s += lo + hi;
  }
  if (s == 1234.5f) out[threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs=%d clock(max, kHz)=%d  nominal FP32 FMA peak = %.2f T/s\n", sms, clk, sms * 128.0 * clk * 1e3 / 1e12);
  float* out;
  cudaMalloc(&out, 4096);
  const int threads = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int occ : {2, 4, 8}) {
    const int blocks = sms * occ;
    auto time_it = [&](const char* name, auto launch) {
      launch();
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double fma = 5.0 * blocks * threads * (double)kIters * kChains;
      printf("%-14s occ=%d  %.3f ms/launch  %.2f T FMA/s (%.1f TFLOP/s)\n", name, occ, ms / 5,
             fma / (ms / 1e3) / 1e12, 2 * fma / (ms / 1e3) / 1e12);
    };
    time_it("ffma_const", [&] { ffma_const<<<blocks, threads>>>(out, 0.999f, 0.5f); });
    time_it("ffma_reg", [&] { ffma_reg<<<blocks, threads>>>(out, 0.999f, 0.5f); });
    time_it("ffma_stencil", [&] { ffma_stencil<<<blocks, threads>>>(out, 0.999f); });
    time_it("ffma2_stencil", [&] { ffma2_stencil<<<blocks, threads>>>(out, 0.999f); });
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
