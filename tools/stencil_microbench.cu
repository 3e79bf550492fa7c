// Register-level microbenchmark of the spatial-pass inner loop (no memory):
//   acc[j] += g[k] * v[j + k], taps g[] from kernel parameters (uniform registers),
// as plain FFMA and as packed FFMA2 (fma.rn.f32x2) with the even/odd tap split that
// keeps every register pair aligned.  Establishes the achievable FP32 ALU ceiling
// for the stencil pattern on this B200.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int R = 24;
constexpr int NT = 2 * R + 1;
constexpr int NO = 16;  // outputs per thread
struct Taps { float g[NT]; };

__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 upk(unsigned long long v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return make_float2(lo, hi);
}
__device__ __forceinline__ void fma2(unsigned long long& acc, float g, unsigned long long v) {
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(pk(g, g)), "l"(v));
}

constexpr int ROWF = 196;  // smem row (floats, == 4 mod 32), 32 rows
__device__ __forceinline__ void fill(float* sm) {
  for (int i = threadIdx.x; i < 32 * ROWF; i += blockDim.x) sm[i] = (i % 97) * 1e-3f;
  __syncthreads();
}
__global__ void __launch_bounds__(128) st_ffma(float* out, const __grid_constant__ Taps T, int iters) {
  __shared__ __align__(16) float sm[32 * ROWF];
  fill(sm);
  float v[NO + 2 * R];
  float tot = 0.f;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
    const float* src = sm + ((lane + it) & 31) * ROWF + NO * (w & 7) / 2 * 2;
#pragma unroll
    for (int i = 0; i < (NO + 2 * R) / 4; ++i) {
      float4 q = *reinterpret_cast<const float4*>(src + 4 * i);
      v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
    }
    float a[NO];
#pragma unroll
    for (int j = 0; j < NO; ++j) a[j] = 0.f;
#pragma unroll
    for (int k = 0; k < NT; ++k)
#pragma unroll
      for (int j = 0; j < NO; ++j) a[j] = fmaf(T.g[k], v[j + k], a[j]);
#pragma unroll
    for (int j = 0; j < NO; ++j) tot += a[j];
  }
  if (tot == 1234.5f) out[threadIdx.x] = tot;
}

__global__ void __launch_bounds__(128) st_ffma2(float* out, const __grid_constant__ Taps T, int iters) {
  __shared__ __align__(16) float sm[32 * ROWF];
  fill(sm);
  float v[NO + 2 * R + 4];
  float tot = 0.f;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
    const float* src = sm + ((lane + it) & 31) * ROWF + NO * (w & 7) / 2 * 2;
#pragma unroll
    for (int i = 0; i < (NO + 2 * R + 4) / 4; ++i) {
      float4 q = *reinterpret_cast<const float4*>(src + 4 * i);
      v[4 * i] = q.x; v[4 * i + 1] = q.y; v[4 * i + 2] = q.z; v[4 * i + 3] = q.w;
    }
    unsigned long long vp[(NO + 2 * R + 2) / 2];
#pragma unroll
    for (int i = 0; i < (NO + 2 * R + 2) / 2; ++i) vp[i] = pk(v[2 * i], v[2 * i + 1]);
    unsigned long long E[NO / 2], O[NO / 2 + 1];
#pragma unroll
    for (int j = 0; j < NO / 2; ++j) E[j] = 0ull;
#pragma unroll
    for (int j = 0; j <= NO / 2; ++j) O[j] = 0ull;
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      if ((k & 1) == 0) {
#pragma unroll
        for (int j = 0; j < NO / 2; ++j) fma2(E[j], T.g[k], vp[j + k / 2]);     // outputs (2j, 2j+1)
      } else {
#pragma unroll
        for (int j = 0; j <= NO / 2; ++j) fma2(O[j], T.g[k], vp[j + (k - 1) / 2]);  // outputs (2j-1, 2j)
      }
    }
#pragma unroll
    for (int j = 0; j < NO / 2; ++j) {
      float2 e = upk(E[j]), o0 = upk(O[j]), o1 = upk(O[j + 1]);
      tot += (e.x + o0.y) + (e.y + o1.x);
    }
  }
  if (tot == 1234.5f) out[threadIdx.x] = tot;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, 4096);
  Taps T;
  for (int i = 0; i < NT; ++i) T.g[i] = 1.0f / NT;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 64;
  for (int occ : {2, 3, 4, 8}) {
    const int blocks = sms * occ, threads = 128;
    auto time_it = [&](const char* name, auto launch, double useful_fma_per_iter) {
      launch();
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double fma = 5.0 * blocks * threads * (double)iters * useful_fma_per_iter;
      printf("%-10s occ=%d  %.3f ms  useful %.2f T FMA/s (%.1f%% of %d SM x 128 x %.0f MHz)\n", name, occ, ms / 5,
             fma / (ms / 1e3) / 1e12, 100.0 * fma / (ms / 1e3) / (sms * 128.0 * clk * 1e3), sms, clk / 1e3);
    };
    time_it("ffma", [&] { st_ffma<<<blocks, threads>>>(out, T, iters); }, (double)NO * NT);
    time_it("ffma2", [&] { st_ffma2<<<blocks, threads>>>(out, T, iters); }, (double)NO * NT);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
