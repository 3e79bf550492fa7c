// Shared device helpers for the SFSeg sm_100a kernels.
//
// Layouts:
//   user buffers: dense [B][T][H][W] fp32 (W fastest);
//   internal volumes (F, iterate p, temporal output v, tape u, adjoints):
//   pitched [B*T][H][Wp] fp32 with Wp = round_up(W, 8) so every row starts on
//   a 32-byte sector and float4 / TMA accesses are aligned.  Pad columns
//   (x >= W) hold zeros or don't-care values; TMA descriptors use width W, so
//   out-of-bounds columns and rows read as zero (= the zero padding of
//   reading A8) without guard memory.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sfseg {

constexpr int kTW = 64;         // output columns per spatial-pass strip
constexpr int kM = 32;          // rows per spatial-pass block
constexpr int kSpassThreads = 128;
constexpr int kSpassWarps = kSpassThreads / 32;
constexpr int kSpassPartSlots = 1;    // norm partial slots per CTA
constexpr int kRingStride = kTW + 4;  // ring row stride in floats (== 4 mod 32: conflict-free)
constexpr int kMaxC = 64;       // channels passed by value in kernel parameters
constexpr int kScal = 8;        // doubles of per-volume scalars

// per-volume scalar slots (double sc[B][kScal])
enum ScalSlot : int {
  SC_S = 0,            // scale applied to the stored iterate (1/nu_{k-1}; 1 at k=1)
  SC_XNORM = 1,        // ||x_{k-1}||_2 used for the gain (||x_0|| at k=1, else 1)
  SC_CN = 2,           // backward: c_k / nu_k
  SC_INV_NU = 3,       // backward: 1 / nu_k
  SC_INV_NU_PREV = 4,  // backward: 1 / nu_{k-1}
  SC_NU = 5,           // last nu
  SC_THETA = 6,        // soft-binarisation: mean of the positive entries of y_k (y units)
};

enum ErrBits : unsigned { ERR_DEGENERATE = 1u, ERR_NONFINITE = 2u };

// Workspace header (first 256 bytes of the workspace).
struct WsHeader {
  unsigned err;
  unsigned counter[15];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ float4 f4_mul(float4 a, float4 b) {
  return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
}
__device__ __forceinline__ float4 f4_scale(float4 a, float s) {
  return make_float4(a.x * s, a.y * s, a.z * s, a.w * s);
}
__device__ __forceinline__ float f4_dot(float4 a, float4 b) {
  return a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
}

// Deterministic block sum of per-thread doubles (fixed tree).  All threads get the result.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red /* smem, NT/32 doubles */) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = (l < NT / 32) ? red[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (l == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// Fixed-order sum of a[0..n) by the whole block (thread i sums i, i+NT, ...; then a tree).
template <int NT>
__device__ __forceinline__ double block_sum_array(const double* a, long n, long stride, double* red) {
  double s = 0.0;
  for (long i = threadIdx.x; i < n; i += NT) s += a[i * stride];
  return block_sum<NT>(s, red);
}

// "Last block done" arrival: returns true in exactly one (the last) block.  All
// threads of the block see the same value.  Caller wrote its partials before.
__device__ __forceinline__ bool last_block_arrive(unsigned* counter, unsigned total, int* flag_smem) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev = atomicAdd(counter, 1u);
    *flag_smem = (prev == total - 1) ? 1 : 0;
  }
  __syncthreads();
  bool last = *flag_smem != 0;
  if (last) __threadfence();
  return last;
}

// First device-detected error wins (a zero norm at k makes every later norm NaN).
__device__ __forceinline__ void flag_norm(unsigned* err, double nu) {
  if (!isfinite(nu)) atomicCAS(err, 0u, (unsigned)ERR_NONFINITE);
  else if (!(nu > 0.0)) atomicCAS(err, 0u, (unsigned)ERR_DEGENERATE);
}

// ---------------------------------------------------------------- mbarrier / TMA (sm_90+ PTX)
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// try_wait with a suspend-time hint: a waiting thread sleeps until the phase
// completes (or the hint expires) instead of spinning -- measured: without the
// hint the try_wait/yield/branch loops were 26 % of the fused 3D kernel's issued
// instructions, stealing issue slots from the compute warps.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                            int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

}  // namespace sfseg
