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
constexpr int kScal = 14;       // doubles of per-volume scalars

// per-volume scalar slots (double sc[B][kScal])
enum ScalSlot : int {
  SC_S = 0,            // scale applied to the stored iterate (1/nu_{k-1}; 1 at k=1)
  SC_XNORM = 1,        // ||x_{k-1}||_2 used for the gain (||x_0|| at k=1, else 1)
  SC_CN = 2,           // backward: c_k / nu_k
  SC_INV_NU = 3,       // backward: 1 / nu_k
  SC_INV_NU_PREV = 4,  // backward: 1 / nu_{k-1}
  SC_NU = 5,           // last nu
  SC_THETA = 6,        // soft-binarisation: mean of the positive entries of y_k (y units)
  SC_CORR = 7,         // backward through a binarised iteration: sum(g) / n_pos (the centre's adjoint)
  SC_VMAX = 8,         // 8 .. 13: max |v| of a temporal pass's output for the fp16 spatial pass that
                       //   reads it (float bits in the slot's first word, atomicMax): slot (k & 1) on
                       //   the hot path, slots 3 (k & 1) + c for the full operator's three inputs.
                       //   With the tcgen05 spatial pass (spass_tc6) slot (k & 1) holds max |p_k| instead
                       //   (written by combine for k = 0 and by the spatial pass of iteration k)
  SC_VEXP = 10,        // tcgen05 pass: exponent e of the fp16 planes of v (v 2^e), written by TP_FWD16
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

// (a, b) -> hi = bf16x2(a, b), lo = bf16x2 of the residuals (a in the low half):
// a = hi + lo to 2^-18 relative (two F2FP, one shift + one LOP3 to widen hi, two FADD).
// The operand split of the tensor-core spatial pass (spass_tc.cuh, A23).
__device__ __forceinline__ void split_bf16x2(float a, float b, uint32_t& hi, uint32_t& lo) {
  uint32_t h;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(b), "f"(a));
  const float ha = __uint_as_float(h << 16), hb = __uint_as_float(h & 0xffff0000u);
  uint32_t l;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(b - hb), "f"(a - ha));
  hi = h;
  lo = l;
}

// (a, b) -> PL bf16x2 planes (a in the low half): plane i holds bf16 of what planes
// 0..i-1 left over, so a = sum_i plane_i to 2^-(9 PL) relative (PL = 3: the full fp32
// significand, 2^-27).  PL = 2 is split_bf16x2.
template <int PL>
__device__ __forceinline__ void split_planes(float a, float b, uint32_t (&o)[PL]) {
#pragma unroll
  for (int i = 0; i < PL; ++i) {
    uint32_t h;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(b), "f"(a));
    o[i] = h;
    if (i + 1 < PL) {
      a -= __uint_as_float(h << 16);
      b -= __uint_as_float(h & 0xffff0000u);
    }
  }
}

// fp16 version of split_planes (the fp16 spatial pass, spass_tc.cuh): a = sum_i plane_i
// to 2^-(11 PL) relative while every plane stays in fp16's normal range (the callers
// scale the data so that max |a| < 2^15).
template <int PL>
__device__ __forceinline__ void split_planes_f16(float a, float b, uint32_t (&o)[PL]) {
#pragma unroll
  for (int i = 0; i < PL; ++i) {
    uint32_t h;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(b), "f"(a));
    o[i] = h;
    if (i + 1 < PL) {
      float lo, hi;
      asm("{.reg .f16 l, h;\n\tmov.b32 {l, h}, %2;\n\tcvt.f32.f16 %0, l;\n\tcvt.f32.f16 %1, h;}"
          : "=f"(lo), "=f"(hi)
          : "r"(h));
      a -= lo;
      b -= hi;
    }
  }
}

// L2 eviction-priority policy (createpolicy) and a hinted 16-byte global store.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_f4_hint(float4* ptr, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}

// Deterministic block sum of per-thread doubles (fixed tree).  All threads get the
// result.  BAR = 0: the whole CTA (__syncthreads); BAR > 0: the named barrier BAR over
// the first NT threads only (kernels whose producer warp has already exited).
template <int NT, int BAR = 0>
__device__ __forceinline__ void nt_sync() {
  if (BAR == 0) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
  }
}
template <int NT, int BAR = 0>
__device__ __forceinline__ double block_sum(double v, double* red /* smem, NT/32 doubles */) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  nt_sync<NT, BAR>();
  if (l == 0) red[w] = v;
  nt_sync<NT, BAR>();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = (l < NT / 32) ? red[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (l == 0) red[0] = t;
  }
  nt_sync<NT, BAR>();
  t = red[0];
  nt_sync<NT, BAR>();
  return t;
}

// Fixed-order sum of a[lo..hi) (element i at a[i * stride]) by the whole block:
// thread t sums lo+t, lo+t+NT, ... with the loads issued 8 at a time (one memory
// latency per 8*NT elements instead of per NT), then a fixed tree.  Deterministic.
// Measured: the finalize of a 296-CTA launch that summed its per-warp partials with
// one warp and no unrolling took 21 us of a 115 us kernel (profiles/f3d trace).
template <int NT, int BAR = 0>
__device__ __forceinline__ double block_sum_range(const double* a, long lo, long hi, long stride, double* red) {
  double s = 0.0;
  long i = lo + threadIdx.x;
  for (; i + 7L * NT < hi; i += 8L * NT) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcg(a + (i + (long)j * NT) * stride);
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
  }
  for (; i < hi; i += NT) s += __ldcg(a + i * stride);
  return block_sum<NT, BAR>(s, red);
}
template <int NT>
__device__ __forceinline__ double block_sum_array(const double* a, long n, long stride, double* red) {
  return block_sum_range<NT>(a, 0, n, stride, red);
}
// Fixed-order sum of a[lo..hi) by one warp (lane l sums lo+l, lo+l+32, ..., loads 8 at a
// time), then a fixed butterfly; all lanes get the result.
__device__ __forceinline__ double warp_sum_range(const double* a, long lo, long hi) {
  const int l = threadIdx.x & 31;
  double s = 0.0;
  long i = lo + l;
  for (; i + 7L * 32 < hi; i += 8L * 32) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcg(a + i + (long)j * 32);
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
  }
  for (; i < hi; i += 32) s += __ldcg(a + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}
// CTA slot range [lo, hi) whose static unit ranges [c*U/G, (c+1)*U/G) intersect the
// units [b*per, (b+1)*per) of volume b (closed form; checked by brute force).
__device__ __forceinline__ void vol_cta_range(long b, long per, long U, long G, long& lo, long& hi) {
  const long x0 = b * per, x1 = (b + 1) * per;
  hi = min(G, (x1 * G + U - 1) / U);
  lo = ((x0 + 1) * G + U - 1) / U - 1;
}

// Counter increment with acquire-release semantics at GPU scope: the release orders
// this thread's earlier writes (and, by cumulativity, the CTA's writes ordered before
// it by a barrier) before the increment; the acquire makes every earlier arrival's
// writes visible to the last arriver.  Replaces __threadfence() + atomicAdd, whose
// MEMBAR.SC.GPU waits for ALL of the thread's outstanding stores (the epilogue's).
__device__ __forceinline__ unsigned atomic_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// "Last block done" arrival: returns true in exactly one (the last) block.  All
// threads of the block see the same value.  Thread 0 wrote the block's partials.
__device__ __forceinline__ bool last_block_arrive(unsigned* counter, unsigned total, int* flag_smem) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomic_add_acq_rel(counter, 1u);
    *flag_smem = (prev == total - 1) ? 1 : 0;
  }
  __syncthreads();
  return *flag_smem != 0;
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
// TMA box -> L2 only (no shared memory, no barrier): raises the bytes a CTA keeps in flight
// beyond its shared-memory stages
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

}  // namespace sfseg
