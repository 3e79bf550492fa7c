// Temporal pass of G_3D: out[t] = scale * sum_{|o|<=RT} g_t[o] * src[t+o]  (zero padded).
//
// One of the "three vector-wise convolutions" of the separable Gaussian
// (PAPER.md:319).  HBM-bound streaming kernel: each thread owns one float4
// column (b, y, 4x..4x+3) of the pitched volume and walks the T frames once,
// keeping the 2RT+1 partial outputs that an input frame touches in a register
// ring (unrolled by 2RT+1 so ring slots are static registers).  Every input
// float4 is read from HBM exactly once and every output written once:
// 8 B/voxel (forward), 16 B/voxel (backward: reads x_bar, F, u).
#pragma once
#include "common.cuh"

namespace sfseg {

constexpr int kMaxRT = 16;

enum TpassMode : int {
  TP_FWD = 0,   // src = p (stored iterate), out = s_{k-1} * G_t * p
  TP_BWD = 1,   // src = F * y_bar_k, y_bar_k = (x_bar_k - [x_k > 0] corr - F u_{k-1} cn) * inv_nu (Appendix A;
                //   corr != 0 only after a soft-binarised iteration, reading A21)
  TP_FWDF = 2,  // full SFSeg operator (f1): src = F^fexp * a, out = s_{k-1} * G_t * src  (Eq.7's three inputs)
  TP_FWD16 = 3, // as TP_FWD, out = the two fp16 planes of v 2^e ([bt][plane][H][Wp] halves, 4 B/voxel) for the
                //   tcgen05 spatial pass (spass_tc6.cuh); e from max |p_{k-1}| so that |v 2^e| < 2^14
  TP_BWD16 = 4, // as TP_BWD, out as TP_FWD16; e from the bound |src| <= max|F| (max|x_bar_k| + |corr| +
                //   max|F| max|u| |cn|) |1/nu_k| (A26)
};

struct TpassParams {
  const float* src;      // FWD: p ; BWD: x_bar_k            pitched [B*T][H][Wp]
  const float* F;        // BWD, FWDF
  const float* u1;       // BWD: tape u_{k-1}
  const float* halo_lo;  // [B][RT][H][Wp] frames t = -RT..-1 (time slabs) or null
  const float* halo_hi;  // [B][RT][H][Wp] frames t = T..T+RT-1 or null
  float* out;            // pitched [B*T][H][Wp]
  const double* sc;      // per-volume scalars [B][kScal]
  unsigned* vmax;        // atomicMax of max |out| per volume (float bits, stride 2 kScal words) or null
  const unsigned* pmax_in;  // FWD16: max |src| per volume (float bits, stride 2 kScal words)
  unsigned* pmax_zero;     // FWD16: slot zeroed for the next spatial pass's max |p_k| (or null)
  double* vexp_out;        // FWD16: sc + SC_VEXP (stride kScal): the exponent e written per volume
  float gsum;              // FWD16: sum of |g| (|v| <= s gsum max |src|)
  const unsigned* fmax_in; // BWD16: max |F|; pmax_in is then max |x_bar_k|
  const unsigned* umax_in; // BWD16: max |F| (u_k, k >= 2) or max |F x_0| (u_1): |u| <= gs3 * it
  float gs3;               // BWD16: sum|g_t| (sum|g_s|)^2
  int lag;               // FWD: no scale (the spatial pass applies s_{k-1}: lagged normalisation, time slabs)
  long frame4;           // H*Wp/4 float4 per frame
  int T;
  int fexp;              // FWDF: exponent of F multiplying the source (1 or 2)
  float g[2 * kMaxRT + 1];  // g[i] = weight of temporal offset i - RT
  unsigned long long g2[2 * kMaxRT + 1];  // {g[i], g[i]} packed for fma.rn.f32x2 (set by fill_tpass_common)
};

constexpr int kTpThreads = 128;
#ifndef TPASS_REV
#define TPASS_REV 0  // A/B: walk the frames last to first (the symmetric taps make it the same filter)
#endif
// Resident CTAs per SM the register budget is sized for: the ring of 2RT+1
// float4 accumulators dominates (RT=6: 52 registers).  At c2 (frame4 = 102,720
// float4 columns) 6 x 128 threads per SM hold every column in ONE wave.
__host__ __device__ constexpr int tpass_min_blocks(int RT) { return RT <= 6 ? 6 : (RT <= 9 ? 4 : 2); }
// cp.async stages per input stream (frames prefetched ahead of the ring).
__host__ __device__ constexpr int tpass_stages(int MODE) {
  return (MODE == TP_FWD || MODE == TP_FWD16) ? 16 : (MODE == TP_FWDF ? 8 : 4);   // powers of two: no modulo code
}
#ifndef TPASS16_HINT
#define TPASS16_HINT 1  // A/B: TP_FWD16 stores v's planes with an L2 evict-last policy (0: .cg stores)
#endif
constexpr int kF16DataExp = 14;  // TP_FWD16: |v 2^e| < 2^14 (fp16 max 65504)
// register-pair (un)packing: mov.b64 lets ptxas allocate the pair instead of emitting shifts / ORs
__device__ __forceinline__ unsigned long long pack_f2(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ float2 unpack_f2(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ float4 unpack_f4(unsigned long long xy, unsigned long long zw) {
  const float2 a = unpack_f2(xy), b = unpack_f2(zw);
  return make_float4(a.x, a.y, b.x, b.y);
}
// acc = w * v + acc on two packed fp32 lanes (sm_100 fma.rn.f32x2: the same rounding as two FFMA)
__device__ __forceinline__ void ffma2(unsigned long long& acc, unsigned long long w, unsigned long long v) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(w), "l"(v));
}
__device__ __forceinline__ void st_u2_hint(uint2* ptr, uint2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1, %2}, %3;" ::"l"(ptr), "r"(v.x), "r"(v.y), "l"(pol)
               : "memory");
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One thread = one float4 column (b, y, 4x..4x+3) of the pitched volume, walked
// through all frames.  Input frames are prefetched NS frames ahead with cp.async
// into a per-thread shared-memory slot (no register cost for loads in flight;
// each thread reads back only its own slots, so no block barrier is needed);
// the 2RT+1 partial outputs an input frame feeds live in a register ring
// (unrolled by 2RT+1 so ring slots are static registers).
template <int RT, int MODE, bool HALO>
__global__ void __launch_bounds__(kTpThreads, tpass_min_blocks(RT)) tpass_kernel(const __grid_constant__ TpassParams P) {
  constexpr int NR = 2 * RT + 1;
  constexpr int NS = tpass_stages(MODE);
  constexpr bool F16 = MODE == TP_FWD16 || MODE == TP_BWD16;   // fp16-plane output
  constexpr bool FWDM = MODE == TP_FWD || MODE == TP_FWD16;     // input p (one stream)
  constexpr int NIN = FWDM ? 1 : (MODE == TP_FWDF ? 2 : 3);
  __shared__ float4 sq[NS][NIN][kTpThreads];
  const int b = blockIdx.y;
  const int tid = threadIdx.x;
  const long e = (long)blockIdx.x * kTpThreads + tid;
  const bool active = e < P.frame4;
  const int T = P.T;
  const long vol4 = (long)T * P.frame4;
  const long ec = active ? e : 0;  // inactive threads keep valid addresses and skip the stores
  const float4* src = reinterpret_cast<const float4*>(P.src) + b * vol4 + ec;
  const float4* Fp = nullptr;
  const float4* U1 = nullptr;
  float cn = 0.f, inv_nu = 0.f, corr = 0.f, scale = 1.f;
  float m16 = 1.f;  // FWD16: s_{k-1} 2^e
  if (FWDM) {
    scale = P.lag ? 1.f : (float)P.sc[b * kScal + SC_S];
    if (F16) {
      const float bound = scale * __uint_as_float(P.pmax_in[(long)b * 2 * kScal]) * P.gsum;
      int ex = 0;
      if (bound > 0.f && bound <= 3.4e38f) frexpf(bound, &ex);  // bound < 2^ex
      const int e = min(max(kF16DataExp - ex, -100), 100);
      m16 = scale * __int_as_float((127 + e) << 23);
      if (blockIdx.x == 0 && tid == 0) {
        P.vexp_out[(long)b * kScal] = (double)e;
        if (P.pmax_zero) P.pmax_zero[(long)b * 2 * kScal] = 0u;
      }
    }
  } else if (MODE == TP_FWDF) {
    scale = (float)P.sc[b * kScal + SC_S];
    Fp = reinterpret_cast<const float4*>(P.F) + b * vol4 + ec;
  } else {
    Fp = reinterpret_cast<const float4*>(P.F) + b * vol4 + ec;
    U1 = reinterpret_cast<const float4*>(P.u1) + b * vol4 + ec;
    cn = (float)P.sc[b * kScal + SC_CN];
    inv_nu = (float)P.sc[b * kScal + SC_INV_NU];
    corr = (float)P.sc[b * kScal + SC_CORR];  // 0 unless iteration k was soft-binarised
    if (F16) {
      const float mf = __uint_as_float(P.fmax_in[(long)b * 2 * kScal]);
      const float bound = mf *
                          (__uint_as_float(P.pmax_in[(long)b * 2 * kScal]) + fabsf(corr) +
                           mf * P.gs3 * __uint_as_float(P.umax_in[(long)b * 2 * kScal]) * fabsf(cn)) *
                          fabsf(inv_nu) * P.gsum;
      int ex = 0;
      if (bound > 0.f && bound <= 3.4e38f) frexpf(bound, &ex);
      const int e = min(max(kF16DataExp - ex, -100), 100);
      m16 = __int_as_float((127 + e) << 23);
      if (blockIdx.x == 0 && tid == 0) {
        P.vexp_out[(long)b * kScal] = (double)e;
        if (P.pmax_zero) P.pmax_zero[(long)b * 2 * kScal] = 0u;
      }
    }
  }
  const float4* hlo = P.halo_lo ? reinterpret_cast<const float4*>(P.halo_lo) + (long)b * RT * P.frame4 + ec : nullptr;
  const float4* hhi = P.halo_hi ? reinterpret_cast<const float4*>(P.halo_hi) + (long)b * RT * P.frame4 + ec : nullptr;
  float4* out = reinterpret_cast<float4*>(P.out) + b * vol4 + ec;

  // jp = j + RT enumerates input frames j = -RT .. T+RT-1; output t = jp - 2RT
  // completes when input j = t + RT arrives.
  // walk index j -> frame (TPASS_REV: T - 1 - j; the taps are symmetric, so the same ring
  // computes the same filter on the mirrored sequence)
  auto frame_src = [&](int jp, int w) -> const float4* {
    const int j = jp - RT;
    if (j >= 0 && j < T) {
      const long o = (long)(TPASS_REV ? T - 1 - j : j) * P.frame4;
      return (w == 0) ? src + o : (w == 1 ? Fp + o : U1 + o);
    }
    if (HALO && w == 0) {  // neighbour slab frames (time-slab sharding)
      if (TPASS_REV) {
        if (j < 0 && j >= -RT && hhi) return hhi + (long)(-1 - j) * P.frame4;
        if (j >= T && j < T + RT && hlo) return hlo + (long)(T - 1 - j + RT) * P.frame4;
      } else {
        if (j < 0 && j >= -RT && hlo) return hlo + (long)(j + RT) * P.frame4;
        if (j >= T && j < T + RT && hhi) return hhi + (long)(j - T) * P.frame4;
      }
    }
    return nullptr;  // zero padding
  };
  const int jend = T + 2 * RT;
  auto issue = [&](int jp) {
    if (jp < jend) {
#pragma unroll
      for (int w = 0; w < NIN; ++w) {
        const float4* g = frame_src(jp, w);
        if (g) cp_async16(&sq[jp % NS][w][tid], g);
      }
    }
    cp_async_commit();  // one group per frame, possibly empty: keeps wait_group counting uniform
  };
  auto fetch = [&](int jp) -> float4 {
    const int j = jp - RT;
    const int sl = jp % NS;
    float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
    if (FWDM) {
      if (frame_src(jp, 0)) val = sq[sl][0][tid];
    } else if (MODE == TP_FWDF) {
      if (j >= 0 && j < T) {
        const float4 a = sq[sl][0][tid], f = sq[sl][1][tid];
        const float4 fe = (P.fexp == 2) ? f4_mul(f, f) : f;
        val = f4_mul(fe, a);
      }
    } else if (j >= 0 && j < T) {
      const float4 xb = sq[sl][0][tid], f = sq[sl][1][tid], u = sq[sl][2][tid];
      val.x = f.x * ((xb.x - (f.x * u.x > 0.f ? corr : 0.f) - f.x * u.x * cn) * inv_nu);
      val.y = f.y * ((xb.y - (f.y * u.y > 0.f ? corr : 0.f) - f.y * u.y * cn) * inv_nu);
      val.z = f.z * ((xb.z - (f.z * u.z > 0.f ? corr : 0.f) - f.z * u.z * cn) * inv_nu);
      val.w = f.w * ((xb.w - (f.w * u.w > 0.f ? corr : 0.f) - f.w * u.w * cn) * inv_nu);
    } else if (HALO) {
      // backward halos arrive pre-multiplied (F * y_bar of the neighbour slab)
      const float4* g = frame_src(jp, 0);
      if (g) val = sq[sl][0][tid];
    }
    return val;
  };

  // forward: keep v in L2 for the spatial pass that reads it next (and its halo re-reads)
  const uint64_t pol = (FWDM || F16) ? l2_policy_evict_last() : 0ull;
  uint2* const o16 = F16 ? reinterpret_cast<uint2*>(P.out) + (long)b * T * 2 * P.frame4 + ec : nullptr;
  // the ring of 2RT+1 partial outputs: float4 as two packed float2 (fma.rn.f32x2 = FFMA2: half
  // the FMA instructions of a pass that is issue-bound, profiles/r02e/tpass_ncu.txt)
  unsigned long long acc[NR][2];
#pragma unroll
  for (int i = 0; i < NR; ++i) acc[i][0] = acc[i][1] = 0ull;
  float vm = 0.f;  // max |out| of this thread (FWD with vmax)
#pragma unroll
  for (int d = 0; d < NS; ++d) issue(d);
  for (int j0 = 0; j0 < jend; j0 += NR) {
#pragma unroll
    for (int d = 0; d < NR; ++d) {
      const int jp = j0 + d;
      if (jp >= jend) break;
      cp_async_wait<NS - 1>();  // frame jp has landed (this thread's own copies)
      const float4 val = fetch(jp);
      issue(jp + NS);  // refill the slot just read
#pragma unroll
      const unsigned long long vxy = pack_f2(val.x, val.y), vzw = pack_f2(val.z, val.w);
#pragma unroll
      for (int ee = 0; ee < NR; ++ee) {
        // input j feeds output t = j - RT + ee with weight g[(j - t) + RT] = g[2RT - ee]
        const int slot = (((d - 2 * RT + ee) % NR) + NR) % NR;
        const unsigned long long w2 = P.g2[2 * RT - ee];
        ffma2(acc[slot][0], w2, vxy);
        ffma2(acc[slot][1], w2, vzw);
      }
      const int slot0 = (((d - 2 * RT) % NR) + NR) % NR;
      const int t = jp - 2 * RT;
      const float4 a4 = unpack_f4(acc[slot0][0], acc[slot0][1]);
      if (F16 && active && t >= 0 && t < T) {
        const float4 o = f4_scale(a4, m16);
        uint32_t h0[2], h1[2];
        split_planes_f16<2>(o.x, o.y, h0);
        split_planes_f16<2>(o.z, o.w, h1);
        uint2* dst = o16 + (long)(TPASS_REV ? T - 1 - t : t) * 2 * P.frame4;
        if (TPASS16_HINT) {
          st_u2_hint(dst, make_uint2(h0[0], h1[0]), pol);
          st_u2_hint(dst + P.frame4, make_uint2(h0[1], h1[1]), pol);
        } else {
          __stcg(dst, make_uint2(h0[0], h1[0]));
          __stcg(dst + P.frame4, make_uint2(h0[1], h1[1]));
        }
      } else if (active && t >= 0 && t < T) {
        const float4 o = f4_scale(a4, scale);
        float4* dst = out + (long)(TPASS_REV ? T - 1 - t : t) * P.frame4;
        if (MODE == TP_FWD) st_f4_hint(dst, o, pol);
        else __stcg(dst, o);
        vm = fmaxf(vm, fmaxf(fmaxf(fabsf(o.x), fabsf(o.y)), fmaxf(fabsf(o.z), fabsf(o.w))));
      }
      acc[slot0][0] = acc[slot0][1] = 0ull;
    }
  }
  cp_async_wait<0>();
  if (P.vmax) {  // max |out| of the volume: the fp16 spatial pass's range (max is order-free)
    __shared__ unsigned wm[kTpThreads / 32];
    const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(vm));
    if ((tid & 31) == 0) wm[tid >> 5] = m;
    __syncthreads();
    if (tid == 0) {
      unsigned mm = wm[0];
#pragma unroll
      for (int i = 1; i < kTpThreads / 32; ++i) mm = max(mm, wm[i]);
      atomicMax(P.vmax + (long)b * 2 * kScal, mm);
    }
  }
}

// ------------------------------------------------------------------ full operator, three inputs
// Row f1's three temporal passes in one ("three linearly independent inputs
// share one G"): reads the stored iterate a and F once per frame and writes
//   out_a = s G_t*(a),  out_b = s G_t*(F^2 a),  out_c = s G_t*(F a)   (s = SC_S),
// 20 B/voxel instead of the 32 B of three single-input passes.  One float2 column per thread
// (three register rings of 2RT+1 float2), 8-byte cp.async prefetch of a and F.
struct Tpass3Params {
  const float* a;          // pitched [B*T][H][Wp]
  const float* F;
  float* out[3];
  unsigned* vmax[3];       // per-output max |out| slots (fp16 spatial pass) or null
  const double* sc;
  // F16 (tcgen05 plain passes): outputs as two fp16 planes of out_c 2^e_c; e_c from the bounds
  // |out_a| <= s gsum max|a|, |out_b| <= s gsum max|F|^2 max|a|, |out_c| <= s gsum max|F| max|a|
  const unsigned* amax_in;   // max |a| (float bits, stride 2 kScal words)
  const unsigned* fmax_in;   // max |F|
  unsigned* amax_zero;       // slot zeroed for the next epilogue's max |a_k| (or null)
  double* vexp_out;          // sc + first exponent slot (stride kScal): e_c at vexp_out[c]
  float gsum;
  long frame2;             // H*Wp/2 float2 per frame
  int T;
  float g[2 * kMaxRT + 1];
  unsigned long long g2[2 * kMaxRT + 1];  // {g[i], g[i]} for fma.rn.f32x2
};

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}

template <int RT, bool F16 = false>
__global__ void __launch_bounds__(kTpThreads) tpass3_kernel(const __grid_constant__ Tpass3Params P) {
  constexpr int NR = 2 * RT + 1;
  constexpr int NS = 8;
  __shared__ float2 sq[NS][2][kTpThreads];
  const int b = blockIdx.y;
  const int tid = threadIdx.x;
  const long e = (long)blockIdx.x * kTpThreads + tid;
  const bool active = e < P.frame2;
  const int T = P.T;
  const long vol2 = (long)T * P.frame2;
  const long ec = active ? e : 0;
  const float2* A = reinterpret_cast<const float2*>(P.a) + b * vol2 + ec;
  const float2* Fp = reinterpret_cast<const float2*>(P.F) + b * vol2 + ec;
  const float scale = (float)P.sc[b * kScal + SC_S];
  float m16[3] = {1.f, 1.f, 1.f};   // F16: s 2^e_c
  if (F16) {
    const float ma = __uint_as_float(P.amax_in[(long)b * 2 * kScal]);
    const float mf = __uint_as_float(P.fmax_in[(long)b * 2 * kScal]);
    const float bound[3] = {scale * ma * P.gsum, scale * mf * mf * ma * P.gsum, scale * mf * ma * P.gsum};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      int ex = 0;
      if (bound[c] > 0.f && bound[c] <= 3.4e38f) frexpf(bound[c], &ex);
      const int e = min(max(kF16DataExp - ex, -100), 100);
      m16[c] = scale * __int_as_float((127 + e) << 23);
      if (blockIdx.x == 0 && tid == 0) P.vexp_out[(long)b * kScal + c] = (double)e;
    }
    if (blockIdx.x == 0 && tid == 0 && P.amax_zero) P.amax_zero[(long)b * 2 * kScal] = 0u;
  }
  const int jend = T + 2 * RT;
  auto issue = [&](int jp) {
    const int j = jp - RT;
    if (jp < jend && j >= 0 && j < T) {
      cp_async8(&sq[jp % NS][0][tid], A + (long)j * P.frame2);
      cp_async8(&sq[jp % NS][1][tid], Fp + (long)j * P.frame2);
    }
    cp_async_commit();
  };
  unsigned long long acc[3][NR];   // packed float2 rings, updated with FFMA2
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int i = 0; i < NR; ++i) acc[c][i] = 0ull;
  float vm[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int d = 0; d < NS; ++d) issue(d);
  for (int j0 = 0; j0 < jend; j0 += NR) {
#pragma unroll
    for (int d = 0; d < NR; ++d) {
      const int jp = j0 + d;
      if (jp >= jend) break;
      cp_async_wait<NS - 1>();
      const int j = jp - RT;
      float2 in[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      if (j >= 0 && j < T) {
        const float2 a = sq[jp % NS][0][tid], f = sq[jp % NS][1][tid];
        in[0] = a;
        in[2] = make_float2(f.x * a.x, f.y * a.y);
        in[1] = make_float2(f.x * in[2].x, f.y * in[2].y);  // F^2 a = F (F a)
      }
      issue(jp + NS);
      const unsigned long long in2[3] = {pack_f2(in[0].x, in[0].y), pack_f2(in[1].x, in[1].y),
                                         pack_f2(in[2].x, in[2].y)};
#pragma unroll
      for (int ee = 0; ee < NR; ++ee) {
        const int slot = (((d - 2 * RT + ee) % NR) + NR) % NR;
        const unsigned long long w2 = P.g2[2 * RT - ee];
#pragma unroll
        for (int c = 0; c < 3; ++c) ffma2(acc[c][slot], w2, in2[c]);
      }
      const int slot0 = (((d - 2 * RT) % NR) + NR) % NR;
      const int t = jp - 2 * RT;
      if (F16 && active && t >= 0 && t < T) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {   // planes [bt][plane][H][Wp] halves: hi, then lo at + frame2
          uint32_t h[2];
          const float2 a2 = unpack_f2(acc[c][slot0]);
          split_planes_f16<2>(a2.x * m16[c], a2.y * m16[c], h);
          uint32_t* o32 = reinterpret_cast<uint32_t*>(P.out[c]) + ((long)b * T + t) * 2 * P.frame2 + ec;
          __stcg(o32, h[0]);
          __stcg(o32 + P.frame2, h[1]);
        }
      } else if (active && t >= 0 && t < T) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float2 a2 = unpack_f2(acc[c][slot0]);
          const float2 o = make_float2(a2.x * scale, a2.y * scale);
          __stcg(reinterpret_cast<float2*>(P.out[c]) + b * vol2 + ec + (long)t * P.frame2, o);
          vm[c] = fmaxf(vm[c], fmaxf(fabsf(o.x), fabsf(o.y)));
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) acc[c][slot0] = 0ull;
    }
  }
  cp_async_wait<0>();
  if (!F16 && P.vmax[0]) {
    __shared__ unsigned wm[3][kTpThreads / 32];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(vm[c]));
      if ((tid & 31) == 0) wm[c][tid >> 5] = m;
    }
    __syncthreads();
    if (tid < 3) {
      unsigned mm = wm[tid][0];
#pragma unroll
      for (int i = 1; i < kTpThreads / 32; ++i) mm = max(mm, wm[tid][i]);
      atomicMax(P.vmax[tid] + (long)b * 2 * kScal, mm);
    }
  }
}

}  // namespace sfseg
