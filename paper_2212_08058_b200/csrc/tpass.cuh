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
  TP_BWD = 1,   // src = F * y_bar_k, y_bar_k = (x_bar_k - F u_{k-1} cn) * inv_nu  (Appendix A)
};

struct TpassParams {
  const float* src;      // FWD: p ; BWD: x_bar_k            pitched [B*T][H][Wp]
  const float* F;        // BWD
  const float* u1;       // BWD: tape u_{k-1}
  const float* halo_lo;  // [B][RT][H][Wp] frames t = -RT..-1 (time slabs) or null
  const float* halo_hi;  // [B][RT][H][Wp] frames t = T..T+RT-1 or null
  float* out;            // pitched [B*T][H][Wp]
  const double* sc;      // per-volume scalars [B][kScal]
  long frame4;           // H*Wp/4 float4 per frame
  int T;
  float g[2 * kMaxRT + 1];  // g[i] = weight of temporal offset i - RT
};

template <int RT, int MODE, bool HALO>
__global__ void __launch_bounds__(256) tpass_kernel(const __grid_constant__ TpassParams P) {
  constexpr int NR = 2 * RT + 1;
  const int b = blockIdx.y;
  const long e = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= P.frame4) return;
  const int T = P.T;
  const long vol4 = (long)T * P.frame4;
  const float4* src = reinterpret_cast<const float4*>(P.src) + b * vol4 + e;
  const float4* Fp = nullptr;
  const float4* U1 = nullptr;
  float cn = 0.f, inv_nu = 0.f, scale = 1.f;
  if (MODE == TP_FWD) {
    scale = (float)P.sc[b * kScal + SC_S];
  } else {
    Fp = reinterpret_cast<const float4*>(P.F) + b * vol4 + e;
    U1 = reinterpret_cast<const float4*>(P.u1) + b * vol4 + e;
    cn = (float)P.sc[b * kScal + SC_CN];
    inv_nu = (float)P.sc[b * kScal + SC_INV_NU];
  }
  const float4* hlo = P.halo_lo ? reinterpret_cast<const float4*>(P.halo_lo) + (long)b * RT * P.frame4 + e : nullptr;
  const float4* hhi = P.halo_hi ? reinterpret_cast<const float4*>(P.halo_hi) + (long)b * RT * P.frame4 + e : nullptr;
  float4* out = reinterpret_cast<float4*>(P.out) + b * vol4 + e;

  float4 acc[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);

  // jp = j + RT enumerates input frames j = -RT .. T+RT-1; output t = jp - 2RT
  // completes when input j = t + RT arrives.  Inputs are software-pipelined NR
  // frames ahead (register queue q[]) so NR loads per thread are in flight.
  auto load = [&](int jp) -> float4 {
    const int j = jp - RT;
    const int jc = min(max(j, 0), T - 1);  // clamped: always a valid address
    float4 val;
    if (MODE == TP_FWD) {
      val = __ldcs(src + (long)jc * P.frame4);
    } else {
      const long o = (long)jc * P.frame4;
      const float4 xb = src[o], f = Fp[o], u = U1[o];
      val.x = f.x * ((xb.x - f.x * u.x * cn) * inv_nu);
      val.y = f.y * ((xb.y - f.y * u.y * cn) * inv_nu);
      val.z = f.z * ((xb.z - f.z * u.z * cn) * inv_nu);
      val.w = f.w * ((xb.w - f.w * u.w * cn) * inv_nu);
    }
    if (HALO) {
      // neighbour slab frames (time-slab sharding); absent halos read as zero
      if (j < 0) val = (hlo != nullptr && j >= -RT) ? hlo[(long)(j + RT) * P.frame4] : make_float4(0.f, 0.f, 0.f, 0.f);
      if (j >= T) val = (hhi != nullptr && j < T + RT) ? hhi[(long)(j - T) * P.frame4] : make_float4(0.f, 0.f, 0.f, 0.f);
    } else if (j < 0 || j >= T) {
      val = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    return val;
  };
  const int jend = T + 2 * RT;
  float4 q[NR];
#pragma unroll
  for (int d = 0; d < NR; ++d) q[d] = load(d);
  for (int j0 = 0; j0 < jend; j0 += NR) {
#pragma unroll
    for (int d = 0; d < NR; ++d) {
      const int jp = j0 + d;
      const float4 val = q[d];
      q[d] = load(jp + NR);  // prefetch (harmless past the end: clamped and zeroed)
#pragma unroll
      for (int ee = 0; ee < NR; ++ee) {
        // input j feeds output t = j - RT + ee with weight g[(j - t) + RT] = g[2RT - ee]
        const int slot = (((d - 2 * RT + ee) % NR) + NR) % NR;
        const float w = P.g[2 * RT - ee];
        acc[slot].x = fmaf(w, val.x, acc[slot].x);
        acc[slot].y = fmaf(w, val.y, acc[slot].y);
        acc[slot].z = fmaf(w, val.z, acc[slot].z);
        acc[slot].w = fmaf(w, val.w, acc[slot].w);
      }
      const int slot0 = (((d - 2 * RT) % NR) + NR) % NR;
      const int t = jp - 2 * RT;
      if (t >= 0 && t < T) out[(long)t * P.frame4] = f4_scale(acc[slot0], scale);
      acc[slot0] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

}  // namespace sfseg
