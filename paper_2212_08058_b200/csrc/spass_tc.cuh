// Tensor-core spatial pass (forward): the x and y Gaussians of G_3D
// as banded Toeplitz products on the warp-level bf16 tensor pipe (mma.sync
// m16n8k16 -> HMMA), fused with the F multiplies and the norm partials (Eq.8)
// exactly like spass_kernel, which stays the FP32-FMA path (backward, megakernel,
// and SFSEG_ALGO_TWO_PASS_FP32).
//
// Why: at radius 24 the FP32 pass does 98 FMA per voxel and is ALU-bound (49 % of
// the FP32 peak, profiles/r01_final); the tensor pipe does the same contraction
// with 3 bf16 products per tap (measured mma.sync bf16 rate 555 TFLOP/s, 7.5x the
// FP32 peak; tools/mma_microbench.cu, profiles/mma).
//
// Precision (reading A23): every operand a is split into PL = 3 bf16
// planes a = a1 + a2 + a3 (a1 = bf16(a), a2 = bf16(a - a1), a3 = bf16(a - a1 - a2);
// |a - a1 - a2 - a3| <= 2^-27 |a|: the 24-bit fp32 significand in three 8-bit pieces),
// the same for the taps g, and every tap product is the six terms a_i g_j with
// i + j <= 4 (a1g1, a2g1, a1g2, a3g1, a2g2, a1g3; the dropped terms are <= 2^-26 of
// the product), accumulated in fp32 by the tensor core: fp32-class arithmetic
// (per product below the 2^-24 rounding unit of an fp32 FMA).  PL = 2 (three terms,
// ~2^-17) is the round-1 variant, kept compilable for A/B only.
//
// FMT = 1 (forward only, reading A25): two fp16 planes and three products
// (a1g1, a2g1, a1g2).  fp16 keeps 11 significant bits, so two planes carry 22 bits
// (|a - a1 - a2| <= 2^-22 |a|) -- half the tensor work of FMT = 0 -- but only while
// both planes stay in fp16's normal range: the data are scaled per volume by 2^e with
// max |v| < 2^(14 - e) from the temporal pass's max (tpass vmax, SC_VMAX), the taps by
// 2^12 (smallest tap at 3 sigma ~ 2^-11 of the largest stays normal), the x-pass output
// by 2^-12 before it is re-split, and the y-pass output by 2^-(12 + e) (all exact
// powers of two).  Entries below 2^-24 of the volume's max |v| lose relative precision
// (absolute error <= 2^-39 max |v|).
//
// Tiling.  Same work list, segments, TMA producer, ring streaming and finalize as
// spass_kernel (spass.cuh header), with:
//   x-pass: D[16 rows x 8 cols] += A[16 rows x 16 box cols] * Tx[16 x 8]; the
//     Toeplitz slice Tx depends only on the output tile's parity (8-column shift
//     inside a 16-column k block) and the k step, so its bf16 fragments live in
//     registers for the whole kernel; warp w: rows 16 (w & 1).., columns 32 (w >> 1)..
//   ring: x-pass output as PL bf16 planes, row-major, row stride 72
//     (conflict-free u32 stores and ldmatrix); the x-block grid starts R rows above
//     the segment so every y window of a 16-row output tile is 16-aligned and never
//     straddles a 32-row slot: no duplicated rows.
//   y-pass: D[16 out rows x 8 cols] += Ty[16 x 16 ring rows] * Ring[16 x 8]; Ty
//     fragments (shift invariant) in shared memory, Ring fragments by
//     ldmatrix.x4.trans.
#pragma once
#include <cuda_bf16.h>

#include "spass.cuh"

namespace sfseg {

constexpr int kTcRingStride = 72;  // bf16 per ring row (64 + 8: conflict-free)
#ifndef SPTC_PLANES
#define SPTC_PLANES 3
#endif
constexpr int kTcPlanes = SPTC_PLANES;  // bf16 planes per operand (3: fp32-class, 6 products)
static_assert(kTcPlanes == 2 || kTcPlanes == 3, "2 or 3 bf16 planes");
// products (i, j) of plane i of the data and plane j of the taps, largest first
__host__ __device__ constexpr int sptc_nprod() { return kTcPlanes == 3 ? 6 : 3; }
__host__ __device__ constexpr int sptc_pa(int p) { return p == 1 ? 1 : p == 3 ? 2 : p == 4 ? 1 : 0; }
__host__ __device__ constexpr int sptc_pb(int p) { return p == 2 ? 1 : p == 4 ? 1 : p == 5 ? 2 : 0; }

__host__ __device__ constexpr int sptc_nkx(int R) { return (16 + spass_ra(R) + R + 15) / 16; }
__host__ __device__ constexpr int sptc_nky(int R) { return (16 + 2 * R + 15) / 16; }
__host__ __device__ constexpr int sptc_boxw(int R) { return 16 * (3 + sptc_nkx(R)) + 8; }  // == 8 or 24 mod 32
__host__ __device__ constexpr int sptc_pro(int R) { return (31 + 2 * R) / 32; }
#ifndef SPTC_ONEBAR
#define SPTC_ONEBAR 0  // A/B: one more ring slot and one block barrier per 32-row block instead of two
#endif
__host__ __device__ constexpr int sptc_nslot(int R) { return sptc_pro(R) + 1 + SPTC_ONEBAR; }
__host__ __device__ constexpr int sptc_planes(int fmt) { return fmt ? 2 : kTcPlanes; }
__host__ __device__ constexpr size_t sptc_smem_for(int R, int stages, int fmt = 0) {
  return sizeof(float) * (size_t)stages * kM * sptc_boxw(R)                                // TMA stages
         + sptc_planes(fmt) * sizeof(uint16_t) * (size_t)sptc_nslot(R) * kM * kTcRingStride  // ring planes
         + (size_t)sptc_nky(R) * sptc_planes(fmt) * 32 * 16                                   // Ty fragments
         + 2 * 8 + 8 * 8 + 16;
}
#ifndef SPTC_MIN_CTAS
#define SPTC_MIN_CTAS 3
#endif
// two TMA stages when SPTC_MIN_CTAS CTAs still share an SM, else one
__host__ __device__ constexpr int sptc_stages(int R, int fmt = 0) {
  return spass_fit_n(sptc_smem_for(R, 2, fmt)) >= SPTC_MIN_CTAS ? 2 : 1;
}
__host__ __device__ constexpr size_t sptc_smem_bytes(int R, int fmt = 0) {
  return sptc_smem_for(R, sptc_stages(R, fmt), fmt);
}
#ifndef SPTC_LB
#define SPTC_LB 3  // resident CTAs per SM the register budget is sized for (launch bounds)
#endif
__host__ __device__ constexpr int sptc_ctas_per_sm(int R, int fmt = 0) {
  return spass_fit_n(sptc_smem_bytes(R, fmt)) < SPTC_LB ? spass_fit_n(sptc_smem_bytes(R, fmt)) : SPTC_LB;
}

template <int FMT = 0>
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  if (FMT)
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  else
    asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <int FMT, int PL>
__device__ __forceinline__ void tc_split(float a, float b, uint32_t (&o)[PL]) {
  if (FMT) split_planes_f16<PL>(a, b, o);
  else split_planes<PL>(a, b, o);
}
// 2^e as a float for |e| <= 126 (exact)
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + e) << 23); }
constexpr int kF16TapExp = 12;  // FMT = 1: taps scaled by 2^12
#ifndef SPTC_F16_ACC3
#define SPTC_F16_ACC3 0  // A/B: FMT = 1 with the two correction products in separate accumulators
#endif
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                              uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// weight of spatial offset d (zero outside the support), from the shared-memory copy of
// the taps: indexing the kernel-parameter array with a runtime index made the fragment
// setup take ~7 us of a 117 us launch (globaltimer trace, profiles/tc/trace_*)
__device__ __forceinline__ float sptc_w(const float* gsm, int d, int R) {
  const int a = d < 0 ? -d : d;
  return a <= R ? gsm[a] : 0.f;
}

// Epilogue variants (compile-time, so the hot forward carries no dead predicated loads:
// measured 5 % of the instructions were the p_{k-1} loads of the Rayleigh option)
// OPT: tape and/or Rayleigh.  FULL: the full operator's combination (row f1, Eq.7) fused into
// the third spatial pass: y = U [(1/alpha - F^2) ua - ub + 2 F uc] with uc this pass's output,
// a_k = U y (y when last), norm partials of y.
enum SptcEpi : int { EPI_PLAIN = 0, EPI_FWD = 1, EPI_FWD_OPT = 2, EPI_FULL = 3 };

template <int R, int EPI, int FMT>
__global__ void __launch_bounds__(kSpassThreads, SPTC_LB) spass_tc_kernel(const __grid_constant__ SpassParams P) {
  constexpr int BOXW = sptc_boxw(R);
  constexpr int RA = spass_ra(R);
  constexpr int NKX = sptc_nkx(R);
  constexpr int NKY = sptc_nky(R);
  constexpr int PRO = sptc_pro(R);
  constexpr int NSLOT = sptc_nslot(R);
  constexpr int NST = sptc_stages(R, FMT);
  constexpr int RSW = kTcRingStride / 2;  // ring row stride in u32 words
  constexpr int PLANE = NSLOT * kM * RSW;  // words per ring plane
  constexpr unsigned STAGE_BYTES = kM * BOXW * sizeof(float);
  static_assert(BOXW <= 256, "TMA box width limit");
  static_assert(16 * NKY <= 16 + 32 * PRO, "y windows stay inside the live ring slots");

  extern __shared__ __align__(128) unsigned char smem[];
  float* stage = reinterpret_cast<float*>(smem);                          // [NST][32][BOXW]
  constexpr int PL = sptc_planes(FMT);
  constexpr int NPR = FMT ? 3 : sptc_nprod();
  constexpr float TSC = FMT ? (float)(1 << kF16TapExp) : 1.f;  // tap scale
  uint32_t* ring = reinterpret_cast<uint32_t*>(stage + NST * kM * BOXW);  // [PL planes][NSLOT*32][RSW]
  uint4* tyf = reinterpret_cast<uint4*>(ring + PL * PLANE);                // [NKY][PL][32]
  uint64_t* bars = reinterpret_cast<uint64_t*>(tyf + NKY * PL * 32);
  double* red = reinterpret_cast<double*>(bars + 2);
  int* flag = reinterpret_cast<int*>(red + 8);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int mt = warp & 1;  // 16-row half of the 32-row block
  const int hh = warp >> 1; // 32-column half of the 64-column strip
  const int H = P.H, W = P.W, Wp = P.Wp, S = P.S, T = P.T, NB = P.NB;
  const long u_begin = (long)blockIdx.x * P.U / P.G;
  const long u_end = (long)(blockIdx.x + 1) * P.U / P.G;

  __shared__ float gsm[kMaxRS + 1];
  if (tid <= R) gsm[tid] = P.g[tid];
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
    prefetch_tmap(&P.tmap);
  }
  __syncthreads();
  // Ty fragments (A operand of the y-pass): A[i][kk] = w(16 s + kk - i - R)
  for (int idx = tid; idx < NKY * PL * 32; idx += kSpassThreads) {
    const int s = idx / (32 * PL), pl = (idx >> 5) % PL, l = idx & 31;
    const int gi = l >> 2, ti = l & 3;
    uint32_t v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = gi + 8 * (j & 1);
      const int kk = 16 * s + 2 * ti + 8 * (j >> 1);
      uint32_t pp[PL];
      tc_split<FMT, PL>(TSC * sptc_w(gsm, kk - i - R, R), TSC * sptc_w(gsm, kk + 1 - i - R, R), pp);
      v[j] = pp[pl];
    }
    tyf[idx] = make_uint4(v[0], v[1], v[2], v[3]);
  }
  // Tx fragments (B operand of the x-pass), registers: B[kk][jj] = w(16 s + kk - jj - 8 par - RA)
  uint32_t bx[PL][2][NKX][2];
#pragma unroll
  for (int par = 0; par < 2; ++par)
#pragma unroll
    for (int s = 0; s < NKX; ++s)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int d = 16 * s + 2 * t + 8 * j - g - 8 * par - RA;
        uint32_t pp[PL];
        tc_split<FMT, PL>(TSC * sptc_w(gsm, d, R), TSC * sptc_w(gsm, d + 1, R), pp);
#pragma unroll
        for (int q = 0; q < PL; ++q) bx[q][par][s][j] = pp[q];
      }
  if (FMT && P.vzero > 0 && blockIdx.x == 0 && tid == 0) {
    // the slot the NEXT temporal pass will max into (this pass's slot, vslot, was filled
    // by the temporal pass that produced v)
    for (int b = 0; b < P.B; ++b) *reinterpret_cast<unsigned*>(P.sc + b * kScal + SC_VMAX + P.vzero - 1) = 0u;
  }
  __syncthreads();

  // ---- producer (thread 0): the x-block sequence of the CTA's unit range
  long pu = u_begin;
  Seg pseg{};
  int pn = 0, pnx = 0, pgs = 0;
  unsigned pseq = 0;
  auto producer_next = [&]() {
    while (pu < u_end) {
      if (pn == 0) {
        pseg = seg_decode(P, pu, u_end);
        pnx = (pseg.yb1 - pseg.yb0) + PRO;
        pgs = pseg.yb0 * kM - R;
      }
      const int row0 = pgs + pn * kM;
      if (++pn == pnx) {
        pn = 0;
        pu += pseg.yb1 - pseg.yb0;
      }
      if (row0 + kM > 0 && row0 < H) {
        const int st = (NST == 2) ? (pseq & 1) : 0;
        ++pseq;
        mbar_arrive_expect_tx(&bars[st], STAGE_BYTES);
        tma_load_3d(stage + st * kM * BOXW, &P.tmap, &bars[st], pseg.s * kTW - RA, row0, pseg.bt);
        return;
      }
    }
  };
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) producer_next();
  }

  constexpr bool plain = EPI == EPI_PLAIN;
  float* const out = P.out;
  const float* const pprev = EPI == EPI_FWD_OPT ? P.pprev : nullptr;
  float* const tape = EPI == EPI_FWD_OPT ? P.tape_u : nullptr;
  const int last = P.last;
  double acc0 = 0.0, acc1 = 0.0;
  int cur_vol = -1;
  float dsc = 1.f, usc = 1.f;  // FMT = 1: data scale 2^e and output scale 2^-(12 + e) (x s_{k-1} when lagged)
  float lag_s = 1.f;           // FMT = 0: s_{k-1} of the volume when the normalisation is lagged (else 1)
  auto flush = [&](int vol) {
    const double s0 = block_sum<kSpassThreads>(acc0, red);
    const double s1 = block_sum<kSpassThreads>(acc1, red);
    if (tid == 0) {
      P.partials[(long)vol * P.G + blockIdx.x] = s0;
      P.partials[(long)(P.B + vol) * P.G + blockIdx.x] = s1;
    }
    acc0 = acc1 = 0.0;
  };
  // ldmatrix lane address parts: matrix mi = lane >> 3 (k half = mi & 1, n tile = mi >> 1)
  const int lm_row = (lane & 7) + 8 * ((lane >> 3) & 1);
  const int lm_nt = lane >> 4;
  const uint32_t ring_s = smem_u32(ring);

  unsigned cseq = 0;
  long u = u_begin;
  while (u < u_end) {
    const Seg sg = seg_decode(P, u, u_end);
    const int nyb = sg.yb1 - sg.yb0;
    const int nxb = nyb + PRO;
    const int gs = sg.yb0 * kM - R;
    const int yend = min(sg.yb1 * kM, H);
    const int vol = sg.bt / T;
    if (vol != cur_vol) {
      if (cur_vol >= 0) flush(cur_vol);
      cur_vol = vol;
      if (!plain && P.lag) lag_s = (float)P.sc[vol * kScal + SC_S];
      if (FMT) {
        const float vmax = __uint_as_float(*reinterpret_cast<const unsigned*>(P.sc + vol * kScal + SC_VMAX + P.vslot));
        int ex = 0;
        if (vmax > 0.f && vmax <= 3.4e38f) frexpf(vmax, &ex);  // max |v| < 2^ex
        const int e = min(max(14 - ex, -100), 100);
        dsc = pow2f(e);
        usc = pow2f(-e - kF16TapExp) * lag_s;
      }
    }
    const int c0 = sg.s * kTW;
    const bool wlive = c0 + 32 * hh < W;  // this warp's 32 columns exist (ragged strip)

    // epilogue geometry: thread element (nl, i) = row 16 mt + g + 8 i, column c0 + 32 hh + 8 nl + 2 t
    const int xt = c0 + 32 * hh + 2 * t;
    float2 cmask[4];  // columns < W (pad columns and beyond: 0)
    bool cst[4];      // pair inside the pitched row (store allowed)
#pragma unroll
    for (int nl = 0; nl < 4; ++nl) {
      const int x = xt + 8 * nl;
      cst[nl] = x < Wp;
      cmask[nl] = make_float2(x < W ? 1.f : 0.f, x + 1 < W ? 1.f : 0.f);
    }
    struct Pre {
      float2 f[4][2], a[4][2];
    };
    auto row_base = [&](int m) -> long { return ((long)sg.bt * H + (sg.yb0 + m) * kM + 16 * mt + g) * Wp + xt; };
    auto prefetch = [&](int m, Pre& pr) {
      const int yb = (sg.yb0 + m) * kM + 16 * mt + g;
      const long base = row_base(m);
      const float* fb = P.F + base;
      const float* ab = EPI == EPI_FULL ? P.Ufull + base : pprev + base;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const bool rok = yb + 8 * i < yend;
#pragma unroll
        for (int nl = 0; nl < 4; ++nl) {
          pr.f[nl][i] = pr.a[nl][i] = make_float2(0.f, 0.f);
          if (!plain && rok && cst[nl]) {
            pr.f[nl][i] = *reinterpret_cast<const float2*>(fb + (long)8 * i * Wp + 8 * nl);
            if ((EPI == EPI_FWD_OPT && pprev) || EPI == EPI_FULL)
              pr.a[nl][i] = __ldcg(reinterpret_cast<const float2*>(ab + (long)8 * i * Wp + 8 * nl));
          }
        }
      }
    };
    auto ypass = [&](int m, const Pre& pr) {
      // acc: the leading product (plane 1 x plane 1) only; acs: the five correction products.
      // The tensor core truncates each accumulation to the accumulator's magnitude, so the
      // corrections (<= 2^-8 of the result) are summed in their own accumulator and added
      // with one round-to-nearest FADD: 4 instead of 24 full-magnitude truncations per pass.
      constexpr bool A3 = FMT && SPTC_F16_ACC3;
      float acc[4][4], acs[4][4], ac2[A3 ? 4 : 1][4];
#pragma unroll
      for (int nl = 0; nl < 4; ++nl)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[nl][i] = acs[nl][i] = 0.f;
          if (A3) ac2[A3 ? nl : 0][i] = 0.f;
        }
      // ring slot of each x-block of this y window (x-blocks m .. m + PRO)
      uint32_t slot_addr[PRO + 1];
      {
        const int sm = m % NSLOT;
#pragma unroll
        for (int j = 0; j <= PRO; ++j) {
          const int sj = sm + j < NSLOT ? sm + j : sm + j - NSLOT;
          slot_addr[j] = ring_s + 4u * (uint32_t)((sj * kM + lm_row) * RSW + 4 * (4 * hh + lm_nt));
        }
      }
#pragma unroll
      for (int s = 0; s < NKY; ++s) {
        uint4 ay[PL];
#pragma unroll
        for (int q = 0; q < PL; ++q) ay[q] = tyf[(PL * s + q) * 32 + lane];
        // window rows 16 mt + 16 s ..: x-block (16 mt + 16 s) >> 5 of the window, mt runtime
        const uint32_t sa = (mt ? slot_addr[(16 + 16 * s) >> 5] + 4u * (uint32_t)(((16 + 16 * s) & 31) * RSW)
                                : slot_addr[(16 * s) >> 5] + 4u * (uint32_t)(((16 * s) & 31) * RSW));
        uint32_t bq[PL][8];  // B fragments of the four n tiles (2 regs each), per ring plane
#pragma unroll
        for (int q = 0; q < PL; ++q)
#pragma unroll
          for (int pp = 0; pp < 2; ++pp) {
            const uint32_t addr = sa + 4u * (uint32_t)(8 * pp + q * PLANE);
            ldsm_x4_trans(addr, bq[q][4 * pp], bq[q][4 * pp + 1], bq[q][4 * pp + 2], bq[q][4 * pp + 3]);
          }
        // product-major order: consecutive HMMAs write different accumulators.  Here the
        // taps are the A operand: product (i, j) = data plane i (B) x tap plane j (A).
#pragma unroll
        for (int p = 0; p < NPR; ++p)
#pragma unroll
          for (int nl = 0; nl < 4; ++nl) {
            const uint4& a = ay[sptc_pb(p)];
            mma16816<FMT>(p == 0 ? acc[nl] : (A3 && p == 2) ? ac2[A3 ? nl : 0] : acs[nl], a.x, a.y, a.z, a.w,
                          bq[sptc_pa(p)][2 * nl], bq[sptc_pa(p)][2 * nl + 1]);
          }
      }
#pragma unroll
      for (int nl = 0; nl < 4; ++nl)
#pragma unroll
        for (int i = 0; i < 4; ++i)
          acc[nl][i] = (acc[nl][i] + (A3 ? acs[nl][i] + ac2[A3 ? nl : 0][i] : acs[nl][i])) * (FMT ? usc : lag_s);
      // epilogue
      float s0 = 0.f, s1 = 0.f;
      const int yb = (sg.yb0 + m) * kM + 16 * mt + g;
      const long base = row_base(m);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const bool rok = yb + 8 * i < yend;
#pragma unroll
        for (int nl = 0; nl < 4; ++nl) {
          if (!(rok && cst[nl])) continue;
          const long off = base + (long)8 * i * Wp + 8 * nl;
          // columns >= W: the forward's outputs are F * (...) and F is zero there (combine
          // writes zero pad columns), so only the plain / tape / Rayleigh variants mask u
          const float2 uu = EPI == EPI_FWD ? make_float2(acc[nl][2 * i], acc[nl][2 * i + 1])
                                           : make_float2(acc[nl][2 * i] * cmask[nl].x, acc[nl][2 * i + 1] * cmask[nl].y);
          if (plain) {
            *reinterpret_cast<float2*>(out + off) = uu;
            continue;
          }
          const float2 f = pr.f[nl][i];
          if (EPI == EPI_FULL) {
            const float2 U = pr.a[nl][i];
            const float2 ua = __ldcs(reinterpret_cast<const float2*>(P.ua + off));
            const float2 ub = __ldcs(reinterpret_cast<const float2*>(P.ub + off));
            const float vx = (P.inv_alpha - f.x * f.x) * ua.x - ub.x + 2.f * f.x * uu.x;
            const float vy = (P.inv_alpha - f.y * f.y) * ua.y - ub.y + 2.f * f.y * uu.y;
            const float2 yv = make_float2(U.x * vx * cmask[nl].x, U.y * vy * cmask[nl].y);
            s0 = fmaf(yv.x, yv.x, fmaf(yv.y, yv.y, s0));
            *reinterpret_cast<float2*>(out + off) = last ? yv : make_float2(U.x * yv.x, U.y * yv.y);
            continue;
          }
          const float2 yv = make_float2(f.x * uu.x, f.y * uu.y);
          s0 = fmaf(yv.x, yv.x, fmaf(yv.y, yv.y, s0));
          if (EPI == EPI_FWD_OPT && pprev) s1 = fmaf(pr.a[nl][i].x, uu.x, fmaf(pr.a[nl][i].y, uu.y, s1));
          if (EPI == EPI_FWD_OPT && tape) *reinterpret_cast<float2*>(tape + off) = uu;
          *reinterpret_cast<float2*>(out + off) = last ? yv : make_float2(f.x * yv.x, f.y * yv.y);
        }
      }
      acc0 += (double)s0;
      acc1 += (double)s1;
    };

    for (int n = 0; n < nxb; ++n) {
      const bool do_y = n >= PRO;
      Pre pre;
      if (do_y && wlive) prefetch(n - PRO, pre);
      const int row0 = gs + n * kM;
      const bool live = (row0 + kM > 0) && (row0 < H);
      const int slot_row = (n % NSLOT) * kM + 16 * mt + g;
      if (wlive) {
        constexpr bool A3 = FMT && SPTC_F16_ACC3;
        float acc[4][4], acs[4][4], ac2[A3 ? 4 : 1][4];  // leading product / corrections (see the y-pass)
#pragma unroll
        for (int nl = 0; nl < 4; ++nl)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            acc[nl][i] = acs[nl][i] = 0.f;
            if (A3) ac2[A3 ? nl : 0][i] = 0.f;
          }
        if (live) {
          const int st = (NST == 2) ? (cseq & 1) : 0;
          mbar_wait(&bars[st], (NST == 2) ? ((cseq >> 1) & 1) : (cseq & 1));
          // ------------------------------------------------------------ x-pass (tensor cores)
          const float* sb = stage + st * kM * BOXW + (16 * mt + g) * BOXW + 2 * t;
          // k block kb = 2 hh + j (j = 0 .. NKX) feeds n tiles 2q, 2q + 1 of the pairs
          // q = 2 hh + qq with step s = j - qq: each block is loaded and split once
#pragma unroll
          for (int j = 0; j <= NKX; ++j) {
            const float* p0 = sb + 16 * (2 * hh + j);
            float2 v00 = *reinterpret_cast<const float2*>(p0);
            float2 v10 = *reinterpret_cast<const float2*>(p0 + 8 * BOXW);
            float2 v01 = *reinterpret_cast<const float2*>(p0 + 8);
            float2 v11 = *reinterpret_cast<const float2*>(p0 + 8 * BOXW + 8);
            if (FMT) {
              v00 = make_float2(v00.x * dsc, v00.y * dsc);
              v10 = make_float2(v10.x * dsc, v10.y * dsc);
              v01 = make_float2(v01.x * dsc, v01.y * dsc);
              v11 = make_float2(v11.x * dsc, v11.y * dsc);
            }
            uint32_t a0[PL], a1[PL], a2[PL], a3[PL];
            tc_split<FMT, PL>(v00.x, v00.y, a0);
            tc_split<FMT, PL>(v10.x, v10.y, a1);
            tc_split<FMT, PL>(v01.x, v01.y, a2);
            tc_split<FMT, PL>(v11.x, v11.y, a3);
            // product-major order: consecutive HMMAs write different accumulators
#pragma unroll
            for (int p = 0; p < NPR; ++p)
#pragma unroll
              for (int qq = 0; qq < 2; ++qq) {
                const int s = j - qq;
                if (s < 0 || s >= NKX) continue;
#pragma unroll
                for (int par = 0; par < 2; ++par) {
                  float(&d)[4] = p == 0 ? acc[2 * qq + par]
                                 : (A3 && p == 2) ? ac2[A3 ? 2 * qq + par : 0] : acs[2 * qq + par];
                  const int qa = sptc_pa(p);
                  const uint32_t* bb = bx[sptc_pb(p)][par][s];
                  mma16816<FMT>(d, a0[qa], a1[qa], a2[qa], a3[qa], bb[0], bb[1]);
                }
              }
          }
        }
        // x-pass output (or the zero padding of a block outside rows [0, H)) -> ring planes
#pragma unroll
        for (int nl = 0; nl < 4; ++nl) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            acc[nl][i] = FMT ? (acc[nl][i] + (A3 ? acs[nl][i] + ac2[A3 ? nl : 0][i] : acs[nl][i])) *
                                   (1.f / (float)(1 << kF16TapExp))
                             : acc[nl][i] + acs[nl][i];
          const int w0 = slot_row * RSW + 4 * (4 * hh + nl) + t;
          uint32_t q0[PL], q1[PL];
          tc_split<FMT, PL>(acc[nl][0], acc[nl][1], q0);
          tc_split<FMT, PL>(acc[nl][2], acc[nl][3], q1);
#pragma unroll
          for (int q = 0; q < PL; ++q) {
            ring[q * PLANE + w0] = q0[q];
            ring[q * PLANE + w0 + 8 * RSW] = q1[q];
          }
        }
      }
      __syncthreads();  // stage consumed; ring slot visible
      if (live) {
        ++cseq;
        // no proxy fence: the stage was only READ through the generic proxy, and every
        // read completed before the barrier (write-after-read needs no cross-proxy fence)
        if (tid == 0) producer_next();
      }
      if (do_y && wlive) ypass(n - PRO, pre);
      // ring slot (n + 1) % NSLOT may be overwritten next.  SPTC_ONEBAR: that slot held x-block
      // n - PRO - 1, whose last reader (the y-pass of the previous iteration) every warp finished
      // before the barrier above, so no second barrier is needed
      if (!SPTC_ONEBAR) __syncthreads();
    }
    u += nyb;
  }
  if (cur_vol >= 0) flush(cur_vol);

  if (plain) return;
  spass_finalize<SP_FWD, kSpassThreads>(P, red, flag);
}

}  // namespace sfseg
