// Fused spatial pass of G_3D (x then y) + elementwise F multiplies
// + per-iteration norm partials (Eq.8) -- the FP32-FMA-bound kernel of the path.
//
// Persistent, statically balanced: the work is the list of "block units"
// (bt, 64-column strip, 32-row block) ordered bt-major, split into G equal
// contiguous ranges, one per CTA.  A range decomposes into column segments
// (bt, strip, ya..yb); each segment streams 32-row x-blocks through:
//   TMA (cp.async.bulk.tensor.3d, OOB zero fill = zero padding in x and y)
//     -> stage[NST][32 rows][BOXW] (mbarrier complete_tx; thread 0 produces)
//   x-pass: lane = row, 16 consecutive outputs per thread (warp w: columns
//     16w..16w+15, skipped when beyond the image width), (2R+1) taps from the
//     kernel-parameter bank (uniform registers) -> q rows written into a ring,
//     the rows a y window can reach past the wrap written twice (every window
//     contiguous: immediate-offset LDS.128)
//   y-pass: lane = column quad, warp = two row quads, 4x4 outputs per thread
//   epilogue: forward  y = F u ; store p = F y (or y on the last iteration);
//             tape u; partials of ||y||^2 and <p_{k-1}, u> (Rayleigh)
//             backward (Appendix A): x_bar_{k-1} = F v, F_bar += y_bar u_{k-1} + x_{k-1} v,
//             partials of <x_{k-1}, x_bar_{k-1}>
// No x- or y-pass FMA is repeated except one 32-row x-block on each side of a
// mid-column range cut.  The last CTA to finish reduces the per-CTA partials of
// each volume (a contiguous CTA range) in fixed order in fp64 (deterministic)
// and writes the per-volume norm / scale for the next launch.
#pragma once
#include "common.cuh"

namespace sfseg {

constexpr int kMaxRS = 48;

// The TMA box starts at column x0 - RA with RA = round_up(R, 4): a box whose start
// is not 16-byte aligned faults on sm_100a (measured: R % 4 != 0 gave
// "illegal instruction"), so the x-pass reads its taps at offset D = RA - R.
__host__ __device__ constexpr int spass_ra(int R) { return (R + 3) / 4 * 4; }
__host__ __device__ constexpr int spass_boxw(int R) {
  // smallest width >= kTW + 2 RA with width == 4 (mod 8): a row stride of 4*odd floats
  // makes the x-pass LDS.128 (lane = row, 8 lanes per phase) bank-conflict free.
  return ((kTW + 2 * spass_ra(R) - 4 + 7) / 8) * 8 + 4;
}
// x-block grid offset: the grid of 32-row x-blocks starts OFF rows above y_a - R.
// OFF = (-R) mod 32 aligns the grid to image rows (blocks entirely above row 0 or
// below row H are then skipped: no FMAs on zero padding) whenever that costs no
// extra ring slot; otherwise 0.
__host__ __device__ constexpr int spass_off(int R) {
  return ((((32 - R % 32) % 32) + 2 * R + kM - 1) / kM == (2 * R + kM - 1) / kM) ? ((32 - R % 32) % 32) : 0;
}
__host__ __device__ constexpr int spass_pro(int R) { return (spass_off(R) + 2 * R + kM - 1) / kM; }
__host__ __device__ constexpr int spass_nslot(int R) { return spass_pro(R) + 1; }
// Ring rows actually addressed: NSLOT*32 rows plus a duplicate of the first
// (max y-window row + 1 - NSLOT*32) rows, so every y window (4 + 2R rows from
// slot base + OFF + 4rq) is contiguous.  Duplicating only those rows instead of
// the whole ring is what lets two TMA stages and 3 CTAs share an SM (R = 24:
// 152 instead of 192 rows).
__host__ __device__ constexpr int spass_ring_alloc(int R) {
  return (spass_nslot(R) - 1) * kM + spass_off(R) + 31 + 2 * R + 1;
}
__host__ __device__ constexpr size_t spass_smem_for(int R, int stages) {
  return sizeof(float) * ((size_t)stages * kM * spass_boxw(R) + (size_t)spass_ring_alloc(R) * kRingStride) + 2 * 8 +
         8 * 8 + 16;
}
constexpr size_t kSmemPerSM = 227 * 1024;
// TMA stages: double-buffered when 3 CTAs still share an SM (measured at c2, profiles/q11
// vs q12: 3 CTAs x 2 stages 161 us, 4 CTAs x 1 stage 166 us -- occupancy is not the limit).
__host__ __device__ constexpr int spass_fit_n(size_t smem) { return (int)(kSmemPerSM / (smem + 1024)); }
__host__ __device__ constexpr int spass_stages(int R) {
  return spass_fit_n(spass_smem_for(R, 2)) >= 3 ? 2 : 1;
}
__host__ __device__ constexpr size_t spass_smem_bytes(int R) { return spass_smem_for(R, spass_stages(R)); }
__host__ __device__ constexpr int spass_ctas_per_sm(int R) {
  return (int)(kSmemPerSM / (spass_smem_bytes(R) + 1024)) < 4 ? (int)(kSmemPerSM / (spass_smem_bytes(R) + 1024)) : 4;
}

enum SpassMode : int { SP_FWD = 0, SP_BWD = 1 };

struct SpassParams {
  CUtensorMap tmap;        // input volume (v): dims {W, H, B*T}, box {BOXW, kM, 1}, fp32
                           //   (tcgen05 pass: the fp16 planes of v, make_planes_tmap)
  CUtensorMap fmap;        // tcgen05 pass: F, dims {W, H, B*T}, box {128, 64, 1}, fp32
  const float* F;          // pitched [B*T][H][Wp]
  float* out;              // FWD: p (or y when last) ; BWD: x_bar (in place)
  float* tape_u;           // FWD: record u (nullable)
  const float* pprev;      // FWD: p_{k-1} for the Rayleigh quotient (nullable; may alias out)
  const float* u1;         // BWD: tape u_{k-1}
  const float* u2;         // BWD: tape u_{k-2} (k >= 2) or null
  const float* x0p;        // BWD: pitched x_0 when the user gave one (k == 1), else null (x_0 = F)
  float* Fbar;             // BWD: accumulated dL/dF
  double* sc;              // per-volume scalars [B][kScal]
  double* partials;        // [2][B][G]
  unsigned* counter;
  unsigned* err;
  double* stats;           // FWD: [B][K][3] (nullable)
  double* loc;             // time-slab mode: per-volume local sums [B][2] (finalize after the allreduce)
  double* tape_nu;         // FWD writes nu_k; BWD reads nu
  long U;                  // total block units = B*T*S*NB (NB = ceil(H/32))
  int B, T, H, W, Wp, S, NB, G;
  int K, k;                // iteration (FWD) or backward step (BWD), 1-based
  int last;                // FWD: write y instead of p
  int plain;               // FWD: write u = G_s v only (no F multiplies, no norm; full-operator path)
  int t_lo, t_cnt;         // t_cnt > 0: units cover frames [t_lo, t_lo + t_cnt) of every volume only
                           //   (time-slab schedule: boundary frames first, interior after); U = B t_cnt S NB
  int lag;                 // FWD: v came unscaled (lagged normalisation): u *= s_{k-1} = sc[SC_S] here
  int loc_acc;             // time-slab mode: add this launch's sums to loc (later launches of one iteration)
  int vslot;               // fp16 tensor-core pass: max |v| in sc[SC_VMAX + vslot] (written by the temporal
                           //   pass that produced v)
  int vzero;               // > 0: the pass zeroes slot vzero - 1 for the next temporal pass (the slot of
                           //   the other iteration parity); 0: none
  int eslot;               // tcgen05 pass: sc slot of the data exponent e (0: SC_VEXP)
  int pslot;               // tcgen05 pass (spass_tc6): > 0 records max |p_k| per volume into
                           //   sc[SC_VMAX + pslot - 1] (the next TP_FWD16 temporal pass's range); 0: none
  const float* ua;         // full operator, fused combination (spass_tc EPI_FULL): G*(S^p X), G*(F^2 S^p X)
  const float* ub;
  const float* Ufull;      //   S^p
  float inv_alpha;         //   1 / alpha
  int full_epi;            //   the launch selects EPI_FULL
  float g[kMaxRS + 1];     // g[d] = weight of spatial offset +-d (same taps for y and x)
};

// Per-volume finalize of forward iteration k from the global sums s0 = ||y_k||^2 and
// s1 = <p_{k-1}, u_k> (used in-kernel on one GPU, by finalize_kernel after an allreduce).
__device__ __forceinline__ void fwd_finalize(double* sc, double* stats, double* tape_nu, unsigned* err, int K, int k,
                                             bool rayleigh, int b, double s0, double s1) {
  const double nu = sqrt(s0);
  const double xn = sc[SC_XNORM];
  if (stats) {
    double* st = stats + ((long)b * K + (k - 1)) * 3;
    st[0] = nu;
    st[1] = nu / xn;
    st[2] = rayleigh ? sc[SC_S] * s1 / (xn * xn) : 0.0;
  }
  if (tape_nu) tape_nu[(long)b * K + (k - 1)] = nu;
  flag_norm(err, nu);
  sc[SC_S] = 1.0 / nu;
  sc[SC_XNORM] = 1.0;
  sc[SC_NU] = nu;
}

// Backward step k produced x_bar_{k-1}; s0 = c_{k-1} = <x_{k-1}, x_bar_{k-1}>.  When iteration
// k-1 was soft-binarised, x_bar holds g = kappa sigma' b_bar and the caller passes
// s0 = sum(x g) - theta sum(g) (= <x, g - [x > 0] sum(g)/n_pos>) and corr = sum(g) / n_pos.
__device__ __forceinline__ void bwd_finalize(double* sc, const double* tape_nu, int K, int k, int b, double s0,
                                             double corr = 0.0) {
  sc[SC_CORR] = corr;
  if (k >= 2) {
    const double nu1 = tape_nu[(long)b * K + (k - 2)];
    sc[SC_CN] = s0 / nu1;
    sc[SC_INV_NU] = 1.0 / nu1;
    sc[SC_INV_NU_PREV] = (k >= 3) ? 1.0 / tape_nu[(long)b * K + (k - 3)] : 0.0;
  }
}

// Last CTA of a spatial-pass launch: fixed-order fp64 reduction of the per-CTA
// partials of each volume (a contiguous CTA range) and the per-volume finalize.
template <int MODE, int NT>
__device__ __forceinline__ void spass_finalize(const SpassParams& P, double* red, int* flag) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (!last_block_arrive(P.counter, (unsigned)P.G, flag)) return;
  const long per_vol = P.U / P.B;  // units per volume
  // few volumes: the whole CTA sums each volume's partials; many volumes: one warp each
  const bool wide = P.B < NW;
  for (int b = wide ? 0 : warp; b < P.B; b += wide ? 1 : NW) {
    long lo, hi;
    vol_cta_range(b, per_vol, P.U, P.G, lo, hi);
    double s0, s1;
    if (wide) {
      s0 = block_sum_range<NT>(P.partials + (long)b * P.G, lo, hi, 1, red);
      s1 = block_sum_range<NT>(P.partials + (long)(P.B + b) * P.G, lo, hi, 1, red);
    } else {
      s0 = warp_sum_range(P.partials + (long)b * P.G, lo, hi);
      s1 = warp_sum_range(P.partials + (long)(P.B + b) * P.G, lo, hi);
    }
    if ((wide && tid == 0) || (!wide && lane == 0)) {
      if (P.loc) {
        if (P.loc_acc) {  // fixed launch order: deterministic
          P.loc[2 * b] += s0;
          P.loc[2 * b + 1] += s1;
        } else {
          P.loc[2 * b] = s0;
          P.loc[2 * b + 1] = s1;
        }
      } else if (MODE == SP_FWD) {
        fwd_finalize(P.sc + b * kScal, P.stats, P.tape_nu, P.err, P.K, P.k, P.pprev != nullptr, b, s0, s1);
      } else {
        bwd_finalize(P.sc + b * kScal, P.tape_nu, P.K, P.k, b, s0);
      }
    }
  }
  if (tid == 0) *P.counter = 0u;
}

template <int R>
struct SpassGeom {
  static constexpr int BOXW = spass_boxw(R);
  static constexpr int NSLOT = spass_nslot(R);
  static constexpr int RING_ROWS = NSLOT * kM;
  static constexpr int RA = spass_ra(R);
  static constexpr int D = RA - R;                           // tap offset inside the aligned box
  static constexpr int XO = 16;                               // x-pass outputs per thread (one row)
  static constexpr int XIN = ((XO + 2 * R + D) + 3) / 4 * 4;  // x-pass inputs per thread (float4 multiple)
  static_assert(BOXW <= 256, "TMA box width limit");
};

struct Seg {
  int bt, s, yb0, yb1;  // column segment: 32-row output blocks [yb0, yb1) of strip s, frame bt
};

__device__ __forceinline__ Seg seg_decode(long u, long u_end, int NB, int S) {
  Seg g;
  const long col = u / NB;
  g.yb0 = (int)(u - col * NB);
  g.s = (int)(col % S);
  g.bt = (int)(col / S);
  g.yb1 = (int)min((long)NB, (long)g.yb0 + (u_end - u));
  return g;
}
#ifndef SPASS_CHUNK
#define SPASS_CHUNK 0  // A/B: > 0 walks each frame in bands of SPASS_CHUNK blocks across all strips
#endif
// the same with a frame range (P.t_cnt > 0): unit frame index -> volume frame b T + t_lo + t
__device__ __forceinline__ Seg seg_decode(const SpassParams& P, long u, long u_end) {
#if SPASS_CHUNK > 0
  // frame-major; inside a frame, band c (blocks [c CH, c CH + len)) of strip 0, 1, ..., S - 1:
  // horizontally adjacent strips of the same rows run back to back (their x-halo re-reads of
  // v hit L2) at the cost of PRO extra x-blocks per band
  Seg g;
  {
    constexpr int CH = SPASS_CHUNK;
    const int NB = P.NB, S = P.S;
    const long per = (long)S * NB;
    g.bt = (int)(u / per);
    const long r = u - (long)g.bt * per;
    const int c = (int)min(r / ((long)CH * S), (long)((NB - 1) / CH));
    const int len = min(CH, NB - c * CH);
    const long r2 = r - (long)c * CH * S;
    g.s = (int)(r2 / len);
    g.yb0 = c * CH + (int)(r2 - (long)g.s * len);
    g.yb1 = (int)min((long)(c * CH + len), (long)g.yb0 + (u_end - u));
  }
#else
  Seg g = seg_decode(u, u_end, P.NB, P.S);
#endif
  if (P.t_cnt > 0) {
    const int b = g.bt / P.t_cnt;
    g.bt = b * P.T + P.t_lo + (g.bt - b * P.t_cnt);
  }
  return g;
}

// One CTA's walk over the block units [u_begin, u_end) (see the header comment).
// TMA stage parity continues across calls through pseq_io / cseq_io (persistent
// callers such as the megakernel run many ranges per CTA); every load a call
// issues is consumed before it returns.  flush_fn(vol, acc0, acc1) receives each
// thread's fp64 partial sums of ||y||^2 and <p_{k-1}, u> whenever the range
// leaves a volume (collective: all threads call it).
template <int R, int MODE, class FlushFn>
__device__ __forceinline__ void spass_run(const SpassParams& P, long u_begin, long u_end, float* stage, float* ring,
                                          uint64_t* bars, unsigned& pseq_io, unsigned& cseq_io, FlushFn&& flush_fn,
                                          float* out_, const float* pprev_, float* tape_, int last_) {
  using Geo = SpassGeom<R>;
  constexpr int BOXW = Geo::BOXW;
  constexpr int NSLOT = spass_nslot(R);
  constexpr int RING_ROWS = NSLOT * kM;
  constexpr int PRO = spass_pro(R);  // x-blocks written before y-block m = n - PRO runs
  constexpr int OFF = spass_off(R);
  constexpr unsigned STAGE_BYTES = kM * BOXW * sizeof(float);
  constexpr int NST = spass_stages(R);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int H = P.H, W = P.W, Wp = P.Wp, S = P.S, T = P.T, NB = P.NB;

  // ---- producer (thread 0): walks the same (segment, x-block) sequence as the
  // consumers and issues a TMA load for every x-block that overlaps rows [0, H).
  long pu = u_begin;
  Seg pseg{};
  int pn = 0, pnx = 0, pgs = 0;
  unsigned pseq = pseq_io;
  auto producer_next = [&]() {
    while (pu < u_end) {
      if (pn == 0) {
        pseg = seg_decode(P, pu, u_end);
        pnx = (pseg.yb1 - pseg.yb0) + PRO;
        pgs = pseg.yb0 * kM - R - OFF;
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
        tma_load_3d(stage + st * kM * BOXW, &P.tmap, &bars[st], pseg.s * kTW - Geo::RA, row0, pseg.bt);
        return;
      }
    }
  };
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) producer_next();
  }

  double acc0 = 0.0, acc1 = 0.0;  // per-thread partial sums of the current volume
  int cur_vol = -1;
  auto flush = [&](int vol) {
    flush_fn(vol, acc0, acc1);
    acc0 = acc1 = 0.0;
  };

  // per-volume scalars for the backward epilogue (refreshed per volume)
  float cn = 0.f, inv_nu = 0.f, inv_nu_prev = 0.f;
  float lag_s = 1.f;  // forward with lagged normalisation: s_{k-1} of the volume

  unsigned cseq = cseq_io;  // consumed TMA loads (stage / parity)
  long u = u_begin;
  while (u < u_end) {
    const Seg sg = seg_decode(P, u, u_end);
    const int nyb = sg.yb1 - sg.yb0;
    const int nxb = nyb + PRO;
    const int gs = sg.yb0 * kM - R - OFF;
    const int yend = min(sg.yb1 * kM, H);
    const int vol = sg.bt / T;
    if (vol != cur_vol) {
      if (cur_vol >= 0) flush(cur_vol);
      cur_vol = vol;
      if (MODE == SP_FWD && P.lag) lag_s = (float)P.sc[vol * kScal + SC_S];
      if (MODE == SP_BWD) {
        cn = (float)P.sc[vol * kScal + SC_CN];
        inv_nu = (float)P.sc[vol * kScal + SC_INV_NU];
        inv_nu_prev = (float)P.sc[vol * kScal + SC_INV_NU_PREV];
      }
    }

    // ---------------------------------------------------------------- y-pass + epilogue
    // thread: column quad cq (4 columns), row quad rq (4 rows) of the 32-row block
    // y-pass: lane -> columns 4cq..4cq+3 (16 quads span the strip), warp -> two row quads
    // (conflict-free LDS.128 on the stride-68 ring).  Measured faster than giving each warp
    // its own 16 columns (which would let the ragged strip skip y work too): 157 vs 163 us.
    const int cq = lane & 15;
    const int rq = warp * 2 + (lane >> 4);
    const int x = sg.s * kTW + 4 * cq;
    const bool wlive = sg.s * kTW + 16 * warp < W;  // x-pass: this warp's 16 columns exist (ragged strip)
    const bool xok = x < W;
    const bool xfull = x + 4 <= W;
    const float4 msk = make_float4(1.f, (x + 1 < W) ? 1.f : 0.f, (x + 2 < W) ? 1.f : 0.f, (x + 3 < W) ? 1.f : 0.f);
    struct Pre {
      float4 f[4], a[4], c[4], d[4], e[4];  // BWD: a = x_bar, c = u_{k-1}, d = u_{k-2} or x_0, e = F_bar
    };
    // issue the epilogue's global loads early so their latency overlaps the FMAs
    auto prefetch = [&](int m, Pre& pr) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int y = (sg.yb0 + m) * kM + 4 * rq + i;
        pr.f[i] = pr.a[i] = pr.c[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (xok && y < yend && !P.plain) {
          const long off = ((long)sg.bt * H + y) * Wp + x;
          pr.f[i] = *reinterpret_cast<const float4*>(P.F + off);
          if (MODE == SP_FWD) {
            if (pprev_) pr.a[i] = __ldcg(reinterpret_cast<const float4*>(pprev_ + off));
          } else {
            pr.a[i] = *reinterpret_cast<const float4*>(out_ + off);
            pr.c[i] = *reinterpret_cast<const float4*>(P.u1 + off);
            if (P.u2) pr.d[i] = *reinterpret_cast<const float4*>(P.u2 + off);
            else if (P.x0p) pr.d[i] = *reinterpret_cast<const float4*>(P.x0p + off);
            pr.e[i] = *reinterpret_cast<const float4*>(P.Fbar + off);
          }
        }
      }
    };
    auto ypass = [&](int m, const Pre& pr) {
      const float* wb = ring + ((m % NSLOT) * kM + OFF + 4 * rq) * kRingStride + 4 * cq;
      float4 a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 4 + 2 * R; ++j) {
        const float4 q = *reinterpret_cast<const float4*>(wb + j * kRingStride);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int kk = j - i;
          if (kk >= 0 && kk <= 2 * R) {
            const float gk = P.g[kk < R ? R - kk : kk - R];
            a[i].x = fmaf(gk, q.x, a[i].x);
            a[i].y = fmaf(gk, q.y, a[i].y);
            a[i].z = fmaf(gk, q.z, a[i].z);
            a[i].w = fmaf(gk, q.w, a[i].w);
          }
        }
      }
      if (!xok) return;
      float s0 = 0.f, s1 = 0.f;  // this block's 16 outputs: fp32, then one fp64 add
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int y = (sg.yb0 + m) * kM + 4 * rq + i;
        if (y >= yend) break;
        const long off = ((long)sg.bt * H + y) * Wp + x;
        float4 f = pr.f[i];
        float4 uu = (MODE == SP_FWD) ? f4_scale(a[i], lag_s) : a[i];
        if (!xfull) {
          f = f4_mul(f, msk);
          uu = f4_mul(uu, msk);
        }
        if (MODE == SP_FWD && P.plain) {
          *reinterpret_cast<float4*>(out_ + off) = uu;
        } else if (MODE == SP_FWD) {
          const float4 yv = f4_mul(f, uu);
          s0 += f4_dot(yv, yv);
          if (pprev_) s1 += f4_dot(pr.a[i], uu);
          if (tape_) *reinterpret_cast<float4*>(tape_ + off) = uu;
          *reinterpret_cast<float4*>(out_ + off) = last_ ? yv : f4_mul(f, yv);
        } else {
          const float4 xb = pr.a[i];
          const float4 u1 = pr.c[i];
          float4 xp;
          if (P.u2) xp = f4_scale(f4_mul(f, pr.d[i]), inv_nu_prev);
          else if (P.x0p) xp = f4_mul(pr.d[i], msk);
          else xp = f;
          float4 yb;
          yb.x = (xb.x - f.x * u1.x * cn) * inv_nu;
          yb.y = (xb.y - f.y * u1.y * cn) * inv_nu;
          yb.z = (xb.z - f.z * u1.z * cn) * inv_nu;
          yb.w = (xb.w - f.w * u1.w * cn) * inv_nu;
          float4 fb = pr.e[i];
          fb.x += yb.x * u1.x + xp.x * uu.x;
          fb.y += yb.y * u1.y + xp.y * uu.y;
          fb.z += yb.z * u1.z + xp.z * uu.z;
          fb.w += yb.w * u1.w + xp.w * uu.w;
          *reinterpret_cast<float4*>(P.Fbar + off) = fb;
          const float4 xn = f4_mul(f, uu);
          *reinterpret_cast<float4*>(out_ + off) = xn;
          s0 += f4_dot(xp, xn);
        }
      }
      acc0 += (double)s0;
      acc1 += (double)s1;
    };

    for (int n = 0; n < nxb; ++n) {
      const bool do_y = n >= PRO;
      Pre pre;
      // forward: the epilogue's loads before the x-pass; backward (five operands): after it,
      // when the x-pass registers are free (the y-pass still covers their latency)
      if (MODE == SP_FWD && do_y) prefetch(n - PRO, pre);
      const int row0 = gs + n * kM;
      const bool live = (row0 + kM > 0) && (row0 < H);
      const int sl = n % NSLOT;
      float* r0 = ring + (sl * kM + lane) * kRingStride;
      float* r1 = r0 + RING_ROWS * kRingStride;
      const bool dup = sl * kM + lane < spass_ring_alloc(R) - RING_ROWS;  // row also needed past the wrap
      if (live && wlive) {
        const int st = (NST == 2) ? (cseq & 1) : 0;
        mbar_wait(&bars[st], (NST == 2) ? ((cseq >> 1) & 1) : (cseq & 1));
        // ------------------------------------------------------------ x-pass of block n
        // thread: one row (lane) x 16 consecutive columns (warp)
        const float* srow = stage + st * kM * BOXW + lane * BOXW + Geo::XO * warp;
        float in[Geo::XIN];
#pragma unroll
        for (int i = 0; i < Geo::XIN / 4; ++i) {
          const float4 v4 = *reinterpret_cast<const float4*>(srow + 4 * i);
          in[4 * i + 0] = v4.x;
          in[4 * i + 1] = v4.y;
          in[4 * i + 2] = v4.z;
          in[4 * i + 3] = v4.w;
        }
        float a[Geo::XO];
#pragma unroll
        for (int j = 0; j < Geo::XO; ++j) a[j] = 0.f;
#pragma unroll
        for (int kk = 0; kk <= 2 * R; ++kk) {
          const float gk = P.g[kk < R ? R - kk : kk - R];
#pragma unroll
          for (int j = 0; j < Geo::XO; ++j) a[j] = fmaf(gk, in[j + kk + Geo::D], a[j]);
        }
#pragma unroll
        for (int q = 0; q < Geo::XO / 4; ++q) {
          const float4 v = make_float4(a[4 * q], a[4 * q + 1], a[4 * q + 2], a[4 * q + 3]);
          *reinterpret_cast<float4*>(r0 + Geo::XO * warp + 4 * q) = v;
          if (dup) *reinterpret_cast<float4*>(r1 + Geo::XO * warp + 4 * q) = v;
        }
      } else if (wlive) {
        // block entirely in the zero padding above row 0 or below row H-1
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < Geo::XO / 4; ++q) {
          *reinterpret_cast<float4*>(r0 + Geo::XO * warp + 4 * q) = z;
          if (dup) *reinterpret_cast<float4*>(r1 + Geo::XO * warp + 4 * q) = z;
        }
      }
      if (MODE == SP_BWD && do_y) prefetch(n - PRO, pre);
      __syncthreads();  // stage consumed; ring slot visible
      if (live) {
        ++cseq;
        if (tid == 0) {
          fence_proxy_async();
          producer_next();
        }
      }
      if (do_y) ypass(n - PRO, pre);
      __syncthreads();  // ring slot (n+1) % NSLOT may be overwritten next
    }
    u += nyb;
  }
  if (cur_vol >= 0) flush(cur_vol);
  pseq_io = pseq;
  cseq_io = cseq;
}

template <int R, int MODE>
__global__ void __launch_bounds__(kSpassThreads, 3) spass_kernel(const __grid_constant__ SpassParams P) {
  using Geo = SpassGeom<R>;
  constexpr int BOXW = Geo::BOXW;
  constexpr int RING_ROWS = spass_nslot(R) * kM;
  constexpr int NST = spass_stages(R);

  extern __shared__ __align__(128) unsigned char smem[];
  float* stage = reinterpret_cast<float*>(smem);
  float* ring = stage + NST * kM * BOXW;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + spass_ring_alloc(R) * kRingStride);
  double* red = reinterpret_cast<double*>(bars + 2);
  int* flag = reinterpret_cast<int*>(red + 8);

  const int tid = threadIdx.x;
  const long u_begin = (long)blockIdx.x * P.U / P.G;
  const long u_end = (long)(blockIdx.x + 1) * P.U / P.G;

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
    prefetch_tmap(&P.tmap);
  }
  __syncthreads();
  unsigned pseq = 0, cseq = 0;
  spass_run<R, MODE>(P, u_begin, u_end, stage, ring, bars, pseq, cseq, [&](int vol, double a0, double a1) {
    const double s0 = block_sum<kSpassThreads>(a0, red);
    const double s1 = block_sum<kSpassThreads>(a1, red);
    if (tid == 0) {
      P.partials[(long)vol * P.G + blockIdx.x] = s0;
      P.partials[(long)(P.B + vol) * P.G + blockIdx.x] = s1;
    }
  }, P.out, P.pprev, P.tape_u, P.last);

  if (P.plain) return;  // no norm in the plain (full-operator) mode
  spass_finalize<MODE, kSpassThreads>(P, red, flag);
}

}  // namespace sfseg
