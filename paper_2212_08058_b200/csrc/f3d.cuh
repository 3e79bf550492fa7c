// Single-pass fused 3D iteration for SMALL radii (r_t <= 3, r_s <= 8): the
// paper's own 3x7x7 support (the "probe" workload) and config 1.
//
//   u = s * G_y G_x G_t p_{k-1},  y_k = F u,  p_k = F y_k   (Eq.7 with p = 1,
//   Eq.8 normalisation carried as the scalar s = 1/nu_{k-1})
//
// For small stencils the iteration is HBM-bound (21 FMA per 12
// algorithmic bytes at the probe), so the design goal is to touch HBM once per
// operand: read p_{k-1} and F, write p_k -- 12 B per voxel-iteration.  The
// two-pass design (tpass + spass) moves 20 B.
//
// A CTA owns a spatial tile (64 output columns x TH output rows) and streams it
// through time: every frame of p_{k-1} is TMA-loaded ONCE as a (TH + 2R) x BOXW
// box (OOB zero fill = the zero padding of reading A8) into a ring of
// 2RT+1+NPF stages; output frame t combines the 2RT+1 resident boxes of frames
// t-RT..t+RT (temporal taps), then the x-pass (lane = box row, warp = 16
// columns) and y-pass (lane = 4 rows x 4 columns) run from a per-warp q
// buffer -- no block barrier in the loop (warps meet only at the stage ring).
// The work list (volume, tile, frame) is split into G equal contiguous ranges
// (static balance); a range is a few runs of consecutive frames of one tile,
// each run re-loading only the 2RT boundary frames it shares with its
// neighbour run.  p_{k-1} and p_k are distinct buffers (ping-pong): a box of
// frame t is read by other tiles' halos and by frames t+-RT.
#pragma once
#include "common.cuh"
#include "spass.cuh"  // fwd_finalize

namespace sfseg {

constexpr int kF3dTW = 64;               // output columns per tile
constexpr int kF3dCW = 4;                // compute warps (16 columns each)
constexpr int kF3dXO = kF3dTW / kF3dCW;  // 16
constexpr int kF3dQS = kF3dXO + 4;       // per-warp q row stride (floats): 20 -> conflict-free LDS/STS.128
constexpr int kF3dThreads = (kF3dCW + 1) * 32;  // + one TMA producer warp
constexpr int kF3dMaxRT = 3;
constexpr int kF3dMaxR = 8;
constexpr int kF3dNPF = 3;  // frames prefetched beyond the 2RT+1 the current output needs

__host__ __device__ constexpr int f3d_ra(int R) { return (R + 3) / 4 * 4; }
// box width >= 64 + 2 RA with width == 4 (mod 8): conflict-free x-pass LDS.128 (lane = row)
__host__ __device__ constexpr int f3d_boxw(int R) { return ((kF3dTW + 2 * f3d_ra(R) - 4 + 7) / 8) * 8 + 4; }
__host__ __device__ constexpr int f3d_th(int R) { return ((32 - 2 * R) / 4) * 4; }  // output rows per tile
__host__ __device__ constexpr int f3d_stages(int RT) { return 2 * RT + 1 + kF3dNPF; }
__host__ __device__ constexpr size_t f3d_smem_bytes(int RT, int R) {
  return sizeof(float) * ((size_t)f3d_stages(RT) * (kM * f3d_boxw(R) + f3d_th(R) * kF3dTW) + (size_t)kF3dCW * kM * kF3dQS) +
         2 * 8 * f3d_stages(RT) + 16 + 16 * kF3dCW;
}
__host__ __device__ constexpr int f3d_fit(size_t smem) {
  return (int)((227 * 1024) / (smem + 1024)) < 4 ? (int)((227 * 1024) / (smem + 1024)) : 4;
}
__host__ __device__ constexpr int f3d_ctas_per_sm(int RT, int R) {
  return f3d_fit(f3d_smem_bytes(RT, R)) < 1 ? 1 : f3d_fit(f3d_smem_bytes(RT, R));
}

struct F3dParams {
  CUtensorMap tmap;        // p_{k-1}: dims {W, H, B*T}, box {BOXW, 32, 1}, fp32, pitched rows (Wp)
  CUtensorMap fmap;        // F: dims {W, H, B*T}, box {64, TH, 1}, fp32, pitched rows (Wp)
  const float* F;          // pitched [B*T][H][Wp]
  float* out;              // p_k (or y_k when last), pitched; must not alias the tmap source
  float* tape_u;           // record u (nullable)
  double* sc;              // per-volume scalars [B][kScal]  (SC_S = s_{k-1} read; finalize writes s_k)
  double* partials;        // [2][B][G] (one slot per CTA)
  unsigned* counter;
  unsigned* err;
  double* stats;           // [B][K][3] (nullable)
  double* tape_nu;         // nu_k (nullable)
  long U;                  // total units = B * TY * TX * T
  int B, T, H, W, Wp, TX, TY, G;
  int K, k, last, rayleigh;
  unsigned long long* trace;    // debug (SFSEG_F3D_TRACE): per CTA {smid, t_start, t_compute_end, t_end} or null
  float gt[2 * kF3dMaxRT + 1];  // temporal taps g_t[o + RT]
  float gs[kF3dMaxR + 1];       // spatial taps g_s[|d|]
};

struct F3dSeg {
  int b, ty, tx, t0, t1;  // frames [t0, t1) of tile (ty, tx) of volume b
};

__device__ __forceinline__ void f3d_compute_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kF3dCW * 32) : "memory");
}
__device__ __forceinline__ void f3d_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// OPT: the epilogue has a tape and/or the Rayleigh operand (compile-time, so the plain
// forward carries no predicated-off work; the same change measured 4 % on spass_tc)
template <int RT, int R, bool OPT>
__global__ void __launch_bounds__(kF3dThreads, f3d_ctas_per_sm(RT, R)) f3d_kernel(const __grid_constant__ F3dParams P) {
  constexpr int BOXW = f3d_boxw(R);
  constexpr int RA = f3d_ra(R);
  constexpr int D = RA - R;
  constexpr int TH = f3d_th(R);
  constexpr int NS = f3d_stages(RT);
  constexpr int XIN = ((kF3dXO + 2 * R + D) + 3) / 4 * 4;
  constexpr unsigned PBOX_BYTES = kM * BOXW * sizeof(float);
  constexpr unsigned FBOX_BYTES = TH * kF3dTW * sizeof(float);
  constexpr int STAGE_FLOATS = kM * BOXW + TH * kF3dTW;  // p box, then (output frames only) the F tile
  static_assert(TH + 2 * R <= kM, "box rows");

  extern __shared__ __align__(128) unsigned char smem[];
  float* stage = reinterpret_cast<float*>(smem);
  float* qbuf = stage + NS * STAGE_FLOATS;
  uint64_t* full = reinterpret_cast<uint64_t*>(qbuf + kF3dCW * kM * kF3dQS);
  uint64_t* empty = full + NS;
  int* flag = reinterpret_cast<int*>(empty + NS);
  double* red = reinterpret_cast<double*>(flag + 4);  // 2 * kF3dCW doubles (partial fold, finalize)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = P.T, H = P.H, W = P.W, Wp = P.Wp;
  const long per_tile = T;
  const long u_begin = (long)blockIdx.x * P.U / P.G;
  const long u_end = (long)(blockIdx.x + 1) * P.U / P.G;
  auto decode = [&](long u) {
    F3dSeg s;
    const long tile = u / per_tile;
    s.t0 = (int)(u - tile * per_tile);
    s.t1 = (int)min((long)T, (long)s.t0 + (u_end - u));
    s.tx = (int)(tile % P.TX);
    const long r = tile / P.TX;
    s.ty = (int)(r % P.TY);
    s.b = (int)(r / P.TY);
    return s;
  };

  unsigned long long tr_start = 0;
  if (P.trace && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_start));
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kF3dCW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kF3dCW) {
    // ---------------------------------------------------------------- producer: one TMA box per frame
    if (lane == 0) {
      prefetch_tmap(&P.tmap);
      prefetch_tmap(&P.fmap);
      unsigned seq = 0;
      long u = u_begin;
      while (u < u_end) {
        const F3dSeg sg = decode(u);
        const int jlo = max(0, sg.t0 - RT), jhi = min(T, sg.t1 + RT);
        for (int j = jlo; j < jhi; ++j) {
          const int st = (int)(seq % NS);
          if (seq >= (unsigned)NS) mbar_wait(&empty[st], ((seq / NS) - 1) & 1);
          const bool outf = j >= sg.t0 && j < sg.t1;  // an output frame of this run: also needs F
          mbar_arrive_expect_tx(&full[st], PBOX_BYTES + (outf ? FBOX_BYTES : 0u));
          float* sb = stage + st * STAGE_FLOATS;
          tma_load_3d(sb, &P.tmap, &full[st], sg.tx * kF3dTW - RA, sg.ty * TH - R, sg.b * T + j);
          if (outf) tma_load_3d(sb + kM * BOXW, &P.fmap, &full[st], sg.tx * kF3dTW, sg.ty * TH, sg.b * T + j);
          ++seq;
        }
        u += sg.t1 - sg.t0;
      }
    }
    return;
  }

  // ------------------------------------------------------------------ compute warps
  float* q = qbuf + warp * (kM * kF3dQS);
  const int rq = lane >> 2, cq = lane & 3;
  double acc0 = 0.0, acc1 = 0.0;
  int cur_vol = -1;
  float s = 1.f;
  const long nslots = (long)P.G;  // partial slots per volume (one per CTA)
  // one partial per CTA and volume (the last CTA then sums G, not G*4, values): the four
  // compute warps reach the same volume boundaries, so the fold is a named-barrier step
  auto flush = [&](int vol) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc0 += __shfl_xor_sync(0xffffffffu, acc0, o);
      acc1 += __shfl_xor_sync(0xffffffffu, acc1, o);
    }
    f3d_compute_bar();  // red[] free (previous fold done)
    if (lane == 0) {
      red[2 * warp] = acc0;
      red[2 * warp + 1] = acc1;
    }
    f3d_compute_bar();
    if (tid == 0) {
      double t0 = 0.0, t1 = 0.0;
      for (int w = 0; w < kF3dCW; ++w) {
        t0 += red[2 * w];
        t1 += red[2 * w + 1];
      }
      P.partials[(long)vol * nslots + blockIdx.x] = t0;
      P.partials[(long)(P.B + vol) * nslots + blockIdx.x] = t1;
    }
    acc0 = acc1 = 0.0;
  };

  unsigned waited = 0, released = 0;  // stage sequence numbers (same order as the producer)
  long u = u_begin;
  while (u < u_end) {
    const F3dSeg sg = decode(u);
    if (sg.b != cur_vol) {
      if (cur_vol >= 0) flush(cur_vol);
      cur_vol = sg.b;
      s = (float)P.sc[sg.b * kScal + SC_S];
    }
    const int jlo = max(0, sg.t0 - RT), jhi = min(T, sg.t1 + RT);
    const unsigned base = waited;  // sequence number of frame jlo
    const int xw = sg.tx * kF3dTW + kF3dXO * warp;
    const bool wlive = xw < W;
    const int x = xw + 4 * cq;
    const bool xok = x < W && 4 * rq < TH;
    const bool xfull = x + 4 <= W;
    const float4 msk = make_float4(1.f, (x + 1 < W) ? 1.f : 0.f, (x + 2 < W) ? 1.f : 0.f, (x + 3 < W) ? 1.f : 0.f);
    const int y0 = sg.ty * TH + 4 * rq;

    for (int t = sg.t0; t < sg.t1; ++t) {
      // frames t-RT..t+RT (clipped to [jlo, jhi)) must be resident
      const int jneed = min(jhi - 1, t + RT);
      while ((int)(waited - base) + jlo <= jneed) {
        mbar_wait(&full[waited % NS], (waited / NS) & 1);
        ++waited;
      }
      if (wlive) {
        // ---------------------------------------------------------- temporal taps + x-pass
        float vin[XIN];
#pragma unroll
        for (int i = 0; i < XIN; ++i) vin[i] = 0.f;
#pragma unroll
        for (int o = -RT; o <= RT; ++o) {
          const int j = t + o;
          if (j < jlo || j >= jhi) continue;  // zero padding in time (warp-uniform)
          const float* srow = stage + ((base + (unsigned)(j - jlo)) % NS) * STAGE_FLOATS + lane * BOXW + kF3dXO * warp;
          const float gt = P.gt[o + RT];
#pragma unroll
          for (int i = 0; i < XIN / 4; ++i) {
            const float4 v4 = *reinterpret_cast<const float4*>(srow + 4 * i);
            vin[4 * i + 0] = fmaf(gt, v4.x, vin[4 * i + 0]);
            vin[4 * i + 1] = fmaf(gt, v4.y, vin[4 * i + 1]);
            vin[4 * i + 2] = fmaf(gt, v4.z, vin[4 * i + 2]);
            vin[4 * i + 3] = fmaf(gt, v4.w, vin[4 * i + 3]);
          }
        }
        float a[kF3dXO];
#pragma unroll
        for (int jj = 0; jj < kF3dXO; ++jj) a[jj] = 0.f;
#pragma unroll
        for (int kk = 0; kk <= 2 * R; ++kk) {
          const float gk = P.gs[kk < R ? R - kk : kk - R];
#pragma unroll
          for (int jj = 0; jj < kF3dXO; ++jj) a[jj] = fmaf(gk, vin[jj + kk + D], a[jj]);
        }
#pragma unroll
        for (int qq = 0; qq < kF3dXO / 4; ++qq)
          *reinterpret_cast<float4*>(q + lane * kF3dQS + 4 * qq) =
              make_float4(a[4 * qq], a[4 * qq + 1], a[4 * qq + 2], a[4 * qq + 3]);
        __syncwarp();
        // ---------------------------------------------------------- y-pass + epilogue
        float4 acc[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        // row quads past the tile (4rq >= TH) recompute the last valid quad (discarded)
        const float* wb = q + (4 * min(rq, TH / 4 - 1)) * kF3dQS + 4 * cq;
#pragma unroll
        for (int jj = 0; jj < 4 + 2 * R; ++jj) {
          const float4 qv = *reinterpret_cast<const float4*>(wb + jj * kF3dQS);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int kk = jj - i;
            if (kk >= 0 && kk <= 2 * R) {
              const float gk = P.gs[kk < R ? R - kk : kk - R];
              acc[i].x = fmaf(gk, qv.x, acc[i].x);
              acc[i].y = fmaf(gk, qv.y, acc[i].y);
              acc[i].z = fmaf(gk, qv.z, acc[i].z);
              acc[i].w = fmaf(gk, qv.w, acc[i].w);
            }
          }
        }
        if (xok) {
          const int jc = t - jlo;  // centre frame stage (Rayleigh operand p_{k-1})
          const float* cst = stage + ((base + (unsigned)jc) % NS) * STAGE_FLOATS;
          const float* fst = cst + kM * BOXW;  // F tile [TH][64] of frame t
          float s0 = 0.f, s1 = 0.f;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int y = y0 + i;
            if (y >= H || 4 * rq + i >= TH) break;
            const long off = (((long)sg.b * T + t) * H + y) * Wp + x;
            float4 f = *reinterpret_cast<const float4*>(fst + (4 * rq + i) * kF3dTW + kF3dXO * warp + 4 * cq);
            float4 uu = f4_scale(acc[i], s);
            if (OPT && !xfull) {  // forward: F is zero past W (TMA zero fill), no mask needed
              f = f4_mul(f, msk);
              uu = f4_mul(uu, msk);
            }
            const float4 yv = f4_mul(f, uu);
            s0 += f4_dot(yv, yv);
            if (OPT && P.rayleigh) {
              const float4 pp = *reinterpret_cast<const float4*>(cst + (4 * rq + i + R) * BOXW + RA + kF3dXO * warp + 4 * cq);
              s1 += f4_dot(pp, uu);
            }
            if (OPT && P.tape_u) *reinterpret_cast<float4*>(P.tape_u + off) = uu;
            *reinterpret_cast<float4*>(P.out + off) = P.last ? yv : f4_mul(f, yv);
          }
          acc0 += (double)s0;
          acc1 += (double)s1;
        }
      }
      __syncwarp();
      // frame t-RT is no longer needed by this run (the next output needs >= t+1-RT)
      const int jdone = (t + 1 == sg.t1) ? jhi - 1 : t - RT;
      while ((int)(released - base) + jlo <= jdone) {
        if (lane == 0) f3d_mbar_arrive(&empty[released % NS]);
        ++released;
      }
    }
    u += sg.t1 - sg.t0;
  }
  if (cur_vol >= 0) flush(cur_vol);

  // ---------------------------------------------------------------- last CTA: fixed-order fp64 finalize
  f3d_compute_bar();
  if (P.trace && tid == 0) {  // debug: {smid, entry, all compute warps done, exit}
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    P.trace[blockIdx.x * 4 + 0] = sm;
    P.trace[blockIdx.x * 4 + 1] = tr_start;
    P.trace[blockIdx.x * 4 + 2] = t1;
  }
  if (tid == 0) {
    const unsigned prev = atomic_add_acq_rel(P.counter, 1u);  // the warps' partials: ordered by the barrier
    *flag = (prev == (unsigned)P.G - 1) ? 1 : 0;
  }
  f3d_compute_bar();
  if (*flag == 0) {
    if (P.trace && tid == 0) {
      unsigned long long t2;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
      P.trace[blockIdx.x * 4 + 3] = t2;
    }
    return;
  }
  const long per_vol = P.U / P.B;
  const bool wide = P.B < kF3dCW;  // few volumes: whole compute group per volume; many: a warp each
  for (int b = wide ? 0 : warp; b < P.B; b += wide ? 1 : kF3dCW) {
    long lo, hi;
    vol_cta_range(b, per_vol, P.U, P.G, lo, hi);
    double s0, s1;
    if (wide) {
      s0 = block_sum_range<kF3dCW * 32, 1>(P.partials + (long)b * nslots, lo, hi, 1, red);
      s1 = block_sum_range<kF3dCW * 32, 1>(P.partials + (long)(P.B + b) * nslots, lo, hi, 1, red);
    } else {
      s0 = warp_sum_range(P.partials + (long)b * nslots, lo, hi);
      s1 = warp_sum_range(P.partials + (long)(P.B + b) * nslots, lo, hi);
    }
    if ((wide && tid == 0) || (!wide && lane == 0))
      fwd_finalize(P.sc + b * kScal, P.stats, P.tape_nu, P.err, P.K, P.k, P.rayleigh != 0, b, s0, s1);
  }
  if (tid == 0) *P.counter = 0u;
  if (P.trace && tid == 0) {
    unsigned long long t2;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
    P.trace[blockIdx.x * 4 + 3] = t2;
  }
}

}  // namespace sfseg
