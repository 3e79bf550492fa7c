// Persistent "wavefront" megakernel: all K forward iterations of the large-radius
// path in ONE launch (single GPU, no tape).
//
// Why: the two-pass iteration is a memory-bound temporal pass (a3, ~8 B/voxel)
// followed by an FP32-FMA-bound fused spatial pass (a4-a7).  Launched as separate
// kernels they serialise, and each spatial launch ends in a load-imbalance tail.
// Here both become work items of one persistent grid (G = resident CTAs) fed by a
// global ticket counter in a fixed, dependency-respecting order:
//   iteration k, volume b: T(fc=0), then for each frame chunk fc (NF frames):
//   T(fc+1), S(fc) -- temporal items run one chunk ahead of the spatial items
//   that consume them:
//     T(k,b,fc,cc)  temporal pass of p~_{k-1} -> v for the chunk's frames, column
//                   chunk cc (each thread walks NCOLS float4 columns through the
//                   NF + 2RT input frames with a register ring, cp.async queue)
//     S(k,b,t,s)    fused spatial pass (spass_run, the standalone kernel's body) of
//                   one full 64-column strip s of frame t: y~_k = F u~, p~_k = F y~_k
// Dependencies (spin-waits on acquire loads; an item only waits for items with
// smaller tickets, and every CTA is resident, so the schedule cannot deadlock):
//   T(k,b,fc) needs S(k-1,b,t) for every frame t in [t0 - RT, t1 + RT)
//   S(k,b,t)  needs all T(k,b,fc(t),*) (the whole frame of v, for the x/y halos)
// Buffers: p~_k lives in pbuf[k & 1] (T(k+1) of a neighbouring chunk may still read
// p~_{k-1}(t) when S(k+1,t) runs), v is single-buffered (its readers S(k,t) are
// exactly the items T(k+1, fc(t)) waits for).
// Normalisation (Eq.8) is LAGGED so no iteration waits for a global norm: T(k)
// scales by sigma_1 = 1/||x_0||, sigma_2 = 1, sigma_k = 1/nu~_{k-2} (k >= 3), where
// nu~_k = ||y~_k|| is finalised by the last S item of (k, b) as a fixed-order fp64
// sum of per-item partials (deterministic).  The map is linear, so
// y~_k = (prod sigma) M^k x_0 and the true per-iteration quantities follow exactly
// (mk_finalize_kernel): nu_1 = nu~_1/sigma_1, nu_k = nu~_k/(sigma_k nu~_{k-1}),
// x_K = y~_K / nu~_K; magnitudes stay within lambda^{+-2} of one (no overflow).
// Data written by other CTAs is read through L2 only: TMA (after a proxy fence),
// cp.async.cg, ld.global.cg.
#pragma once
#include "common.cuh"
#include "spass.cuh"
#include "tpass.cuh"

namespace sfseg {

constexpr int kMkThreads = kSpassThreads;  // 128

struct MkParams {
  SpassParams sp;         // S-item template: tmap of v, F, dims, spatial taps, U/NB/S; out/pprev set per item
  float* pbuf0;           // p~_{k} for even k (p~_0 from the combine)
  float* pbuf1;           // p~_{k} for odd k
  float* v;               // temporal-pass output, pitched [B*T][H][Wp]
  const double* sc;       // per-volume scalars from the combine (SC_XNORM = ||x_0||)
  double* part;           // [K+1][B][T*S][2] S-item partials (||y~||^2, <p~_{k-1}, u~>)
  double* nu;             // [K+1][B][2]: nu~_k, s1~_k (finalised sums)
  unsigned* ticket;       // [1]
  unsigned* tdone;        // [K+1][B][NFC]   T items done
  unsigned* sdone;        // [K+1][B][T]     S items done per frame
  unsigned* sall;         // [K+1][B]        S items done per (k, b)
  unsigned* nready;       // [K+1][B]        nu~ of (k, b) published
  long frame4;            // float4 per pitched frame (H*Wp/4)
  int B, T, S, K, NF, NFC, NCC, NCOLS, rayleigh;
  unsigned long long* trace;  // debug (SFSEG_MK_TRACE): per ticket {smid|kind, t_grab, t_ready, t_done} or null
  float gt[2 * kMaxRT + 1];
};

__device__ __forceinline__ unsigned long long mk_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned mk_smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// thread 0 spins until *c >= target (the caller broadcasts with __syncthreads)
__device__ __forceinline__ void spin_geq(const unsigned* c, unsigned target) {
  if (ld_acquire_u32(c) >= target) return;
  unsigned ns = 32;
  while (ld_acquire_u32(c) < target) {
    __nanosleep(ns);
    ns = ns < 256 ? ns * 2 : 256;
  }
}

// Frames per T item (compile-time: the output-stationary accumulators are registers).
__host__ __device__ constexpr int mk_nf(int RT) { return 2 * RT + 2; }

// One T item: v(t) = sigma * sum_o g_t[o] p~_{k-1}(t + o) for frames t in [t0, t1) of
// volume b, columns e = cbase + c*128 + tid (c < NCOLS).  Zero padding outside [0, T).
// Output-stationary: NF float4 accumulators per thread, the NF + 2RT input frames
// streamed once through a per-thread cp.async queue; the fully unrolled input loop
// issues exactly the (2RT+1) FMAs per output the convolution needs (no warm-up
// waste at the chunk edges).
template <int RT>
__device__ __forceinline__ void mk_titem(const MkParams& P, const float4* src, float4* dst, int t0, int t1,
                                         long cbase, float sigma, float4* sq /* smem [NF+2RT][128] */) {
  constexpr int NF = mk_nf(RT);
  constexpr int NIN = NF + 2 * RT;
  const int tid = threadIdx.x;
  const int T = P.T;
  const long f4 = P.frame4;
  const int jlo = t0 - RT;  // first input frame
  for (int c = 0; c < P.NCOLS; ++c) {
    const long e = cbase + (long)c * kMkThreads + tid;
    if (e >= f4) break;
    const float4* s = src + e;
    float4* d = dst + e;
    // all NIN input frames of this column in flight at once (one memory latency per column)
#pragma unroll
    for (int jp = 0; jp < NIN; ++jp) {
      const int j = jlo + jp;
      if (j >= 0 && j < T) cp_async16(&sq[jp * kMkThreads + tid], s + (long)j * f4);
    }
    cp_async_commit();
    cp_async_wait<0>();
    float4 acc[NF];
#pragma unroll
    for (int o = 0; o < NF; ++o) acc[o] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int jp = 0; jp < NIN; ++jp) {
      const int j = jlo + jp;
      float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
      if (j >= 0 && j < T) val = sq[jp * kMkThreads + tid];
#pragma unroll
      for (int o = 0; o < NF; ++o) {
        const int tap = jp - o;  // input t0 + o + (tap - RT)
        if (tap >= 0 && tap <= 2 * RT) {
          const float w = P.gt[tap];
          acc[o].x = fmaf(w, val.x, acc[o].x);
          acc[o].y = fmaf(w, val.y, acc[o].y);
          acc[o].z = fmaf(w, val.z, acc[o].z);
          acc[o].w = fmaf(w, val.w, acc[o].w);
        }
      }
    }
#pragma unroll
    for (int o = 0; o < NF; ++o)
      if (t0 + o < t1) __stcg(d + (long)(t0 + o) * f4, f4_scale(acc[o], sigma));
  }
}

// dynamic smem: max(S-item stage + ring, T-item input frames) + 256 bytes of scratch at the end
__host__ __device__ constexpr size_t mk_smem_bytes(int R, int RT) {
  return (sizeof(float) * ((size_t)spass_stages(R) * kM * spass_boxw(R) + (size_t)spass_ring_alloc(R) * kRingStride) >
                  (size_t)(mk_nf(RT) + 2 * RT) * kMkThreads * 16
              ? sizeof(float) * ((size_t)spass_stages(R) * kM * spass_boxw(R) + (size_t)spass_ring_alloc(R) * kRingStride)
              : (size_t)(mk_nf(RT) + 2 * RT) * kMkThreads * 16) +
         256;
}

template <int R, int RT>
__global__ void __launch_bounds__(kMkThreads, 3) mk_kernel(const __grid_constant__ MkParams P) {
  using Geo = SpassGeom<R>;
  constexpr int BOXW = Geo::BOXW;
  constexpr int RING_ROWS = spass_nslot(R) * kM;
  constexpr int NST = spass_stages(R);

  extern __shared__ __align__(128) unsigned char smem[];
  float* stage = reinterpret_cast<float*>(smem);
  float* ring = stage + NST * kM * BOXW;
  // barriers / reduction scratch / ticket words live in the last 256 bytes, past both the
  // S-item layout and the T-item input frames (which alias the stage + ring)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + mk_smem_bytes(R, RT) - 256);
  double* red = reinterpret_cast<double*>(bars + 2);
  unsigned* sh = reinterpret_cast<unsigned*>(red + 8);  // [0] ticket, [1] next ticket, [2] last flag
  float4* sq = reinterpret_cast<float4*>(smem);         // T-item input frames alias the (idle) S stage + ring


  const int tid = threadIdx.x;
  const int B = P.B, T = P.T, S = P.S, K = P.K, NF = P.NF, NFC = P.NFC, NCC = P.NCC;
  const long per_chunk = (long)NCC + (long)NF * S;        // T(fc+1) + S(fc) block of a full frame chunk
  const long per_vol = (long)NFC * NCC + (long)T * S;     // items of one volume in one iteration
  const long per_iter = (long)B * per_vol;
  const long total = (long)K * per_iter;
  const long f4 = P.frame4;
  const long vol4 = (long)T * f4;
  const long NB = P.sp.NB;

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_barrier_init();
    prefetch_tmap(&P.sp.tmap);
    sh[0] = atomicAdd(P.ticket, 1u);
  }
  __syncthreads();
  unsigned pseq = 0, cseq = 0;
  long tk = sh[0];
  // NOTE: the next ticket is taken only when this item is done.  Taking it early
  // (to hide the atomic) lets a CTA stuck waiting in one item hold a T item that
  // other CTAs' S items wait for: a convoy (measured: 70 % of CTA time waiting).
  while (tk < total) {
    unsigned long long tr0 = 0, tr1 = 0;
    if (P.trace && tid == 0) tr0 = mk_now();
    const int k = (int)(tk / per_iter) + 1;
    long r = tk % per_iter;
    const int b = (int)(r / per_vol);
    r -= (long)b * per_vol;
    // decode: [T(0)] then blocks fc = 0..NFC-1 of [T(fc+1) (if fc+1 < NFC)] [S(fc)]
    bool is_t;
    int fc, cc = 0;
    long si = 0;
    if (r < NCC) {
      is_t = true;
      fc = 0;
      cc = (int)r;
    } else {
      const long r2 = r - NCC;
      fc = (int)min(r2 / per_chunk, (long)NFC - 1);
      const long rr = r2 - (long)fc * per_chunk;
      if (fc + 1 < NFC && rr < NCC) {
        is_t = true;
        cc = (int)rr;
        fc += 1;
      } else {
        is_t = false;
        si = (fc + 1 < NFC) ? rr - NCC : rr;
      }
    }
    r = is_t ? 0 : NCC;  // trace kind
    const int t0 = fc * NF, t1 = min(T, t0 + NF);
    float* pout = (k & 1) ? P.pbuf1 : P.pbuf0;
    float* pin = (k & 1) ? P.pbuf0 : P.pbuf1;
    if (is_t) {
      // ------------------------------------------------------------ T item
      double sig = 1.0;
      if (tid == 0) {
        if (k >= 2) {
          const unsigned* sd = P.sdone + ((long)(k - 1) * B + b) * T;
          for (int t = max(0, t0 - RT); t < min(T, t1 + RT); ++t) spin_geq(sd + t, (unsigned)S);
        }
        if (k >= 3) spin_geq(P.nready + (long)(k - 2) * B + b, 1u);
      }
      __syncthreads();
      if (P.trace && tid == 0) tr1 = mk_now();
      if (k == 1) sig = 1.0 / P.sc[b * kScal + SC_XNORM];
      else if (k >= 3) sig = 1.0 / __ldcg(P.nu + ((long)(k - 2) * B + b) * 2);
      mk_titem<RT>(P, reinterpret_cast<const float4*>(pin) + (long)b * vol4,
                   reinterpret_cast<float4*>(P.v) + (long)b * vol4, t0, t1, (long)cc * P.NCOLS * kMkThreads,
                   (float)sig, sq);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(P.tdone + ((long)k * B + b) * NFC + fc, 1u);
      }
    } else {
      // ------------------------------------------------------------ S item
      const int t = t0 + (int)(si / S), s = (int)(si % S);
      if (tid == 0) {
        spin_geq(P.tdone + ((long)k * B + b) * NFC + fc, (unsigned)NCC);
        fence_proxy_async_global();  // TMA (async proxy) reads what other CTAs stored (generic proxy)
      }
      __syncthreads();
      if (P.trace && tid == 0) tr1 = mk_now();
      const long col = ((long)b * T + t) * S + s;
      double* pp = P.part + (((long)k * B + b) * ((long)T * S) + (long)t * S + s) * 2;
      spass_run<R, SP_FWD>(P.sp, col * NB, col * NB + NB, stage, ring, bars, pseq, cseq,
                           [&](int, double a0, double a1) {
                             const double s0 = block_sum<kMkThreads>(a0, red);
                             const double s1 = block_sum<kMkThreads>(a1, red);
                             if (tid == 0) {
                               pp[0] = s0;
                               pp[1] = s1;
                             }
                           },
                           pout, P.rayleigh ? pin : nullptr, nullptr, k == K ? 1 : 0);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(P.sdone + ((long)k * B + b) * T + t, 1u);
        const unsigned prev = atomicAdd(P.sall + (long)k * B + b, 1u);
        sh[2] = (prev == (unsigned)(T * S) - 1u) ? 1u : 0u;
      }
      __syncthreads();
      if (sh[2]) {
        // last S item of (k, b): fixed-order fp64 sum of the per-item partials -> nu~_k
        __threadfence();
        const double* pb = P.part + ((long)k * B + b) * ((long)T * S) * 2;
        const double a = block_sum_array<kMkThreads>(pb, (long)T * S, 2, red);
        const double c = block_sum_array<kMkThreads>(pb + 1, (long)T * S, 2, red);
        if (tid == 0) {
          P.nu[((long)k * B + b) * 2] = sqrt(a);
          P.nu[((long)k * B + b) * 2 + 1] = c;
          __threadfence();
          st_release_u32(P.nready + (long)k * B + b, 1u);
        }
      }
    }
    if (P.trace && tid == 0) {
      unsigned long long* tr = P.trace + tk * 4;
      tr[0] = ((unsigned long long)mk_smid() << 8) | (r < NCC ? 0ull : 1ull);
      tr[1] = tr0;
      tr[2] = tr1;
      tr[3] = mk_now();
    }
    __syncthreads();
    if (tid == 0) sh[1] = atomicAdd(P.ticket, 1u);
    __syncthreads();
    tk = sh[1];
  }
}

// Per-volume statistics and final scale from the lagged sums (one thread per volume).
struct MkFinParams {
  const double* nu;      // [K+1][B][2]
  double* sc;            // SC_S <- 1/nu~_K (final_scale), SC_NU <- nu_K
  double* stats;         // [B][K][3] or null
  unsigned* err;
  int B, K, rayleigh;
};
static __global__ void mk_finalize_kernel(const __grid_constant__ MkFinParams P) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= P.B) return;
  double* sc = P.sc + b * kScal;
  const double x0n = sc[SC_XNORM];
  double prev = 0.0;  // nu~_{k-1}
  double last_nu = 0.0;
  for (int k = 1; k <= P.K; ++k) {
    const double nut = P.nu[((long)k * P.B + b) * 2];
    const double s1t = P.nu[((long)k * P.B + b) * 2 + 1];
    const double sig = (k == 1) ? 1.0 / x0n : (k == 2 ? 1.0 : 1.0 / P.nu[((long)(k - 2) * P.B + b) * 2]);
    const double nu = (k == 1) ? nut / sig : nut / (sig * prev);   // ||M x_{k-1}|| (x_0 unnormalised)
    const double xn = (k == 1) ? x0n : 1.0;
    if (P.stats) {
      double* st = P.stats + ((long)b * P.K + (k - 1)) * 3;
      st[0] = nu;
      st[1] = nu / xn;
      st[2] = P.rayleigh ? ((k == 1) ? s1t / (sig * x0n * x0n) : s1t / (sig * prev * prev)) : 0.0;
    }
    flag_norm(P.err, nu);
    last_nu = nu;
    prev = nut;
  }
  sc[SC_S] = 1.0 / prev;  // x_K = y~_K / nu~_K
  sc[SC_NU] = last_nu;
  sc[SC_XNORM] = 1.0;
}

}  // namespace sfseg
