// Spatial pass of G_3D (y then x Gaussian) on the 5th-generation tensor
// cores: tcgen05.mma (UTCHMMA) with the operands' fp32 values split into three bf16 planes
// and six products per tap (fp32-class arithmetic, reading A23), accumulators
// and the streaming data operand in tensor memory (TMEM), fused with the F multiplies and
// the norm partials (Eq.8) exactly like spass_tc_kernel (the mma.sync version).
//
// Both 1D passes are contractions with a banded Toeplitz matrix; each is laid out so the
// filtered axis is the MMA's N (y-pass) or K (x-pass) and the data never needs a transpose:
//
//   strip: 128 input columns x_in (TMEM lanes) = 80 output columns + a 24-column halo on
//   each side (radii <= 24); rows stream down the frame: 32-row TMA input blocks, 64-row
//   output blocks (the MMAs' N = 64: below N = 128 a tcgen05.mma costs ~51 cycles whatever
//   its N -- tools/tc05_rate.cu -- so N = 64 halves the cost per row of N = 32).
//   y-pass  D1[x_in][y_out] += A[x_in][y_in] * B[y_in][y_out]
//     A = the temporal-pass output v of the strip's 128 columns, written into TMEM by the
//         worker warps (thread = column = lane) as three bf16 planes, a ring of six 32-row
//         input blocks (the window of output block m is input blocks 2m-1 .. 2m+2);
//     B = Ty^T, shift invariant: one tall banded matrix in shared memory, the k-step's
//         operand is a descriptor offset into it (K-major, no swizzle).
//     M = 128 (x_in), N = 64 (y_out), K = 16 per step over the window's rows (8 at R = 24).
//   D1 is drained by the workers (thread = x_in), summed over the leading / correction
//   accumulators, split into three bf16 planes and stored as the x-pass B operand Q^T
//   (MN-major, no swizzle: each thread writes its column's 32 y values as 16-byte rows).
//   x-pass  D2[x_out][y_out] += A[x_out][x_in] * B[x_in][y_out]
//     A = Tx^T (constant, shift invariant: one tall band in shared memory, three planes);
//     B = Q^T.  M = 128 (x_out, 80 valid), N = 64, K = 128 (8 steps), both from smem.
//   Product order: the five correction products first, the leading one last, into ONE
//   accumulator: the tensor core truncates each accumulation at the accumulator's
//   magnitude, so only the last 8 accumulations per pass happen at full magnitude (the
//   same count as a separate leading-product accumulator would see).
//   Epilogue: workers drain D2 (thread = x_out = lane, 32 rows), y = F u, p = F y (or y on
//   the last iteration), tape / Rayleigh options, fp64 norm partials.
//
// Warp roles (one CTA per SM: the CTA owns all 512 TMEM columns):
//   warps 0-3  workers (TMEM lane quarter = warp): planes, D1 drain + Q^T, epilogue;
//   warp 4     TMA producer (one thread): 128 x 32 fp32 boxes of v, 3 stages;
//   warp 5     MMA issuer (one thread): y-pass of block i, then x-pass of block i-1.
// mbarriers carry every hand-off (TMA -> workers -> issuer -> workers); the TMEM / smem
// reuse is ordered by tcgen05.commit completions.  Tensor work per 80 x 32 outputs:
// 6 x (NKY + 8) MMAs of M = 128, N = 64 per 80 x 64 outputs (~51 cycles each).
#pragma once
#include <cstdio>

#include "spass_tc.cuh"

namespace sfseg {

constexpr int k5Lanes = 128;        // input columns per strip (TMEM lanes of the y-pass)
constexpr int k5Halo = 24;          // left halo of the window: radii <= 24
constexpr int k5OW = k5Lanes - 2 * k5Halo;  // 80 output columns per strip
constexpr int k5NR = 64;            // output rows per y-block (the MMAs' N)
constexpr int k5IR = 32;            // rows per TMA input block
constexpr int k5Workers = 128;      // one worker group: 4 warps (one TMEM lane quarter each)
constexpr int k5Threads = 320;      // planes group (warps 0-3), producer (4), MMA issuer (5), epilogue group (6-9)
constexpr int k5NST = 4;            // TMA stages
constexpr int k5Slots = 6;          // TMEM ring of input blocks: a window of 4 + the next 2
constexpr uint32_t k5ColA = 0;      // 3 planes x 6 slots x 16 columns
constexpr uint32_t k5PlaneCols = 16 * k5Slots;
constexpr uint32_t k5ColD1 = 3 * k5PlaneCols, k5ColD2 = k5ColD1 + k5NR;   // 288, 352
constexpr uint32_t k5TmemCols = 512;

__host__ __device__ constexpr int t5_jlo(int R) { return -((R + 15) / 16); }   // first 16-row k-step of a y window
__host__ __device__ constexpr int t5_jhi(int R) { return (k5NR + R + 15) / 16; }
__host__ __device__ constexpr int t5_nky(int R) { return t5_jhi(R) - t5_jlo(R); }
__host__ __device__ constexpr int t5_imin(int R) { return -16 * (t5_jhi(R) - 1); }
__host__ __device__ constexpr int t5_trows(int R) { return k5NR - 16 * t5_jlo(R) - t5_imin(R); }  // Ty^T rows
constexpr int k5TxRows = k5Lanes + 16 * 7;                       // Tx^T band rows: i = x_out - 16 s
// shared memory: TMA stages, Q^T (2 buffers x 3 planes), Ty^T and Tx^T bands (3 planes each), barriers
constexpr uint32_t k5StageBytes = k5IR * k5Lanes * 4;          // 16 KB
constexpr uint32_t k5QPlane = k5Lanes * k5NR * 2;              // 16 KB
constexpr uint32_t k5TxPlane = k5TxRows / 8 * 256;             // 7.5 KB
__host__ __device__ constexpr uint32_t t5_typlane(int R) { return (uint32_t)t5_trows(R) / 8 * 256; }
__host__ __device__ constexpr size_t t5_smem_bytes(int R) {
  return 1024 + (size_t)k5NST * k5StageBytes + 2 * 3 * k5QPlane + 3 * t5_typlane(R) + 3 * k5TxPlane + 256 + 256;
}

__device__ __forceinline__ uint64_t t5_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // sm_100 shared-memory matrix descriptor, SWIZZLE_NONE: start >> 4, LBO >> 4, SBO >> 4,
  // version 1 at bit 46 (validated by tools/tc05_probe.cu)
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// kind::f16 instruction descriptor: fp32 accumulate, bf16 A and B, M = 128, N = k5NR
__host__ __device__ constexpr uint32_t t5_idesc(int b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(k5NR >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void t5_mma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d),
               "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void t5_mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(d),
               "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void t5_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void t5_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void t5_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void t5_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 16 consecutive 32-bit TMEM columns of this warp's lane quarter <-> registers
// (.sync.aligned: the warp must be converged -- the mbarrier polls before these can leave its
// lanes at different points, hence the __syncwarp)
__device__ __forceinline__ void t5_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  __syncwarp();
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void t5_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  __syncwarp();
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// wait for the phase of parity `par` to complete (parity ^ 1 on a fresh barrier returns at once).
// Bounded: a pipeline that stops making progress (a protocol bug) traps after ~2^16 suspended
// polls instead of hanging the GPU.
__device__ __forceinline__ void t5_wait(uint64_t* bar, unsigned par) {
  for (unsigned i = 0;; ++i) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(par), "r"(20000u)
        : "memory");
    if (ok) return;
    if (i > (1u << 20)) __trap();
  }
}

// weight of a spatial offset (0 outside the support), from the shared-memory tap copy
__device__ __forceinline__ float t5_w(const float* gsm, int d, int R) {
  const int a = d < 0 ? -d : d;
  return a <= R ? gsm[a] : 0.f;
}

// -DT5_PROFILE: CTA 0 prints, per role, its cycles and the cycles spent in each barrier wait
// (how the pipeline balance below was measured; not part of the product build)
#ifdef T5_PROFILE
#define T5W(site, bar, par)                 \
  do {                                      \
    const long long _t0 = clock64();        \
    t5_wait(bar, par);                      \
    prof[site] += clock64() - _t0;          \
  } while (0)
#else
#define T5W(site, bar, par) t5_wait(bar, par)
#endif

template <int R, int EPI>
__global__ void __launch_bounds__(k5Threads, 1) spass_tc5_kernel(const __grid_constant__ SpassParams P) {
  static_assert(R <= k5Halo, "tcgen05 spatial pass: radii <= 24");
  constexpr int JLO = t5_jlo(R), NKY = t5_nky(R), IMIN = t5_imin(R), TROWS = t5_trows(R);
  constexpr uint32_t TYPL = t5_typlane(R);
  constexpr int PL = 3, NPR = 6;
  constexpr int TXMIN = -16 * 7;   // first row of the Tx^T band
  constexpr bool plain = EPI == EPI_PLAIN;
  static_assert(JLO >= -2 && JLO + NKY <= 6, "a y window spans input blocks 2m-1 .. 2m+2");

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* stage = reinterpret_cast<float*>(smem);                                   // [NST][32][128] fp32
  unsigned char* qbuf = smem + k5NST * k5StageBytes;                               // [2][3 planes][16 KB]
  unsigned char* tyb = qbuf + 2 * 3 * k5QPlane;                                    // [3 planes][TYPL]
  unsigned char* txb = tyb + 3 * TYPL;                                             // [3 planes][TxPlane]
  uint64_t* bars = reinterpret_cast<uint64_t*>(txb + 3 * k5TxPlane);
  uint64_t* b_tfull = bars;              // [4] TMA -> planes group
  uint64_t* b_tempty = bars + 4;         // [4] planes group -> producer (count 4)
  uint64_t* b_pfull = bars + 8;          // [6] planes written (count 4)
  uint64_t* b_sfree = bars + 14;         // [6] slot's last y-pass done (commit)
  uint64_t* b_d1full = bars + 20;        // y-pass done (commit)
  uint64_t* b_d1empty = bars + 21;       // D1 drained (count 4)
  uint64_t* b_qfull = bars + 22;         // [2] Q^T written (count 4)
  uint64_t* b_qempty = bars + 24;        // [2] x-pass done reading Q^T (commit)
  uint64_t* b_d2full = bars + 26;        // x-pass done (commit)
  uint64_t* b_d2empty = bars + 27;       // D2 drained (count 4)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 28);
  double* red = reinterpret_cast<double*>(bars + 30);   // 16 doubles
  int* flag = reinterpret_cast<int*>(red + 16);
  __shared__ float gsm[kMaxRS + 1];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int H = P.H, W = P.W, Wp = P.Wp, S = P.S, T = P.T, NB = P.NB;
#ifdef T5_PROFILE
  long long prof[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const long long prof_t0 = clock64();
#endif
  const long u_begin = (long)blockIdx.x * P.U / P.G;
  const long u_end = (long)(blockIdx.x + 1) * P.U / P.G;

  if (tid <= R) gsm[tid] = P.g[tid];
  if (tid == 0) {
    for (int i = 0; i < k5NST; ++i) {
      mbar_init(&b_tfull[i], 1);
      mbar_init(&b_tempty[i], 4);
    }
    for (int i = 0; i < k5Slots; ++i) {
      mbar_init(&b_pfull[i], 4);
      mbar_init(&b_sfree[i], 1);
    }
    mbar_init(b_d1full, 1);
    mbar_init(b_d1empty, 4);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&b_qfull[i], 4);
      mbar_init(&b_qempty[i], 1);
    }
    mbar_init(b_d2full, 1);
    mbar_init(b_d2empty, 4);
    fence_barrier_init();
    prefetch_tmap(&P.tmap);
  }
  __syncwarp();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(k5TmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  // the two shift-invariant Toeplitz bands (K-major, no swizzle, three bf16 planes each):
  //   Ty^T row i = n - 16 j (output row n, k step j), column k: g(k - i)          (y-pass B)
  //   Tx^T row i = x_out - 16 s (k step s), column k:          g(k - i - 24)     (x-pass A)
  for (int e = tid; e < (TROWS + k5TxRows) * 16; e += k5Threads) {
    const bool isx = e >= TROWS * 16;
    const int ee = isx ? e - TROWS * 16 : e;
    const int ii = ee >> 4, k = ee & 15;
    float a = isx ? t5_w(gsm, k - (ii + TXMIN) - k5Halo, R) : t5_w(gsm, k - (ii + IMIN), R);
    const uint32_t off = (uint32_t)(ii / 8) * 256 + (uint32_t)(k / 8) * 128 + (uint32_t)(ii % 8) * 16 + (uint32_t)(k % 8) * 2;
    unsigned char* base = isx ? txb : tyb;
    const uint32_t pls = isx ? k5TxPlane : TYPL;
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      const __nv_bfloat16 h = __float2bfloat16_rn(a);
      *reinterpret_cast<__nv_bfloat16*>(base + q * pls + off) = h;
      a -= __bfloat162float(h);
    }
  }
  fence_proxy_async();  // bands (generic stores) -> tensor core reads (async proxy)
  t5_fence_before();
  __syncthreads();
  t5_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lanebase = tmem + ((uint32_t)(32 * (warp & 3)) << 16);   // this warp's TMEM lane quarter
  const int xl = 32 * (warp & 3) + lane;                                    // this thread's TMEM lane

  if (warp == 4) {
    // ================================================================== TMA producer
    if (lane == 0) {
      unsigned ib = 0;
      for (long u = u_begin; u < u_end;) {
        const Seg sg = seg_decode(u, u_end, NB, S);
        for (int n = 2 * sg.yb0 - 1; n <= 2 * sg.yb1; ++n, ++ib) {   // 32-row input blocks of the segment
          const unsigned st = ib % k5NST;
          T5W(0, &b_tempty[st], ((ib / k5NST) & 1) ^ 1);
          mbar_arrive_expect_tx(&b_tfull[st], k5StageBytes);
          tma_load_3d(stage + st * (k5IR * k5Lanes), &P.tmap, &b_tfull[st], sg.s * k5OW - k5Halo, n * k5IR, sg.bt);
        }
        u += sg.yb1 - sg.yb0;
      }
    }
  } else if (warp == 5) {
    // ================================================================== MMA issuer
    if (lane == 0) {
      const uint32_t idy = t5_idesc(0), idx = t5_idesc(1);
      const uint32_t ty0 = smem_u32(tyb), tx0 = smem_u32(txb), q0 = smem_u32(qbuf);
      unsigned ib = 0, ny = 0, pfull_ph = 0;   // pfull_ph: phase bit per ring slot
      auto xpass = [&](unsigned yb) {
        const unsigned qb = yb & 1;
        T5W(1, &b_qfull[qb], (yb >> 1) & 1);
        T5W(2, b_d2empty, (yb & 1) ^ 1);
        t5_fence_after();
        const uint32_t d = tmem + k5ColD2;
#pragma unroll
        for (int pp = 0; pp < NPR; ++pp) {
          const int p = pp + 1 < NPR ? pp + 1 : 0;   // corrections first, the leading product last
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            const uint64_t ad = t5_desc(tx0 + sptc_pb(p) * k5TxPlane + (uint32_t)(-16 * s - TXMIN) * 32, 128, 256);
            const uint64_t bd = t5_desc(q0 + (qb * 3 + sptc_pa(p)) * k5QPlane + s * 256, 128, 2048);
            t5_mma_ss(d, ad, bd, idx, (pp > 0 || s > 0) ? 1u : 0u);
          }
        }
        t5_commit(b_d2full);
        t5_commit(&b_qempty[qb]);
      };
      for (long u = u_begin; u < u_end;) {
        const Seg sg = seg_decode(u, u_end, NB, S);
        for (int m = sg.yb0; m < sg.yb1; ++m, ++ny) {
          const unsigned nnew = m == sg.yb0 ? 4u : 2u;
          for (unsigned i = 0; i < nnew; ++i, ++ib) {
            const unsigned sl = ib % k5Slots;
            T5W(3, &b_pfull[sl], (pfull_ph >> sl) & 1u);
            pfull_ph ^= 1u << sl;
          }
          const unsigned ib0 = ib - 4;   // the window's first input block (= 2m - 1)
          T5W(4, b_d1empty, (ny & 1) ^ 1);
          t5_fence_after();
          const uint32_t d = tmem + k5ColD1;
#pragma unroll
          for (int pp = 0; pp < NPR; ++pp) {
            const int p = pp + 1 < NPR ? pp + 1 : 0;
#pragma unroll
            for (int jj = 0; jj < NKY; ++jj) {
              const int j = JLO + jj;                       // rows 16 j .. 16 j + 15 relative to row 64 m
              const int blk = (j + 2) >> 1;                 // 0..3: input blocks 2m-1 .. 2m+2
              const int half = (j + 2) & 1;
              const uint32_t sl = (ib0 + (unsigned)blk) % k5Slots;
              const uint32_t a = tmem + k5ColA + k5PlaneCols * sptc_pa(p) + 16 * sl + 8 * half;
              const uint64_t bd = t5_desc(ty0 + sptc_pb(p) * TYPL + (uint32_t)(-16 * j - IMIN) * 32, 128, 256);
              t5_mma_ts(d, a, bd, idy, (pp > 0 || jj > 0) ? 1u : 0u);
            }
          }
          t5_commit(b_d1full);
          // the window's first two input blocks are dead now (all four at the end of a segment)
          t5_commit(&b_sfree[ib0 % k5Slots]);
          t5_commit(&b_sfree[(ib0 + 1) % k5Slots]);
          if (m + 1 == sg.yb1) {
            t5_commit(&b_sfree[(ib0 + 2) % k5Slots]);
            t5_commit(&b_sfree[(ib0 + 3) % k5Slots]);
          }
          if (ny >= 1) xpass(ny - 1);
        }
        u += sg.yb1 - sg.yb0;
      }
      if (ny >= 1) xpass(ny - 1);
    }
  } else if (warp < 4) {
    // ================================================================== planes group (warps 0-3)
    unsigned ib = 0, ny = 0, sfree_ph = 0;
    auto write_planes = [&]() {   // one input block: fp32 TMA box -> three bf16 planes, TMEM ring slot
      const unsigned st = ib % k5NST, sl = ib % k5Slots;
      T5W(5, &b_tfull[st], (ib / k5NST) & 1);
      const float* col = stage + st * (k5IR * k5Lanes) + xl;
      float v[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = col[r * k5Lanes];
      __syncwarp();
      if (lane == 0) t5_arrive(&b_tempty[st]);
      uint32_t pl[PL][16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        uint32_t pp[PL];
        split_planes<PL>(v[2 * c], v[2 * c + 1], pp);
#pragma unroll
        for (int q = 0; q < PL; ++q) pl[q][c] = pp[q];
      }
      T5W(6, &b_sfree[sl], ((sfree_ph >> sl) & 1u) ^ 1u);
      sfree_ph ^= 1u << sl;
      t5_fence_after();
#pragma unroll
      for (int q = 0; q < PL; ++q) t5_st16(lanebase + k5ColA + k5PlaneCols * q + 16 * sl, pl[q]);
      __syncwarp();
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      t5_fence_before();
      __syncwarp();
      if (lane == 0) t5_arrive(&b_pfull[sl]);
      ++ib;
    };
    auto drain_d1 = [&](unsigned yb) {   // D1 (64 rows) -> three planes of Q^T (MN-major) in smem
      T5W(7, b_d1full, yb & 1);
      t5_fence_after();
      float a[32], b[32];
      t5_ld32(lanebase + k5ColD1, a);
      t5_ld32(lanebase + k5ColD1 + 32, b);
      t5_fence_before();
      __syncwarp();
      if (lane == 0) t5_arrive(b_d1empty);
      const unsigned qb = yb & 1;
      T5W(8, &b_qempty[qb], ((yb >> 1) & 1) ^ 1);
      unsigned char* qp = qbuf + qb * 3 * k5QPlane + (uint32_t)xl * 16;   // k = xl: (k/8)*128 + (k%8)*16
#pragma unroll
      for (int g = 0; g < 8; ++g) {   // n group g: rows 8g .. 8g + 7
        const float* src = g < 4 ? a + 8 * g : b + 8 * (g - 4);
        uint32_t w[PL][4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t pp[PL];
          split_planes<PL>(src[2 * i], src[2 * i + 1], pp);
#pragma unroll
          for (int q = 0; q < PL; ++q) w[q][i] = pp[q];
        }
#pragma unroll
        for (int q = 0; q < PL; ++q)
          *reinterpret_cast<uint4*>(qp + q * k5QPlane + g * 2048) = make_uint4(w[q][0], w[q][1], w[q][2], w[q][3]);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) t5_arrive(&b_qfull[qb]);
    };
    for (long u = u_begin; u < u_end;) {
      const Seg sg = seg_decode(u, u_end, NB, S);
      for (int m = sg.yb0; m < sg.yb1; ++m, ++ny) {
        if (m == sg.yb0) {
          write_planes();
          write_planes();
        }
        write_planes();
        write_planes();
        if (ny >= 1) drain_d1(ny - 1);
      }
      u += sg.yb1 - sg.yb0;
    }
    if (ny >= 1) drain_d1(ny - 1);
  } else {
    // ================================================================== epilogue group (warps 6-9)
    const int wg = warp - 6;          // 0..3 within the group
    double acc0 = 0.0, acc1 = 0.0;
    int cur_vol = -1;
    auto flush = [&](int vol) {       // fixed-order sum over the group's 128 threads (named barrier 1)
      double s0 = acc0, s1 = acc1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (lane == 0) {
        red[wg] = s0;
        red[4 + wg] = s1;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (wg == 0 && lane == 0) {
        P.partials[(long)vol * P.G + blockIdx.x] = ((red[0] + red[1]) + red[2]) + red[3];
        P.partials[(long)(P.B + vol) * P.G + blockIdx.x] = ((red[4] + red[5]) + red[6]) + red[7];
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      acc0 = acc1 = 0.0;
    };
    // walk the CTA's y-blocks; per y-block 8 chunks of 8 rows (a compact loop: the four roles
    // run different code at once, and a fully unrolled 64-row body thrashed the instruction
    // cache -- ncu: stall_no_instruction was the epilogue's top reason).  F of the next chunk
    // is in registers before it is needed; F of the next y-block is prefetched into L2.
    long u = u_begin;
    Seg sg{};
    int m = 0;
    bool have = false;
    auto advance = [&]() -> bool {   // next y-block of the CTA's range into (sg, m)
      if (have) {
        if (++m < sg.yb1) return true;
        u += sg.yb1 - sg.yb0;
      }
      if (u >= u_end) return false;
      sg = seg_decode(u, u_end, NB, S);
      m = sg.yb0;
      have = true;
      return true;
    };
    auto prefetch_l2 = [&](int bt, int s, int mm) {   // the 64 rows of F this thread will read
      const int x = s * k5OW + xl;
      if (plain || !(xl < k5OW && x < Wp)) return;
      const int y0 = mm * k5NR;
      const long base = ((long)bt * H + y0) * Wp + x;
      const int nrow = min(k5NR, H - y0);
      for (int i = 0; i < nrow; i += 8)   // one 32-byte sector per 8 rows is enough per warp row
        asm volatile("prefetch.global.L2 [%0];" ::"l"(P.F + base + (long)i * Wp));
    };
    bool more = advance();
    unsigned yb = 0;
    while (more) {
      const int bt = sg.bt, s = sg.s, mm = m;
      more = advance();
      if (more) {
#pragma unroll 1
        for (int r = 0; r < 8; ++r) prefetch_l2(sg.bt, sg.s, m);   // (loop form keeps the code small)
      }
      const int vol = bt / T;
      if (vol != cur_vol) {
        if (cur_vol >= 0) flush(cur_vol);
        cur_vol = vol;
      }
      const int x = s * k5OW + xl;
      const bool xin = xl < k5OW && x < Wp;
      const int y0 = mm * k5NR;
      const long base = ((long)bt * H + y0) * Wp + x;
      const int nrow = H - y0;
      const float cmask = x < W ? 1.f : 0.f;
      float fc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) fc[i] = (!plain && xin && i < nrow) ? __ldg(P.F + base + (long)i * Wp) : 0.f;
      T5W(9, b_d2full, yb & 1);
      t5_fence_after();
      float s0 = 0.f, s1 = 0.f;
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        float fn[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = 8 * (c + 1) + i;
          fn[i] = (!plain && c < 7 && xin && r < nrow) ? __ldg(P.F + base + (long)r * Wp) : 0.f;
        }
        uint32_t q[8];
        __syncwarp();
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7])
                     : "r"(lanebase + k5ColD2 + 8 * c)
                     : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = 8 * c + i;
          if (!(xin && r < nrow)) continue;
          const long off = base + (long)r * Wp;
          const float uu = __uint_as_float(q[i]) * cmask;
          if (plain) {
            P.out[off] = uu;
            continue;
          }
          const float yv = fc[i] * uu;
          s0 = fmaf(yv, yv, s0);
          if (EPI == EPI_FWD_OPT) {
            if (P.pprev) s1 = fmaf(__ldcg(P.pprev + off), uu, s1);
            if (P.tape_u) P.tape_u[off] = uu;
          }
          P.out[off] = P.last ? yv : fc[i] * yv;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) fc[i] = fn[i];
      }
      t5_fence_before();
      __syncwarp();
      if (lane == 0) t5_arrive(b_d2empty);
      ++yb;
      acc0 += (double)s0;
      acc1 += (double)s1;
    }
    if (cur_vol >= 0) flush(cur_vol);
  }
#ifdef T5_PROFILE
  if (blockIdx.x == 0 && lane == 0 && (warp == 0 || warp == 4 || warp == 5 || warp == 6))
    printf("[t5prof] warp %d total %lld waits: tempty %lld qfull %lld d2empty %lld pfull %lld d1empty %lld tfull %lld "
           "sfree %lld d1full %lld qempty %lld d2full %lld\n",
           warp, clock64() - prof_t0, prof[0], prof[1], prof[2], prof[3], prof[4], prof[5], prof[6], prof[7], prof[8],
           prof[9]);
#endif
  t5_fence_before();
  __syncthreads();
  if (warp == 0) {
    t5_fence_after();
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(k5TmemCols));
  }
  if (plain) return;
  spass_finalize<SP_FWD, k5Threads>(P, red, flag);
}

}  // namespace sfseg
