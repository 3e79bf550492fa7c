// Forward spatial pass of G_3D (x then y Gaussian) on the 5th-generation
// tensor cores with dense-rate MMA shapes, fused with the F multiplies, the norm partials
// (Eq.8) and max |p_k| (the next temporal pass's fp16 range).
//
// Arithmetic (reading A25, the same as spass_tc's FMT = 1): every operand in two
// fp16 planes and three products per tap (a1g1 + a2g1 + a1g2, 22-bit operands), fp32
// accumulation in TMEM.  The input v arrives ALREADY SPLIT: the temporal pass (TP_FWD16)
// writes v * 2^e as two fp16 planes [bt][plane][H][Wp] (same 4 B/voxel as fp32), with e
// chosen from max |p_{k-1}| so that |v 2^e| < 2^14; the taps are scaled by 2^12.
//
// Both 1D passes are contractions with a banded Toeplitz matrix, laid out so that the TMEM
// lanes are the strip's 128 OUTPUT columns in both passes (no lane is spent on the x-halo):
//
//   x-pass  D1[x_out][row] += Tx^T[x_out][x_in] * V[row][x_in]^T              (SS)
//     A = Tx^T: one shift-invariant band in shared memory (K-major, no swizzle); the
//         k step's operand is a descriptor offset into it;
//     B = V: the TMA box of the two data planes, rows x (128 + 2 RA) columns, K-major,
//         SWIZZLE_128B (three 64-column boxes per plane; the k step advances the
//         descriptor's start address 32 B inside the swizzle atom);
//     M = 128 (x_out), N = 128 rows per x-block (dense rate), K = 16 per step (NKX steps).
//   D1 is drained by the splitter warps (thread = x_out = lane), scaled by 2^-12, split
//   into two fp16 planes and stored back into TMEM as the y-pass A operand Q (a ring of
//   eight 32-row chunks: column = row pair).
//   y-pass  D2[x_out][y_out] += Q[x_out][y_in] * Ty^T[y_in][y_out]^T          (TS)
//     A = Q from TMEM, B = Ty^T: shift-invariant band in shared memory;
//     M = 128, N = 64 output rows per y-block (two D2 buffers), K = 16 per step over the
//     y window (NKY = 4 + 2 ceil(R/16) steps, 16-row aligned).
//   Epilogue (thread = x_out): u = D2 2^-(e+12); y = F u; p = F y (y when last);
//   ||y||^2 partials in fp64; max |p|; optional tape u / Rayleigh <p_{k-1}, u>.
//
// Row geometry of a segment (frame bt, strip s, y-blocks [yb0, yb1)): origin R0 = 64 yb0;
// local chunk c = rows [R0 - 32 + 32 c, +32); x-block i = chunks 4i .. 4i+3; y-block j reads
// chunks 2j .. 2j + (JHI+1)/2 (rows R0 + 64 j + 16 kk, kk in [JLO, JHI)).
//
// Warp roles (one CTA per SM: all 512 TMEM columns, 224 KB of shared memory):
//   warp 0     TMA producer (one thread) + TMEM allocation;
//   warp 1     MMA issuer (one thread): x(n), then every y-block whose chunks were split
//              before x(n) was issued (the split of x(n-1) runs under x(n));
//   warps 2-5  splitters (TMEM lane quarter = warp & 3): D1 -> Q;
//   warps 6-9  epilogue (lane quarter = warp & 3).
// Every hand-off is an mbarrier (tcgen05.commit for MMA completion); waits are bounded
// (a protocol bug traps instead of hanging the GPU).
//
// TMEM columns: Q ring [0, 256) (slot q: 32 q + 16 plane), D1 [256, 384), D2 [384, 512).
#pragma once
#include <cstdio>

#include "spass_tc.cuh"
#include "tpass.cuh"

namespace sfseg {

#ifndef T6_LDALL
#define T6_LDALL 0  // A/B: splitters / epilogue read a whole D1 / D2 buffer in one TMEM round trip and release it
#endif              //      before their stores (0: 32- / 16-column loads, each waited, buffer released at the end)
#ifndef T6_XSTACK
#define T6_XSTACK 1 // x-pass: the data planes stacked along N (one M128 N128 MMA per k step gives a_hi g_hi and
#endif              //   a_lo g_hi side by side, one N64 MMA a_hi g_lo): 14 KB of operand reads per k step instead
                    //   of 18 KB; D1 single-buffered (128 columns)
#ifndef T6_L2PF
#define T6_L2PF 0   // A/B: x-blocks (v boxes + F tile) the producer prefetches into L2 ahead of its loads (0: none)
#endif

constexpr int k6M = 128;        // output columns per strip (TMEM lanes, MMA M)
constexpr int k6XN = 64;        // rows per x-block (x-pass MMA N): two ring chunks
constexpr int k6YN = 64;        // rows per y-block (y-pass MMA N)
constexpr int k6Threads = 320;
constexpr int k6Slots = 8;      // Q ring chunks (32 rows each)
constexpr uint32_t k6ColQ = 0, k6ColD1 = 256, k6ColD2 = 384;  // D1, D2: two 64-column buffers each
constexpr uint32_t k6TmemCols = 512;
constexpr int k6BoxW = 64;      // TMA box columns: 128 B, SWIZZLE_128B
constexpr uint32_t k6PlaneBox = k6XN * k6BoxW * 2;       // 8 KB: one plane of one box
constexpr uint32_t k6BoxBytes = 2 * k6PlaneBox;          // both planes (one TMA)
constexpr int k6Stages = 2;
constexpr uint32_t k6FBytes = k6YN * k6M * 4;            // 32 KB: the F tile of one y-block (fp32)

__host__ __device__ constexpr int t6_ra(int R) { return 8 * ((R + 7) / 8); }
__host__ __device__ constexpr int t6_nkx(int R) { return (k6M + 2 * t6_ra(R)) / 16; }
__host__ __device__ constexpr int t6_jlo(int R) { return -((R + 15) / 16); }
__host__ __device__ constexpr int t6_jhi(int R) { return 4 + (R + 15) / 16; }
__host__ __device__ constexpr int t6_txmin(int R) { return -16 * (t6_nkx(R) - 1); }
__host__ __device__ constexpr int t6_txrows(int R) { return k6M - t6_txmin(R); }
__host__ __device__ constexpr int t6_tymin(int R) { return -16 * (t6_jhi(R) - 1); }
__host__ __device__ constexpr int t6_tyrows(int R) { return k6YN - 16 * t6_jlo(R) - t6_tymin(R); }
// 64-column TMA boxes per stage (3 for r_s <= 32, 4 for r_s = 36) and the stage size
__host__ __device__ constexpr int t6_nbox(int R) { return (16 * t6_nkx(R) + k6BoxW - 1) / k6BoxW; }
__host__ __device__ constexpr uint32_t t6_stage_bytes(int R) { return (uint32_t)t6_nbox(R) * k6BoxBytes; }
// chunk origin: local chunk c covers rows R0 - 32 OFF + 32 c (OFF = 1 for r_s <= 32, 2 above), so
// the first y-block's window never starts before chunk 0; y-block j's k step kk reads chunk
// 2j + (kk + 2 OFF) / 2 (half (kk + 2 OFF) & 1)
__host__ __device__ constexpr int t6_off(int R) { return (R + 31) / 32; }
__host__ __device__ constexpr int t6_cfirst(int R) { return (t6_jlo(R) + 2 * t6_off(R)) / 2; }    // + 2j
__host__ __device__ constexpr int t6_clast(int R) { return (t6_jhi(R) - 1 + 2 * t6_off(R)) / 2; }  // + 2j
// the x-block (two chunks) holding y-block j's last chunk, and x-blocks per segment of ny y-blocks
__host__ __device__ constexpr int t6_xneed(int R, int j) { return (2 * j + t6_clast(R)) / 2; }
__host__ __device__ constexpr int t6_nx(int R, int ny) { return t6_xneed(R, ny - 1) + 1; }
__host__ __device__ constexpr size_t t6_smem_bytes(int R) {
  return 1024 + (size_t)k6Stages * t6_stage_bytes(R) + 2 * (size_t)k6FBytes + 2 * 32 * (size_t)t6_txrows(R) +
         2 * 32 * (size_t)t6_tyrows(R) + 512;   // 512: 30 mbarriers, the TMEM slot, 16 doubles, a flag
}

__device__ __forceinline__ uint64_t t6_desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // SWIZZLE_NONE K-major: start >> 4, LBO >> 4 (K-adjacent core matrices), SBO >> 4 (M/N-adjacent), version 1
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ uint64_t t6_desc_sw128(uint32_t saddr) {
  // SWIZZLE_128B K-major: LBO unused (1), SBO = 1024 B (8 rows x 128 B), layout type 2 (bits 61-63)
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16 instruction descriptor: fp32 accumulate, fp16 A and B, both K-major, M = 128
__host__ __device__ constexpr uint32_t t6_idesc(int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void t6_mma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d),
               "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void t6_mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(d),
               "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
// warp-converged forms: every lane executes them, one elected lane issues (the operands are
// warp-uniform, so they stay in uniform registers: no per-MMA R2UR broadcast loop)
__device__ __forceinline__ void t6_mma_ss_e(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{.reg .pred p, e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void t6_mma_ts_e(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{.reg .pred p, e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void t6_commit_e(uint64_t* bar) {
  asm volatile(
      "{.reg .pred e; elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void t6_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void t6_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void t6_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void t6_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 16 consecutive 32-bit TMEM columns of this warp's lane quarter <- registers
__device__ __forceinline__ void t6_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// 32 consecutive 32-bit TMEM columns -> registers (no wait: the caller issues tcgen05.wait::ld)
__device__ __forceinline__ void t6_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void t6_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// wait for the phase of parity `par` (parity ^ 1 on a fresh barrier returns at once); bounded:
// a protocol bug traps after ~2^20 suspended polls instead of hanging the GPU
__device__ __forceinline__ void t6_wait(uint64_t* bar, unsigned par) {
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
// -DT6_PROFILE: CTA 0 prints, per role, its cycles and the cycles spent in each barrier wait
// (pipeline balance measurement; not part of the product build)
#ifdef T6_PROFILE
#define T6W(site, bar, par)          \
  do {                               \
    const long long _t0 = clock64(); \
    t6_wait(bar, par);               \
    prof[site] += clock64() - _t0;   \
  } while (0)
#else
#define T6W(site, bar, par) t6_wait(bar, par)
#endif
__device__ __forceinline__ float t6_w(const float* gsm, int d, int R) {
  const int a = d < 0 ? -d : d;
  return a <= R ? gsm[a] : 0.f;
}
// the data exponent e of volume b (written by the temporal pass: TP_FWD16 into SC_VEXP, the stacked
// full-operator pass into the slot P.eslot names)
__device__ __forceinline__ int t6_vexp(const SpassParams& P, int b) {
  return (int)P.sc[b * kScal + (P.eslot > 0 ? P.eslot : (int)SC_VEXP)];
}

// Segment walker shared by the roles.  Units are (volume b, strip s, frame t, 64-row y-block),
// in that order (volume-major: the finalize's per-volume CTA ranges; strip-major inside a
// volume: with the grid a multiple of B x S every CTA owns a frame range of ONE strip, and the
// CTAs of the S strips walk the same frames and rows at the same pace, so a strip's x-halo
// columns are read from L2 right after its neighbour fetched them).  A CTA's unit range
// [u_begin, u_end) decomposes into column segments of ny y-blocks and ny + 1 x-blocks.
struct T6Seg {
  int bt, s, yb0, ny;
};
// Frame-range launches (time-slab schedule, P.t_cnt > 0): the units cover frames
// [t_lo, t_lo + t_cnt) of every volume only; T6Frames carries the range.
struct T6Frames {
  int T, t_lo, t_cnt;   // frames per volume, first frame and frame count of the launch
};
__device__ __forceinline__ T6Seg t6_seg(long u, long u_end, int NBY, int S, T6Frames fr) {
  const long col = u / NBY;                 // (b, s, t)
  const int yb0 = (int)(u - col * NBY);
  const int t = (int)(col % fr.t_cnt);
  const long bs = col / fr.t_cnt;
  const int s = (int)(bs % S);
  const int b = (int)(bs / S);
  return T6Seg{b * fr.T + fr.t_lo + t, s, yb0, (int)min((long)NBY - yb0, u_end - u)};
}

template <int R, int EPI>
__global__ void __launch_bounds__(k6Threads, 1) spass_tc6_kernel(const __grid_constant__ SpassParams P) {
  static_assert(R <= 40 && t6_jlo(R) >= -2 * t6_off(R), "tcgen05 spatial pass: radii <= 40");
  // Q ring: x(n) overwrites chunks 2n - 8, 2n - 7; every y-block reading them needs x-blocks <= n - 1
  static_assert(t6_clast(R) - t6_cfirst(R) + 1 <= 6, "a y window spans at most six ring chunks");
  constexpr int NBOX = t6_nbox(R), OFF = t6_off(R), CF = t6_cfirst(R);
  constexpr uint32_t SBYTES = t6_stage_bytes(R);
  constexpr int RA = t6_ra(R), NKX = t6_nkx(R), JLO = t6_jlo(R), JHI = t6_jhi(R);
  constexpr int TXMIN = t6_txmin(R), TYMIN = t6_tymin(R);
  constexpr uint32_t TXPL = 32u * t6_txrows(R), TYPL = 32u * t6_tyrows(R);
  constexpr bool OPT = EPI == EPI_FWD_OPT;
  constexpr bool PLAIN = EPI == EPI_PLAIN;   // u = G_xy v only (no F, no norm): the full operator's passes
  constexpr float TSC = (float)(1 << kF16TapExp);

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* stage = smem;                                    // [2][3 boxes][2 planes][64 rows][128 B]
  float* fbuf = reinterpret_cast<float*>(stage + k6Stages * SBYTES);  // [2][64 rows][128 cols]
  unsigned char* txb = reinterpret_cast<unsigned char*>(fbuf) + 2 * k6FBytes;   // [2 planes][TXPL]
  unsigned char* tyb = txb + 2 * TXPL;                            // [2 planes][TYPL]
  uint64_t* bars = reinterpret_cast<uint64_t*>(tyb + 2 * TYPL);
  uint64_t* b_sfull = bars;        // [2] v planes landed
  uint64_t* b_sempty = bars + 2;   // [2] x-pass done reading the stage (commit)
  uint64_t* b_d1full = bars + 4;   // [2] x-pass done (commit)
  uint64_t* b_d1empty = bars + 6;  // [2] D1 split into Q (4 splitter warps)
  uint64_t* b_d2full = bars + 8;   // [2] y-pass done (commit)
  uint64_t* b_d2empty = bars + 10; // [2] D2 drained (4 epilogue warps)
  uint64_t* b_ffull = bars + 12;   // [2] F tile landed
  uint64_t* b_sfree = bars + 14;   // [8] ring chunk dead (commit after its last y-pass)
  // [8] x-block n's Q chunks written (4 splitter warps), barrier n & 7: the splitter can finish
  // x-blocks up to 3 ahead of the issuer's wait (r_s > 32: a segment's y-blocks need the x-block
  // two past their own), so two barriers by parity would alias phases
  uint64_t* b_qfull = bars + 22;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 30);
  double* red = reinterpret_cast<double*>(bars + 32);   // 16 doubles
  int* flag = reinterpret_cast<int*>(red + 16);
  float* const gsm = reinterpret_cast<float*>(stage);   // the taps, only until the bands are built

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int H = P.H, W = P.W, Wp = P.Wp, S = P.S, T = P.T, NBY = P.NB;
  const T6Frames FR{T, P.t_cnt > 0 ? P.t_lo : 0, P.t_cnt > 0 ? P.t_cnt : T};
#ifdef T6_PROFILE
  long long prof[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const long long prof_t0 = clock64();
  unsigned long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
#endif
  const long u_begin = (long)blockIdx.x * P.U / P.G;
  const long u_end = (long)(blockIdx.x + 1) * P.U / P.G;

  if (tid <= R) gsm[tid] = P.g[tid];
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&b_sfull[i], 1);
      mbar_init(&b_sempty[i], 1);
      mbar_init(&b_d1full[i], 1);
      mbar_init(&b_d1empty[i], 4);
      mbar_init(&b_d2full[i], 1);
      mbar_init(&b_d2empty[i], 4);
      mbar_init(&b_ffull[i], 1);
    }
    for (int i = 0; i < k6Slots; ++i) {
      mbar_init(&b_sfree[i], 1);
      mbar_init(&b_qfull[i], 4);
    }
    fence_barrier_init();
    prefetch_tmap(&P.tmap);
    prefetch_tmap(&P.fmap);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(k6TmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  // the two shift-invariant Toeplitz bands (K-major, no swizzle: core matrix = 8 rows x 16 B,
  // K-adjacent at +128 B, row-group-adjacent at +256 B), two fp16 planes of g 2^12 each:
  //   Tx^T row i = x_out - 16 s (k step s), column k: g(k - i - RA)     (x-pass A)
  //   Ty^T row i = y_out - 16 kk (k step kk), column k: g(k - i)        (y-pass B)
  for (int e = tid; e < (t6_txrows(R) + t6_tyrows(R)) * 16; e += k6Threads) {
    const bool isx = e < t6_txrows(R) * 16;
    const int ee = isx ? e : e - t6_txrows(R) * 16;
    const int ii = ee >> 4, k = ee & 15;
    const float a = TSC * (isx ? t6_w(gsm, k - (ii + TXMIN) - RA, R) : t6_w(gsm, k - (ii + TYMIN), R));
    const uint32_t off = (uint32_t)(ii / 8) * 256 + (uint32_t)(k / 8) * 128 + (uint32_t)(ii % 8) * 16 + (uint32_t)(k % 8) * 2;
    unsigned char* base = isx ? txb : tyb;
    const uint32_t pls = isx ? TXPL : TYPL;
    const __half h = __float2half_rn(a);
    *reinterpret_cast<__half*>(base + off) = h;
    *reinterpret_cast<__half*>(base + pls + off) = __float2half_rn(a - __half2float(h));
  }
  fence_proxy_async();  // bands (generic stores) -> tensor core reads (async proxy)
  t6_fence_before();
  __syncthreads();
  t6_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lanebase = tmem + ((uint32_t)(32 * (warp & 3)) << 16);   // this warp's TMEM lane quarter
  const int xl = 32 * (warp & 3) + lane;                                    // this thread's TMEM lane (x_out)

  if (warp == 0) {
    // ================================================================== TMA producer
    if (lane == 0) {
#if T6_L2PF > 0
      // L2 prefetch cursor T6_L2PF x-blocks ahead of the loads (and the F tile of the y-block
      // with the same index): DRAM latency is covered beyond the two shared-memory stages
      long pu = u_begin;
      int pi = 0;
      T6Seg ps = pu < u_end ? t6_seg(pu, u_end, NBY, S, FR) : T6Seg{};
      auto l2pf = [&]() {
        if (pu >= u_end) return;
        const int prow = k6YN * ps.yb0 - 32 * OFF + k6XN * pi;
#pragma unroll
        for (int bx = 0; bx < NBOX; ++bx) tma_prefetch_3d(&P.tmap, ps.s * k6M - RA + k6BoxW * bx, prow, 2 * ps.bt);
        if (!PLAIN && pi < ps.ny) tma_prefetch_3d(&P.fmap, ps.s * k6M, k6YN * (ps.yb0 + pi), ps.bt);
        if (++pi >= t6_nx(R, ps.ny)) {
          pu += ps.ny;
          pi = 0;
          if (pu < u_end) ps = t6_seg(pu, u_end, NBY, S, FR);
        }
      };
      for (int k = 0; k < T6_L2PF; ++k) l2pf();
#endif
      unsigned n = 0;
      for (long u = u_begin; u < u_end;) {
        const T6Seg sg = t6_seg(u, u_end, NBY, S, FR);
        const int x0 = sg.s * k6M - RA;
        for (int i = 0; i < t6_nx(R, sg.ny); ++i, ++n) {
#if T6_L2PF > 0
          l2pf();
#endif
          const unsigned st = n & 1;
          T6W(0, &b_sempty[st], ((n >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&b_sfull[st], SBYTES);
          const int row0 = k6YN * sg.yb0 - 32 * OFF + k6XN * i;
#pragma unroll
          for (int bx = 0; bx < NBOX; ++bx)
            tma_load_3d(stage + st * SBYTES + bx * k6BoxBytes, &P.tmap, &b_sfull[st], x0 + k6BoxW * bx, row0,
                        2 * sg.bt);
        }
        u += sg.ny;
      }
    }
  } else if (warp == 1) {
    // ================================================================== MMA issuer (warp-converged)
    {
      const uint32_t idx = t6_idesc(k6XN), idy = t6_idesc(k6YN);
      const uint32_t st0 = smem_u32(stage);
      const uint64_t ad0 = t6_desc_none(smem_u32(txb), 128, 256), yd0 = t6_desc_none(smem_u32(tyb), 128, 256);
      long yu = u_begin;
      T6Seg ys{};
      int yj = 0, yrel = 0;
      bool yhave = false;
      unsigned yg0 = 0, ny = 0, nq = 0, nx = 0;
      auto y_next = [&]() -> bool {
        if (yhave && ++yj < ys.ny) return true;
        if (yhave) {
          yu += ys.ny;
          yg0 += (unsigned)t6_nx(R, ys.ny);
        }
        if (yu >= u_end) return false;
        ys = t6_seg(yu, u_end, NBY, S, FR);
        yj = 0;
        yrel = 0;
        yhave = true;
        return true;
      };
#if T6_XSTACK
      const uint32_t idx2 = t6_idesc(2 * k6XN);
      auto issue_x = [&]() {
        const unsigned st = nx & 1;
        T6W(2, &b_sfull[st], (nx >> 1) & 1);
        T6W(3, &b_d1empty[0], (nx & 1) ^ 1);
        t6_fence_after();
        const uint32_t d = tmem + k6ColD1;
        const uint64_t bd0 = t6_desc_sw128(st0 + st * SBYTES);
        // A: tap plane pg at k step s; B: k step s of the box, from data plane 0 (N = 64: plane 0 only,
        // N = 128: planes 0 and 1, contiguous 64-row halves of the box)
        auto adesc = [&](int pg, int s) {
          return ad0 + (uint64_t)((pg * TXPL + (uint32_t)(-16 * s - TXMIN) * 32) >> 4);
        };
        auto bdesc = [&](int s) { return bd0 + (uint64_t)(((s >> 2) * k6BoxBytes + (s & 3) * 32) >> 4); };
        // k step 0 of the leading tap plane initialises both halves [a_hi g_hi | a_lo g_hi]; then the
        // correction a_hi g_lo (hi half), then the remaining leading k steps
        t6_mma_ss_e(d, adesc(0, 0), bdesc(0), idx2, 0u);
#pragma unroll
        for (int s = 0; s < NKX; ++s) t6_mma_ss_e(d, adesc(1, s), bdesc(s), idx, 1u);
#pragma unroll
        for (int s = 1; s < NKX; ++s) t6_mma_ss_e(d, adesc(0, s), bdesc(s), idx2, 1u);
        t6_commit_e(&b_sempty[st]);
        t6_commit_e(&b_d1full[0]);
        ++nx;
      };
#else
      auto issue_x = [&]() {
        const unsigned st = nx & 1, db = nx & 1;
        T6W(2, &b_sfull[st], (nx >> 1) & 1);
        T6W(3, &b_d1empty[db], ((nx >> 1) & 1) ^ 1);
        t6_fence_after();
        const uint32_t d = tmem + k6ColD1 + k6XN * db;
        const uint64_t bd0 = t6_desc_sw128(st0 + st * SBYTES);
        // products (data plane, tap plane): the two corrections first, the leading one last.
        // Descriptor start addresses advance by (byte offset >> 4) in the low field.
#pragma unroll
        for (int pp = 0; pp < 3; ++pp) {
          const int pa = pp == 0 ? 1 : 0, pg = pp == 1 ? 1 : 0;
#pragma unroll
          for (int s = 0; s < NKX; ++s) {
            const uint64_t ad = ad0 + (uint64_t)((pg * TXPL + (uint32_t)(-16 * s - TXMIN) * 32) >> 4);
            const uint64_t bd = bd0 + (uint64_t)(((s >> 2) * k6BoxBytes + pa * k6PlaneBox + (s & 3) * 32) >> 4);
            t6_mma_ss_e(d, ad, bd, idx, (pp > 0 || s > 0) ? 1u : 0u);
          }
        }
        t6_commit_e(&b_sempty[st]);
        t6_commit_e(&b_d1full[db]);
        ++nx;
      };
#endif
      auto issue_y = [&]() {
        const unsigned need = yg0 + (unsigned)t6_xneed(R, yj);
        while (nq <= need) {
          T6W(4, &b_qfull[nq & 7], (nq >> 3) & 1);
          ++nq;
        }
        const unsigned buf = ny & 1;
        T6W(5, &b_d2empty[buf], ((ny >> 1) & 1) ^ 1);
        t6_fence_after();
        const uint32_t d = tmem + k6ColD2 + k6YN * buf;
        const uint32_t c0 = 2u * yg0 + 2u * (unsigned)yj;   // first chunk of the window (CTA-wide index)
#pragma unroll
        for (int pp = 0; pp < 3; ++pp) {
          const int pa = pp == 0 ? 1 : 0, pg = pp == 1 ? 1 : 0;
#pragma unroll
          for (int kk = JLO; kk < JHI; ++kk) {
            const uint32_t slot = (c0 + (unsigned)((kk + 2 * OFF) / 2)) % k6Slots;
            const uint32_t a = tmem + k6ColQ + 32 * slot + 16 * pa + 8 * ((kk + 2 * OFF) & 1);
            const uint64_t bd = yd0 + (uint64_t)((pg * TYPL + (uint32_t)(-16 * kk - TYMIN) * 32) >> 4);
            t6_mma_ts_e(d, a, bd, idy, (pp > 0 || kk > JLO) ? 1u : 0u);
          }
        }
        t6_commit_e(&b_d2full[buf]);
        // chunks no later y-block of the segment reads are dead
        const int target = (yj + 1 < ys.ny) ? 2 * (yj + 1) + CF : 2 * t6_nx(R, ys.ny);
        for (; yrel < target; ++yrel) t6_commit_e(&b_sfree[(2u * yg0 + (unsigned)yrel) % k6Slots]);
        ++ny;
      };
      bool ymore = y_next();
      for (long u = u_begin; u < u_end;) {
        const T6Seg sg = t6_seg(u, u_end, NBY, S, FR);
        for (int i = 0; i < t6_nx(R, sg.ny); ++i) {
          issue_x();
          // y-blocks whose x-blocks were all issued before this one (their split ran under it)
          while (ymore && yg0 + (unsigned)t6_xneed(R, yj) + 2 <= nx) {
            issue_y();
            ymore = y_next();
          }
        }
        u += sg.ny;
      }
      while (ymore) {
        issue_y();
        ymore = y_next();
      }
    }
  } else if (warp < 6) {
    // ================================================================== splitters (warps 2-5)
    unsigned total = 0;
    for (long u = u_begin; u < u_end;) {
      const T6Seg sg = t6_seg(u, u_end, NBY, S, FR);
      total += (unsigned)t6_nx(R, sg.ny);
      u += sg.ny;
    }
    constexpr float QSC = 1.f / (float)(1 << kF16TapExp);
#pragma unroll 1
    for (unsigned n = 0; n < total; ++n) {
#if T6_XSTACK
      // D1 (single buffer) = [hi half | lo half]: the two halves summed in fp32, D1 released as soon as
      // both 32-row chunks are in registers
      T6W(6, &b_d1full[0], n & 1);
      t6_fence_after();
      float sum[2][32];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t a[32], b[32];
        __syncwarp();
        t6_ld32(lanebase + k6ColD1 + 32 * c, a);
        t6_ld32(lanebase + k6ColD1 + k6XN + 32 * c, b);
        t6_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) sum[c][i] = __uint_as_float(a[i]) + __uint_as_float(b[i]);
      }
      t6_fence_before();
      __syncwarp();
      if (lane == 0) t6_arrive(&b_d1empty[0]);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          uint32_t pl[2];
          split_planes_f16<2>(sum[c][2 * i] * QSC, sum[c][2 * i + 1] * QSC, pl);
          hi[i] = pl[0];
          lo[i] = pl[1];
        }
        const unsigned gc = 2 * n + c, slot = gc % k6Slots;
        T6W(7, &b_sfree[slot], ((gc / k6Slots) & 1) ^ 1);
        t6_fence_after();
        __syncwarp();
        t6_st16(lanebase + k6ColQ + 32 * slot, hi);
        t6_st16(lanebase + k6ColQ + 32 * slot + 16, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      t6_fence_before();
      __syncwarp();
      if (lane == 0) t6_arrive(&b_qfull[n & 7]);
#else
      const unsigned db = n & 1;
      T6W(6, &b_d1full[db], (n >> 1) & 1);
      t6_fence_after();
#endif
#if T6_XSTACK
#elif T6_LDALL
      // both 32-row halves of D1 in one round trip; D1 is released before the split (the
      // issuer's next x-pass into this buffer no longer waits for the stores into the ring)
      uint32_t d[2][32];
      __syncwarp();
      t6_ld32(lanebase + k6ColD1 + k6XN * db, d[0]);
      t6_ld32(lanebase + k6ColD1 + k6XN * db + 32, d[1]);
      t6_wait_ld();
      t6_fence_before();
      __syncwarp();
      if (lane == 0) t6_arrive(&b_d1empty[db]);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          uint32_t pl[2];
          split_planes_f16<2>(__uint_as_float(d[c][2 * i]) * QSC, __uint_as_float(d[c][2 * i + 1]) * QSC, pl);
          hi[i] = pl[0];
          lo[i] = pl[1];
        }
        const unsigned gc = 2 * n + c, slot = gc % k6Slots;
        T6W(7, &b_sfree[slot], ((gc / k6Slots) & 1) ^ 1);
        t6_fence_after();
        __syncwarp();
        t6_st16(lanebase + k6ColQ + 32 * slot, hi);
        t6_st16(lanebase + k6ColQ + 32 * slot + 16, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      t6_fence_before();
      __syncwarp();
      if (lane == 0) t6_arrive(&b_qfull[n & 7]);
#else
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t d[32];
        __syncwarp();
        t6_ld32(lanebase + k6ColD1 + k6XN * db + 32 * c, d);
        t6_wait_ld();
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          uint32_t pl[2];
          split_planes_f16<2>(__uint_as_float(d[2 * i]) * QSC, __uint_as_float(d[2 * i + 1]) * QSC, pl);
          hi[i] = pl[0];
          lo[i] = pl[1];
        }
        const unsigned gc = 2 * n + c, slot = gc % k6Slots;
        T6W(7, &b_sfree[slot], ((gc / k6Slots) & 1) ^ 1);
        t6_fence_after();
        __syncwarp();
        t6_st16(lanebase + k6ColQ + 32 * slot, hi);
        t6_st16(lanebase + k6ColQ + 32 * slot + 16, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      t6_fence_before();
      __syncwarp();
      if (lane == 0) {
        t6_arrive(&b_d1empty[db]);
        t6_arrive(&b_qfull[n & 7]);
      }
#endif
    }
  } else {
    // ================================================================== epilogue (warps 6-9)
    const int wg = warp - 6;
    double acc0 = 0.0, acc1 = 0.0;
    float pmax = 0.f;
    int cur_vol = -1;
    float usc = 1.f;
    auto flush = [&](int vol) {   // fixed-order sum over the group's 128 threads (named barrier 1)
      double s0 = acc0, s1 = acc1;
      float mx = pmax;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (lane == 0) {
        red[wg] = s0;
        red[4 + wg] = s1;
        reinterpret_cast<float*>(red + 8)[wg] = mx;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (wg == 0 && lane == 0) {
        P.partials[(long)vol * P.G + blockIdx.x] = ((red[0] + red[1]) + red[2]) + red[3];
        P.partials[(long)(P.B + vol) * P.G + blockIdx.x] = ((red[4] + red[5]) + red[6]) + red[7];
        if (P.pslot > 0) {   // max |p_k| of the volume for the next temporal pass (order-free)
          const float* mm = reinterpret_cast<const float*>(red + 8);
          const float m4 = fmaxf(fmaxf(mm[0], mm[1]), fmaxf(mm[2], mm[3]));
          atomicMax(reinterpret_cast<unsigned*>(P.sc + vol * kScal + SC_VMAX + P.pslot - 1), __float_as_uint(m4));
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      acc0 = acc1 = 0.0;
      pmax = 0.f;
    };
    // F tiles: loaded by TMA two y-blocks ahead by thread 0 of the group (lookahead cursor fu/fj)
    const bool fissuer = wg == 0 && lane == 0;
    long fu = u_begin;
    T6Seg fs{};
    int fj = 0;
    bool fhave = false;
    auto f_issue = [&](unsigned fb) {   // next F tile of the lookahead cursor into buffer fb
      if (fhave && ++fj >= fs.ny) {
        fu += fs.ny;
        fhave = false;
      }
      if (!fhave) {
        if (fu >= u_end) return;
        fs = t6_seg(fu, u_end, NBY, S, FR);
        fj = 0;
        fhave = true;
      }
      mbar_arrive_expect_tx(&b_ffull[fb], k6FBytes);
      tma_load_3d(reinterpret_cast<unsigned char*>(fbuf) + fb * k6FBytes, &P.fmap, &b_ffull[fb], fs.s * k6M,
                  k6YN * (fs.yb0 + fj), fs.bt);
    };
    if (fissuer && !PLAIN) {
      f_issue(0);
      f_issue(1);
    }
    unsigned m = 0;
    for (long u = u_begin; u < u_end;) {
      const T6Seg sg = t6_seg(u, u_end, NBY, S, FR);
      const int vol = sg.bt / T;
      if (vol != cur_vol) {
        if (cur_vol >= 0 && !PLAIN) flush(cur_vol);
        cur_vol = vol;
        usc = pow2f(-t6_vexp(P, vol) - kF16TapExp) * (P.lag ? (float)P.sc[vol * kScal + SC_S] : 1.f);
      }
      const int x = sg.s * k6M + xl;
      const bool xin = x < Wp;
      const float cmask = x < W ? 1.f : 0.f;
#pragma unroll 1
      for (int j = 0; j < sg.ny; ++j, ++m) {
        const int y0 = k6YN * (sg.yb0 + j);
        const int nrow = min(k6YN, H - y0);
        const long base = ((long)sg.bt * H + y0) * Wp + x;
        const unsigned buf = m & 1;
        const float* ft = fbuf + buf * (k6FBytes / 4) + xl;
        if (!PLAIN) T6W(8, &b_ffull[buf], (m >> 1) & 1);
        T6W(9, &b_d2full[buf], (m >> 1) & 1);
        t6_fence_after();
        float s0 = 0.f, s1 = 0.f;
#if T6_LDALL
        // the whole 64-row D2 buffer in one round trip, released before the stores
        uint32_t qa[2][32];
        __syncwarp();
        t6_ld32(lanebase + k6ColD2 + k6YN * buf, qa[0]);
        t6_ld32(lanebase + k6ColD2 + k6YN * buf + 32, qa[1]);
        t6_wait_ld();
        t6_fence_before();
        __syncwarp();
        if (lane == 0) t6_arrive(&b_d2empty[buf]);
#pragma unroll
        for (int c = 0; c < k6YN / 16; ++c) {
          const uint32_t* q = &qa[c >> 1][16 * (c & 1)];
          if (!xin) break;
#else
#pragma unroll 1
        for (int c = 0; c < k6YN / 16; ++c) {
          uint32_t q[16];
          __syncwarp();
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
                "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
              : "r"(lanebase + k6ColD2 + k6YN * buf + 16 * c)
              : "memory");
          t6_wait_ld();
          if (!xin) continue;
#endif
          // one element per row: F from the shared tile, p (and the options) stored through
          // running pointers; full 16-row chunks take the branch-free path
          const int r0 = 16 * c;
          const float* fr = ft + r0 * k6M;
          float* op = P.out + base + (long)r0 * Wp;
          if (PLAIN) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if (r0 + i >= nrow) break;
              *op = __uint_as_float(q[i]) * usc * cmask;
              op += Wp;
            }
          } else if (r0 + 16 <= nrow && (!OPT || !P.pprev)) {
            // full chunk: branch-free, running pointers (the training forward's tape u included)
            float* tp = OPT ? P.tape_u + (base + (long)r0 * Wp) : nullptr;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float f = fr[i * k6M];
              const float uu = __uint_as_float(q[i]) * usc;
              const float yv = f * uu;
              s0 = fmaf(yv, yv, s0);
              const float pv = P.last ? yv : f * yv;
              pmax = fmaxf(pmax, fabsf(pv));
              *op = pv;
              op += Wp;
              if (OPT && tp) {
                *tp = uu * cmask;
                tp += Wp;
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              if (r0 + i >= nrow) break;
              const long off = base + (long)(r0 + i) * Wp;
              const float f = fr[i * k6M];
              const float uu = __uint_as_float(q[i]) * usc;
              const float yv = f * uu;
              s0 = fmaf(yv, yv, s0);
              if (OPT) {
                if (P.pprev) s1 = fmaf(__ldcg(P.pprev + off), uu * cmask, s1);
                if (P.tape_u) P.tape_u[off] = uu * cmask;
              }
              const float pv = P.last ? yv : f * yv;
              pmax = fmaxf(pmax, fabsf(pv));
              P.out[off] = pv;
            }
          }
        }
#if !T6_LDALL
        t6_fence_before();
        __syncwarp();
        if (lane == 0) t6_arrive(&b_d2empty[buf]);
#endif
        if (!PLAIN) {
          asm volatile("bar.sync 2, 128;" ::: "memory");   // the group is done reading F tile buf
          if (fissuer) f_issue(buf);
        }
        acc0 += (double)s0;
        acc1 += (double)s1;
      }
      u += sg.ny;
    }
    if (cur_vol >= 0 && !PLAIN) flush(cur_vol);
  }
#ifdef T6_PROFILE
  if (warp == 6 && lane == 0) {
    unsigned long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    printf("[t6cta] %d %lld %llu %llu\n", blockIdx.x, clock64() - prof_t0, g0, g1);
  }
  if (blockIdx.x == 0 && lane == 0 && (warp <= 2 || warp == 6))
    printf("[t6prof] warp %d total %lld waits: prod sempty %lld fempty %lld | iss sfull %lld d1empty %lld qfull %lld "
           "d2empty %lld | split d1full %lld sfree %lld | epi ffull %lld d2full %lld\n",
           warp, clock64() - prof_t0, prof[0], prof[1], prof[2], prof[3], prof[4], prof[5], prof[6], prof[7], prof[8],
           prof[9]);
#endif
  t6_fence_before();
  __syncthreads();
  if (warp == 0) {
    t6_fence_after();
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(k6TmemCols));
  }
  if (!PLAIN) spass_finalize<SP_FWD, k6Threads>(P, red, flag);
}

}  // namespace sfseg
