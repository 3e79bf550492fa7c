// Once-per-solve kernels: channel combine (Eq.9), final normalisation (Eq.8),
// hard threshold (reading A12), and the backward's set-up and
// final contraction (Appendix A).  All are HBM-streaming elementwise kernels
// over the pitched volume; reductions use per-block partials and a fixed-order
// fp64 finalize in the last block (deterministic).
#pragma once
#include "common.cuh"
#include "spass.cuh"

namespace sfseg {

constexpr int kEwThreads = 256;

// ------------------------------------------------------------------ combine (+ x_0, p_0, ||x_0||)
struct CombineParams {
  const float* ch;      // dense [B][C][T][H][W]
  const float* x0;      // dense [B][T][H][W] or null (x_0 = F)
  float* F;             // pitched [B*T][H][Wp]
  float* p0;            // pitched: p_0 = F * x_0 (null: skip)
  float* F_out;         // dense or null
  float* x0p;           // pitched copy of x0 (null: skip)
  double* sc;
  double* partials;     // [B][T*gx]
  unsigned* counter;
  unsigned* err;
  double* loc;          // time-slab mode: per-volume local sum of x_0^2 -> loc[2b]
  unsigned* pmax;       // max |p_0| per volume (float bits, stride 2 kScal words; tcgen05 pass) or null
  unsigned* fmax;       // max |F| per volume (the tcgen05 backward's range bound) or null
  int B, C, T, H, W, Wp, act, gx;
  int in_T, in_t0;      // ch / x0 buffers hold in_T frames; this call's frame t is buffer frame in_t0 + t
  float bias;
  float w[kMaxC];
};

// Row-parallel layout shared by the streaming kernels: grid (gx, B*T); block
// (bx, bt) handles rows y = bx*kRows + j (+ gx*kRows per pass) of frame bt;
// thread tid covers columns tid + i*kEwThreads.  Lanes map to consecutive
// columns (coalesced 128-byte rows for dense and pitched layouts alike); kRows
// rows x kCols column chunks are unrolled so every thread keeps kRows*kCols
// independent loads in flight (HBM latency hiding without any index division).
constexpr int kRows = 4;
constexpr int kCols = 4;

__global__ void __launch_bounds__(kEwThreads) combine_kernel(const __grid_constant__ CombineParams P) {
  __shared__ double red[kEwThreads / 32];
  __shared__ int flag;
  const int bt = blockIdx.y;
  const int b = bt / P.T, t = bt - b * P.T;
  const long HWp = (long)P.H * P.Wp, HW = (long)P.H * P.W;
  const long vol_dense = (long)P.in_T * HW;
  const float* chf = P.ch + (long)b * P.C * vol_dense + (long)(P.in_t0 + t) * HW;  // frame base, channel 0
  const long dbase = (long)b * vol_dense + (long)(P.in_t0 + t) * HW;              // dense x0 / F_out frame base
  double acc = 0.0;
  float pm = 0.f, fm = 0.f;
  for (int y0 = blockIdx.x * kRows; y0 < P.H; y0 += P.gx * kRows) {
    for (int c0 = 0; c0 < P.Wp; c0 += kEwThreads * kCols) {
      float z[kRows][kCols];
#pragma unroll
      for (int r = 0; r < kRows; ++r)
#pragma unroll
        for (int i = 0; i < kCols; ++i) z[r][i] = P.bias;
      for (int c = 0; c < P.C; ++c) {
        float v[kRows][kCols];
#pragma unroll
        for (int r = 0; r < kRows; ++r)
#pragma unroll
          for (int i = 0; i < kCols; ++i) {
            const int y = y0 + r, x = c0 + i * kEwThreads + threadIdx.x;
            v[r][i] = (y < P.H && x < P.W) ? __ldcs(chf + (long)c * vol_dense + (long)y * P.W + x) : 0.f;
          }
#pragma unroll
        for (int r = 0; r < kRows; ++r)
#pragma unroll
          for (int i = 0; i < kCols; ++i) z[r][i] = fmaf(P.w[c], v[r][i], z[r][i]);
      }
      float xv[kRows][kCols];
#pragma unroll
      for (int r = 0; r < kRows; ++r)
#pragma unroll
        for (int i = 0; i < kCols; ++i) {
          const int y = y0 + r, x = c0 + i * kEwThreads + threadIdx.x;
          xv[r][i] = 0.f;
          if (P.x0 && y < P.H && x < P.W) xv[r][i] = __ldcs(P.x0 + dbase + (long)y * P.W + x);
        }
      float ps = 0.f;  // ||x_0||^2 of this thread's kRows x kCols values in fp32, then into the fp64 sum
                       // (as the spatial pass's norm partials: one fp64 add per 16 values, not per value)
#pragma unroll
      for (int r = 0; r < kRows; ++r)
#pragma unroll
        for (int i = 0; i < kCols; ++i) {
          const int y = y0 + r, x = c0 + i * kEwThreads + threadIdx.x;
          if (y >= P.H || x >= P.Wp) continue;
          const long po = (long)bt * HWp + (long)y * P.Wp + x;
          float f = 0.f, pv = 0.f, xx = 0.f;
          if (x < P.W) {
            f = (P.act == 1) ? 1.f / (1.f + expf(-z[r][i])) : z[r][i];
            xx = P.x0 ? xv[r][i] : f;
            pv = f * xx;
            pm = fmaxf(pm, fabsf(pv));
            fm = fmaxf(fm, fabsf(f));
            if (P.F_out) P.F_out[dbase + (long)y * P.W + x] = f;
            ps = fmaf(xx, xx, ps);
          }
          P.F[po] = f;  // pad columns x >= W hold zeros
          if (P.p0) P.p0[po] = pv;
          if (P.x0p) P.x0p[po] = xx;
        }
      acc += (double)ps;
    }
  }
  if (P.pmax) {   // order-free max: one atomic per warp
    const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(pm));
    if ((threadIdx.x & 31) == 0) atomicMax(P.pmax + (long)b * 2 * kScal, m);
  }
  if (P.fmax) {
    const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(fm));
    if ((threadIdx.x & 31) == 0) atomicMax(P.fmax + (long)b * 2 * kScal, m);
  }
  if (P.partials == nullptr) return;  // plain combine (sfseg_combine_channels): no reduction
  const double s = block_sum<kEwThreads>(acc, red);
  const long nper = (long)P.T * P.gx;
  if (threadIdx.x == 0) P.partials[(long)b * nper + (long)t * P.gx + blockIdx.x] = s;
  if (!last_block_arrive(P.counter, gridDim.x * gridDim.y, &flag)) return;
  for (int bb = 0; bb < P.B; ++bb) {
    const double tot = block_sum_array<kEwThreads>(P.partials + (long)bb * nper, nper, 1, red);
    if (threadIdx.x == 0) {
      if (P.loc) {
        P.loc[2 * bb] = tot;
        P.loc[2 * bb + 1] = 0.0;
      } else {
        const double xn = sqrt(tot);
        P.sc[bb * kScal + SC_XNORM] = xn;
        P.sc[bb * kScal + SC_S] = 1.0;
        flag_norm(P.err, xn);
      }
    }
  }
  if (threadIdx.x == 0) *P.counter = 0u;
}

// ------------------------------------------------------------------ time-slab finalizers (after the allreduce)
struct FinParams {
  const double* glob;   // [B][2] global sums
  double* sc;
  double* stats;
  double* tape_nu;
  unsigned* err;
  int B, K, k, rayleigh;
};

// k == 0: combine (||x_0||); k >= 1: forward iteration k.
__global__ void finalize_kernel(const __grid_constant__ FinParams P) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= P.B) return;
  double* sc = P.sc + b * kScal;
  if (P.k == 0) {
    const double xn = sqrt(P.glob[2 * b]);
    sc[SC_XNORM] = xn;
    sc[SC_S] = 1.0;
    flag_norm(P.err, xn);
  } else {
    fwd_finalize(sc, P.stats, P.tape_nu, P.err, P.K, P.k, P.rayleigh != 0, b, P.glob[2 * b], P.glob[2 * b + 1]);
  }
}

// In-process "allreduce" for emulated ranks on one GPU: glob_r = sum over ranks (rank order) of loc_r.
constexpr int kMaxLocalRanks = 16;
struct LocalReduceParams {
  const double* loc[kMaxLocalRanks];
  double* glob[kMaxLocalRanks];
  int nranks, n;
};
__global__ void local_allreduce_kernel(const __grid_constant__ LocalReduceParams P) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  double s = 0.0;
  for (int r = 0; r < P.nranks; ++r) s += P.loc[r][i];
  for (int r = 0; r < P.nranks; ++r) P.glob[r][i] = s;
}

// ------------------------------------------------------------------ final normalisation x_K = y_K / nu_K
// x (dense, buffer of out_T frames per volume; this slab starts at frame out_t0).  grid (gx, B*T).
__global__ void __launch_bounds__(kEwThreads) final_scale_kernel(const float* __restrict__ y, float* __restrict__ x,
                                                                 const double* sc, int T, int H, int W, int Wp,
                                                                 int out_T, int out_t0) {
  const int bt = blockIdx.y, b = bt / T, t = bt - b * T;
  const float s = (float)sc[b * kScal + SC_S];
  const long HW = (long)H * W;
  float* xo = x + ((long)b * out_T + out_t0 + t) * HW;
  const float* yi = y + (long)bt * H * Wp;
  for (int y0 = blockIdx.x * kRows; y0 < H; y0 += gridDim.x * kRows) {
    for (int c0 = 0; c0 < W; c0 += kEwThreads * kCols) {
      float v[kRows][kCols];
#pragma unroll
      for (int r = 0; r < kRows; ++r)
#pragma unroll
        for (int i = 0; i < kCols; ++i) {
          const int yy = y0 + r, xx = c0 + i * kEwThreads + threadIdx.x;
          v[r][i] = (yy < H && xx < W) ? __ldcs(yi + (long)yy * Wp + xx) : 0.f;
        }
#pragma unroll
      for (int r = 0; r < kRows; ++r)
#pragma unroll
        for (int i = 0; i < kCols; ++i) {
          const int yy = y0 + r, xx = c0 + i * kEwThreads + threadIdx.x;
          if (yy < H && xx < W) xo[(long)yy * W + xx] = v[r][i] * s;   // plain store: the threshold's frame max reads x next
        }
    }
  }
}

// ------------------------------------------------------------------ time-slab fp16 range
// Time slabs on the tcgen05 path: the temporal pass TP_FWD16 picks its fp16 exponent from
// max |p_{k-1}| over every frame it reads, and the r_t halo frames received from the neighbour
// slabs are among them.  halo_absmax_kernel folds max |halo| of volume blockIdx.y (halo
// blockIdx.z: 0 lower, 1 upper; [B][n4] float4 each, null = absent) into the volume's slot
// (float bits, order-free atomicMax; stride 2 kScal words as the spatial pass's own maximum).
__global__ void __launch_bounds__(kEwThreads) halo_absmax_kernel(const float4* __restrict__ lo,
                                                                 const float4* __restrict__ hi, long n4,
                                                                 unsigned* slot) {
  const float4* h = blockIdx.z == 0 ? lo : hi;
  if (h == nullptr) return;
  h += (long)blockIdx.y * n4;
  float m = 0.f;
  const long step = (long)gridDim.x * kEwThreads;
  long e = (long)blockIdx.x * kEwThreads + threadIdx.x;
  for (; e + 3 * step < n4; e += 4 * step) {
    float4 a[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = __ldg(h + e + i * step);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      m = fmaxf(m, fmaxf(fmaxf(fabsf(a[i].x), fabsf(a[i].y)), fmaxf(fabsf(a[i].z), fabsf(a[i].w))));
  }
  for (; e < n4; e += step) {
    const float4 a = __ldg(h + e);
    m = fmaxf(m, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
  }
  const unsigned w = __reduce_max_sync(0xffffffffu, __float_as_uint(m));
  if ((threadIdx.x & 31) == 0 && w != 0u) atomicMax(slot + (long)blockIdx.y * 2 * kScal, w);
}

// ------------------------------------------------------------------ threshold
// Per-frame maximum in two deterministic steps (max is order independent):
// frame_max_kernel writes one partial per (frame, block) -> part[bt * gx + bx],
// threshold_kernel folds the gx partials of its frame (or of the whole volume).
constexpr int kThrGx = 16;

__global__ void __launch_bounds__(kEwThreads) frame_max_kernel(const float* __restrict__ x, float* part, long HW) {
  __shared__ float red[kEwThreads / 32];
  // frames last to first: x was just written first to last (final scale), so the frames still in
  // L2 are read first; the threshold kernel then walks first to last over what this pass read last
  const long bt = (long)gridDim.y - 1 - blockIdx.y;
  const float* xf = x + bt * HW;
  float m = -INFINITY;
  const bool vec = ((HW & 3) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  if (vec) {
    const float4* x4 = reinterpret_cast<const float4*>(xf);
    const long n4 = HW >> 2;
    long e = (long)blockIdx.x * kEwThreads + threadIdx.x;
    const long step = (long)gridDim.x * kEwThreads;
    for (; e + 3 * step < n4; e += 4 * step) {
      float4 a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = __ldg(x4 + e + i * step);
#pragma unroll
      for (int i = 0; i < 4; ++i) m = fmaxf(m, fmaxf(fmaxf(a[i].x, a[i].y), fmaxf(a[i].z, a[i].w)));
    }
    for (; e < n4; e += step) {
      const float4 a = __ldg(x4 + e);
      m = fmaxf(m, fmaxf(fmaxf(a.x, a.y), fmaxf(a.z, a.w)));
    }
  } else {
    for (long e = (long)blockIdx.x * kEwThreads + threadIdx.x; e < HW; e += (long)gridDim.x * kEwThreads)
      m = fmaxf(m, __ldg(xf + e));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float r = red[0];
    for (int i = 1; i < kEwThreads / 32; ++i) r = fmaxf(r, red[i]);
    part[bt * gridDim.x + blockIdx.x] = r;
  }
}

// grid (gx, B*T); `part` holds npart partials per frame (ignored for mode 2).
__global__ void __launch_bounds__(kEwThreads) threshold_kernel(const float* __restrict__ x, uint8_t* __restrict__ mask,
                                                               const float* part, int npart, int T, long HW, float tau,
                                                               int mode) {
  const int bt = blockIdx.y, b = bt / T;
  float thr;
  bool none = false;
  if (mode == 2) {
    thr = tau;
  } else {
    float m = -INFINITY;
    const int f0 = (mode == 0) ? bt : b * T, f1 = (mode == 0) ? bt + 1 : (b + 1) * T;
    for (long i = (long)f0 * npart; i < (long)f1 * npart; ++i) m = fmaxf(m, part[i]);
    none = !(m > 0.f);
    thr = tau * m;
  }
  const long base = (long)bt * HW;
  const bool vec = ((HW & 3) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(mask) & 3) == 0);
  if (vec) {
    const float4* x4 = reinterpret_cast<const float4*>(x + base);
    uchar4* m4 = reinterpret_cast<uchar4*>(mask + base);
    const long n4 = HW >> 2;
    for (long e = (long)blockIdx.x * kEwThreads + threadIdx.x; e < n4; e += (long)gridDim.x * kEwThreads) {
      const float4 a = __ldcs(x4 + e);
      uchar4 o;
      o.x = (!none && a.x > thr) ? 1 : 0;
      o.y = (!none && a.y > thr) ? 1 : 0;
      o.z = (!none && a.z > thr) ? 1 : 0;
      o.w = (!none && a.w > thr) ? 1 : 0;
      __stcs(m4 + e, o);
    }
  } else {
    for (long e = (long)blockIdx.x * kEwThreads + threadIdx.x; e < HW; e += (long)gridDim.x * kEwThreads)
      mask[base + e] = (!none && x[base + e] > thr) ? 1 : 0;
  }
}

// ------------------------------------------------------------------ backward set-up: x_bar_K, F_bar = 0, c_K
struct BwdInitParams {
  const float* g;       // dense dL/dx_K [B][T][H][W]
  const float* F;       // pitched
  const float* uK1;     // tape u_{K-1} pitched
  float* xbar;          // pitched
  float* Fbar;          // pitched (zeroed)
  const double* tape_nu;
  double* sc;
  double* partials;
  unsigned* counter;
  const double* tape_bin;  // [B][K][2] of the binarised iterations (row f2)
  float kappa;             // steepness of iteration K (0: not binarised; then g is dL/dx_K)
  double* loc;             // time slabs: per-volume local sums [B][2] (finalized after the allreduce)
  int B, T, H, W, Wp, K, gx;
  int g_T, g_t0;           // dL/dx buffer frames per volume and this slab's first frame in it
  unsigned* xbmax;         // max |x_bar_K| per volume (float bits, stride 2 kScal words) or null
};

// x_bar_K = dL/dx_K, c_K = <x_K, x_bar_K>.  When iteration K was soft-binarised the output is
// b_K = sigma(kappa (x_K - theta)) and g is its adjoint: x_bar holds kappa sigma' g and the
// finalize forms corr and c_K as in bwd_epi_kernel (bwd.cuh).
__global__ void __launch_bounds__(kEwThreads) bwd_init_kernel(const __grid_constant__ BwdInitParams P) {
  __shared__ double red[kEwThreads / 32];
  __shared__ int flag;
  const int bt = blockIdx.y;
  const int b = bt / P.T, t = bt - b * P.T;
  const long HWp = (long)P.H * P.Wp, HW = (long)P.H * P.W;
  const float* gf = P.g + ((long)b * P.g_T + P.g_t0 + t) * HW;
  const bool bin = P.kappa > 0.f;
  const float inv_nuK = (float)(1.0 / P.tape_nu[(long)b * P.K + (P.K - 1)]);
  const float theta = bin ? (float)P.tape_bin[((long)b * P.K + (P.K - 1)) * 2] : 0.f;
  double acc = 0.0, acc2 = 0.0;
  float xm = 0.f;
  // row-parallel (see combine_kernel): no per-element index division
  for (int y = blockIdx.x; y < P.H; y += P.gx) {
    for (int c0 = 0; c0 < P.Wp; c0 += kEwThreads * kCols) {
      float gv[kCols], fv[kCols], uv[kCols];
#pragma unroll
      for (int i = 0; i < kCols; ++i) {  // all loads of the kCols columns first (memory parallelism)
        const int x = c0 + i * kEwThreads + threadIdx.x;
        const long po = (long)bt * HWp + (long)y * P.Wp + x;
        const bool in = x < P.W;
        gv[i] = in ? __ldcs(gf + (long)y * P.W + x) : 0.f;
        fv[i] = in ? P.F[po] : 0.f;
        uv[i] = in ? __ldcs(P.uK1 + po) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < kCols; ++i) {
        const int x = c0 + i * kEwThreads + threadIdx.x;
        if (x >= P.Wp) continue;
        const long po = (long)bt * HWp + (long)y * P.Wp + x;
        if (bin) {
          const float xk = fv[i] * uv[i] * inv_nuK;
          const float sg = 1.f / (1.f + expf(-P.kappa * (xk - theta)));
          const float gg = (x < P.W) ? P.kappa * sg * (1.f - sg) * gv[i] : 0.f;
          acc += (double)xk * (double)gg;
          acc2 += (double)gg;
          P.xbar[po] = gg;
          xm = fmaxf(xm, fabsf(gg));
        } else {
          acc += (double)gv[i] * (double)fv[i] * (double)uv[i];
          P.xbar[po] = gv[i];
          xm = fmaxf(xm, fabsf(gv[i]));
        }
        P.Fbar[po] = 0.f;
      }
    }
  }
  if (P.xbmax) {
    const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(xm));
    if ((threadIdx.x & 31) == 0) atomicMax(P.xbmax + (long)b * 2 * kScal, m);
  }
  const double s = block_sum<kEwThreads>(acc, red);
  const double s2 = bin ? block_sum<kEwThreads>(acc2, red) : 0.0;
  const long nper = (long)P.T * P.gx;
  if (threadIdx.x == 0) {
    P.partials[(long)b * nper + (long)t * P.gx + blockIdx.x] = s;
    if (bin) P.partials[(long)(P.B + b) * nper + (long)t * P.gx + blockIdx.x] = s2;
  }
  if (!last_block_arrive(P.counter, gridDim.x * gridDim.y, &flag)) return;
  for (int bb = 0; bb < P.B; ++bb) {
    const double tot = block_sum_array<kEwThreads>(P.partials + (long)bb * nper, nper, 1, red);
    const double sg = bin ? block_sum_array<kEwThreads>(P.partials + (long)(P.B + bb) * nper, nper, 1, red) : 0.0;
    if (threadIdx.x == 0 && P.loc) {
      P.loc[2 * bb] = tot;
      P.loc[2 * bb + 1] = sg;
    } else if (threadIdx.x == 0) {
      const double nuK = P.tape_nu[(long)bb * P.K + (P.K - 1)];
      if (bin) {
        // c_K = <x_K, g - [x_K > 0] corr> = sum(x g) - theta sum(g); cn = c_K / nu_K
        const double* tb = P.tape_bin + ((long)bb * P.K + (P.K - 1)) * 2;
        P.sc[bb * kScal + SC_CN] = (tot - tb[0] * sg) / nuK;
        P.sc[bb * kScal + SC_CORR] = tb[1] > 0.0 ? sg / tb[1] : 0.0;
      } else {
        // c_K = <x_K, x_bar_K> = sum(g F u_{K-1}) / nu_K ; cn = c_K / nu_K
        P.sc[bb * kScal + SC_CN] = tot / (nuK * nuK);
        P.sc[bb * kScal + SC_CORR] = 0.0;
      }
      P.sc[bb * kScal + SC_INV_NU] = 1.0 / nuK;
      P.sc[bb * kScal + SC_INV_NU_PREV] = (P.K >= 2) ? 1.0 / P.tape_nu[(long)bb * P.K + (P.K - 2)] : 0.0;
    }
  }
  if (threadIdx.x == 0) *P.counter = 0u;
}

// Time slabs: the bwd_init finalize from the allreduced sums glob[B][2] = (sum(x g) or
// sum(g F u_{K-1}), sum(g) of a binarised iteration K).
struct BwdInitFinParams {
  const double* glob;
  double* sc;
  const double* tape_nu;
  const double* tape_bin;
  float kappa;
  int B, K;
};
__global__ void bwd_init_finalize_kernel(const __grid_constant__ BwdInitFinParams P) {
  const int bb = blockIdx.x * blockDim.x + threadIdx.x;
  if (bb >= P.B) return;
  const double tot = P.glob[2 * bb], sg = P.glob[2 * bb + 1];
  const double nuK = P.tape_nu[(long)bb * P.K + (P.K - 1)];
  if (P.kappa > 0.f) {
    const double* tb = P.tape_bin + ((long)bb * P.K + (P.K - 1)) * 2;
    P.sc[bb * kScal + SC_CN] = (tot - tb[0] * sg) / nuK;
    P.sc[bb * kScal + SC_CORR] = tb[1] > 0.0 ? sg / tb[1] : 0.0;
  } else {
    P.sc[bb * kScal + SC_CN] = tot / (nuK * nuK);
    P.sc[bb * kScal + SC_CORR] = 0.0;
  }
  P.sc[bb * kScal + SC_INV_NU] = 1.0 / nuK;
  P.sc[bb * kScal + SC_INV_NU_PREV] = (P.K >= 2) ? 1.0 / P.tape_nu[(long)bb * P.K + (P.K - 2)] : 0.0;
}

// Time slabs, backward halos: the temporal pass of backward step k at a slab boundary needs
// the neighbour's F y_bar_k on r_t frames (tpass TP_BWD reads halos pre-multiplied).  This
// kernel forms F y_bar_k = F (x_bar_k - [F u_{k-1} > 0] corr - F u_{k-1} cn) inv_nu on the
// first and last RT frames of every volume into send_lo / send_hi [B][RT][H][Wp].
struct BwdHaloParams {
  const float* xbar;
  const float* F;
  const float* u1;
  const double* sc;
  float* send_lo;
  float* send_hi;
  long frame;   // H * Wp
  int T, RT;
};
__global__ void __launch_bounds__(kEwThreads) bwd_halo_kernel(const __grid_constant__ BwdHaloParams P) {
  const int b = blockIdx.z, j = blockIdx.y;   // j < RT: first frames (send_lo), else last frames (send_hi)
  const bool hi = j >= P.RT;
  const int t = hi ? P.T - 2 * P.RT + j : j;
  const float cn = (float)P.sc[b * kScal + SC_CN], inv_nu = (float)P.sc[b * kScal + SC_INV_NU];
  const float corr = (float)P.sc[b * kScal + SC_CORR];
  const long src = ((long)b * P.T + t) * P.frame;
  float* dst = (hi ? P.send_hi : P.send_lo) + ((long)b * P.RT + (hi ? j - P.RT : j)) * P.frame;
  for (long e = (long)blockIdx.x * kEwThreads + threadIdx.x; e < P.frame; e += (long)gridDim.x * kEwThreads) {
    const float f = P.F[src + e], fu = f * P.u1[src + e];
    dst[e] = f * ((P.xbar[src + e] - (fu > 0.f ? corr : 0.f) - fu * cn) * inv_nu);
  }
}

// ------------------------------------------------------------------ backward contraction dw, db
struct ContractParams {
  const float* ch;      // dense [B][C][T][H][W]
  const float* Fbar;    // pitched
  const float* xbar0;   // pitched x_bar_0 (added when x_0 = F) or null
  double* partials;     // [G][C+1]
  double* out;          // [C+1] : dw_0..dw_{C-1}, db
  unsigned* counter;
  int B, C, T, H, W, Wp, act;
  int in_T, in_t0;      // channel buffer frames per volume and this slab's first frame in it
  float bias;
  float w[kMaxC];
};

// grid (gx, B*T), row-parallel; partials [(bt * gx + bx)][CMAX + 1]
template <int CMAX>
__global__ void __launch_bounds__(kEwThreads) contract_kernel(const __grid_constant__ ContractParams P) {
  __shared__ double red[kEwThreads / 32];
  __shared__ int flag;
  double acc[CMAX + 1];
#pragma unroll
  for (int c = 0; c <= CMAX; ++c) acc[c] = 0.0;
  const int bt = blockIdx.y;
  const int b = bt / P.T, t = bt - b * P.T;
  const long HW = (long)P.H * P.W, vol = (long)P.in_T * HW, HWp = (long)P.H * P.Wp;
  const float* chf = P.ch + (long)b * P.C * vol + (long)(P.in_t0 + t) * HW;
  for (int y = blockIdx.x; y < P.H; y += gridDim.x) {
#pragma unroll 2
    for (int x = threadIdx.x; x < P.W; x += kEwThreads) {
      const long po = (long)bt * HWp + (long)y * P.Wp + x;
      const long d = (long)y * P.W + x;
      float fb = __ldcs(P.Fbar + po);
      if (P.xbar0) fb += __ldcs(P.xbar0 + po);
      float cv[CMAX];
      float z = P.bias;
#pragma unroll
      for (int c = 0; c < CMAX; ++c) {
        cv[c] = (c < P.C) ? __ldcs(chf + (long)c * vol + d) : 0.f;
        z = fmaf(P.w[c], cv[c], z);  // w[c] == 0 for c >= C (host zero-fills)
      }
      float dphi = 1.f;
      if (P.act == 1) {
        const float sg = 1.f / (1.f + expf(-z));
        dphi = sg * (1.f - sg);
      }
      const double zb = (double)fb * (double)dphi;
#pragma unroll
      for (int c = 0; c < CMAX; ++c) acc[c] += zb * (double)cv[c];
      acc[CMAX] += zb;
    }
  }
  const long slot = (long)bt * gridDim.x + blockIdx.x;
#pragma unroll
  for (int c = 0; c <= CMAX; ++c) {
    const double s = block_sum<kEwThreads>(acc[c], red);
    if (threadIdx.x == 0) P.partials[slot * (CMAX + 1) + c] = s;
  }
  if (!last_block_arrive(P.counter, gridDim.x * gridDim.y, &flag)) return;
  const long nslot = (long)gridDim.x * gridDim.y;
  for (int c = 0; c <= CMAX; ++c) {
    const double tot = block_sum_array<kEwThreads>(P.partials + c, nslot, CMAX + 1, red);
    if (threadIdx.x == 0) {
      if (c < P.C) P.out[c] = tot;
      if (c == CMAX) P.out[P.C] = tot;
    }
  }
  if (threadIdx.x == 0) *P.counter = 0u;
}

}  // namespace sfseg
