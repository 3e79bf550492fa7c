// Full SFSeg / SFSeg++ operator: the general power
// iteration of Eq.7 / Eq.10 with a unary map S
// (exponent p), a pairwise map F and the Taylor bracket of Eq.2:
//
//   X_crt = S^p [ (alpha^-1 - F^2) G*(S^p X) - G*(F^2 S^p X) + 2 F G*(F S^p X) ]
//
// per iteration: one stacked temporal pass (tpass3_kernel: inputs a, F^2 a, F a with
// a = S^p X carried as the stored iterate and the normaliser folded in; a and F read
// once), three spatial passes (spass, plain mode: u = G_s v), then this file's epilogue
// combining the three filtered volumes per voxel (+ norm partials).  Eq.9 gives
// S and F (combine_full_kernel); x_0 = S (Alg.1 line 3) or a user x0.
#pragma once
#include "common.cuh"
#include "misc.cuh"
#include "spass.cuh"

namespace sfseg {

struct CombineFullParams {
  const float* s_ch;    // dense [B][Cs][T][H][W] (unary channels)
  const float* f_ch;    // dense [B][Cf][T][H][W] (pairwise channels)
  const float* x0;      // dense [B][T][H][W] or null (x_0 = S)
  float* U;             // pitched: S^p
  float* F;             // pitched: pairwise map
  float* a0;            // pitched: U * x_0
  double* sc;
  double* partials;     // [B][T*gx]
  unsigned* counter;
  unsigned* err;
  unsigned* amax;       // tcgen05 plain passes: max |a_0| (float bits, stride 2 kScal words) or null
  unsigned* fmax;       // ... and max |F| per volume
  int B, Cs, Cf, T, H, W, Wp, act_s, act_f, gx;
  float bs, bf, p;
  float ws[kMaxC];
  float wf[kMaxC];
};

// Eq.9 for both maps, U = S^p (reading A19: 0^p = 0; S < 0 gives NaN -> NONFINITE),
// a_0 = U x_0, ||x_0||.  Row-parallel like combine_kernel; grid (gx, B*T).
__global__ void __launch_bounds__(kEwThreads) combine_full_kernel(const __grid_constant__ CombineFullParams P) {
  __shared__ double red[kEwThreads / 32];
  __shared__ int flag;
  const int bt = blockIdx.y;
  const int b = bt / P.T, t = bt - b * P.T;
  const long HWp = (long)P.H * P.Wp, HW = (long)P.H * P.W;
  const long vol = (long)P.T * HW;
  const float* sf = P.s_ch + (long)b * P.Cs * vol + (long)t * HW;
  const float* ff = P.f_ch + (long)b * P.Cf * vol + (long)t * HW;
  const long dbase = (long)b * vol + (long)t * HW;
  double acc = 0.0;
  float am = 0.f, fm = 0.f;
  for (int y = blockIdx.x; y < P.H; y += P.gx) {
    for (int x = threadIdx.x; x < P.Wp; x += kEwThreads) {
      const long po = (long)bt * HWp + (long)y * P.Wp + x;
      float u = 0.f, f = 0.f, a = 0.f;
      if (x < P.W) {
        const long d = (long)y * P.W + x;
        float zs = P.bs, zf = P.bf;
        for (int c = 0; c < P.Cs; ++c) zs = fmaf(P.ws[c], __ldg(sf + (long)c * vol + d), zs);
        for (int c = 0; c < P.Cf; ++c) zf = fmaf(P.wf[c], __ldg(ff + (long)c * vol + d), zf);
        const float s = (P.act_s == 1) ? 1.f / (1.f + expf(-zs)) : zs;
        f = (P.act_f == 1) ? 1.f / (1.f + expf(-zf)) : zf;
        u = (P.p == 1.f) ? s : ((s == 0.f) ? 0.f : powf(s, P.p));
        const float xv = P.x0 ? __ldg(P.x0 + dbase + d) : s;
        a = u * xv;
        acc += (double)xv * (double)xv;
      }
      P.U[po] = u;
      P.F[po] = f;
      P.a0[po] = a;
      am = fmaxf(am, fabsf(a));
      fm = fmaxf(fm, fabsf(f));
    }
  }
  if (P.amax) {   // order-free maxima, one atomic per warp
    const unsigned ma = __reduce_max_sync(0xffffffffu, __float_as_uint(am));
    const unsigned mf = __reduce_max_sync(0xffffffffu, __float_as_uint(fm));
    if ((threadIdx.x & 31) == 0) {
      atomicMax(P.amax + (long)b * 2 * kScal, ma);
      atomicMax(P.fmax + (long)b * 2 * kScal, mf);
    }
  }
  const double s = block_sum<kEwThreads>(acc, red);
  const long nper = (long)P.T * P.gx;
  if (threadIdx.x == 0) P.partials[(long)b * nper + (long)t * P.gx + blockIdx.x] = s;
  if (!last_block_arrive(P.counter, gridDim.x * gridDim.y, &flag)) return;
  for (int bb = 0; bb < P.B; ++bb) {
    const double tot = block_sum_array<kEwThreads>(P.partials + (long)bb * nper, nper, 1, red);
    if (threadIdx.x == 0) {
      const double xn = sqrt(tot);
      P.sc[bb * kScal + SC_XNORM] = xn;
      P.sc[bb * kScal + SC_S] = 1.0;
      flag_norm(P.err, xn);
    }
  }
  if (threadIdx.x == 0) *P.counter = 0u;
}

struct FullEpiParams {
  const float* ua;      // pitched G * (s a)
  const float* ub;      // pitched G * (s F^2 a)
  const float* uc;      // pitched G * (s F a)
  const float* U;       // S^p
  const float* F;
  float* out;           // a_k = U y_k (or y_k when last)
  double* sc;
  double* partials;
  unsigned* counter;
  unsigned* err;
  double* stats;
  unsigned* amax;       // tcgen05 plain passes: max |a_k| per volume (the next stacked temporal pass's range)
  int B, T, H, Wp, W, K, k, last, gx;
  float inv_alpha;
};

// y_k = U [ (alpha^-1 - F^2) ua - ub + 2 F uc ]  (Eq.7), a_k = U y_k, ||y_k||^2 partials,
// last block: fwd_finalize (nu_k, gain; the Rayleigh slot is 0 on this path).
__global__ void __launch_bounds__(kEwThreads) full_epilogue_kernel(const __grid_constant__ FullEpiParams P) {
  __shared__ double red[kEwThreads / 32];
  __shared__ int flag;
  const int bt = blockIdx.y;
  const int b = bt / P.T, t = bt - b * P.T;
  const long HWp = (long)P.H * P.Wp;
  const long W4 = P.Wp / 4;
  double acc = 0.0;
  float am = 0.f;
  for (int y = blockIdx.x; y < P.H; y += P.gx) {
    for (long x4 = threadIdx.x; x4 < W4; x4 += kEwThreads) {
      const long po = (long)bt * HWp + (long)y * P.Wp + 4 * x4;
      const float4 a = __ldcs(reinterpret_cast<const float4*>(P.ua + po));
      const float4 bb = __ldcs(reinterpret_cast<const float4*>(P.ub + po));
      const float4 c = __ldcs(reinterpret_cast<const float4*>(P.uc + po));
      const float4 u = *reinterpret_cast<const float4*>(P.U + po);
      const float4 f = *reinterpret_cast<const float4*>(P.F + po);
      float yv[4], o[4];
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {bb.x, bb.y, bb.z, bb.w}, cv[4] = {c.x, c.y, c.z, c.w};
      const float uv[4] = {u.x, u.y, u.z, u.w}, fv[4] = {f.x, f.y, f.z, f.w};
      float s2 = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool in = 4 * x4 + i < P.W;
        const float fi = fv[i];
        const float val = (P.inv_alpha - fi * fi) * av[i] - bv[i] + 2.f * fi * cv[i];
        yv[i] = in ? uv[i] * val : 0.f;
        o[i] = P.last ? yv[i] : uv[i] * yv[i];
        s2 = fmaf(yv[i], yv[i], s2);
      }
      *reinterpret_cast<float4*>(P.out + po) = make_float4(o[0], o[1], o[2], o[3]);
      am = fmaxf(am, fmaxf(fmaxf(fabsf(o[0]), fabsf(o[1])), fmaxf(fabsf(o[2]), fabsf(o[3]))));
      acc += (double)s2;
    }
  }
  if (P.amax) {
    const unsigned ma = __reduce_max_sync(0xffffffffu, __float_as_uint(am));
    if ((threadIdx.x & 31) == 0) atomicMax(P.amax + (long)b * 2 * kScal, ma);
  }
  const double s = block_sum<kEwThreads>(acc, red);
  const long nper = (long)P.T * P.gx;
  if (threadIdx.x == 0) P.partials[(long)b * nper + (long)t * P.gx + blockIdx.x] = s;
  if (!last_block_arrive(P.counter, gridDim.x * gridDim.y, &flag)) return;
  for (int v = 0; v < P.B; ++v) {
    const double tot = block_sum_array<kEwThreads>(P.partials + (long)v * nper, nper, 1, red);
    if (threadIdx.x == 0) fwd_finalize(P.sc + v * kScal, P.stats, nullptr, P.err, P.K, P.k, false, v, tot, 0.0);
  }
  if (threadIdx.x == 0) *P.counter = 0u;
}

// ------------------------------------------------------------------ soft-binarisation (row f2)
// Alg.1 STEP 3, reading A21: x_k <- sigma(kappa (y_k/nu_k - theta)),
// theta = mean of the positive entries of y_k/nu_k.  Two streaming passes after the
// iteration's norm finalize: pos_stats (sum and count of the positive y, fp64 fixed
// order) and binarize (the sigmoid, the next stored iterate a = U x or the dense
// output, and ||x|| for the next gain).
struct BinParams {
  const float* y;       // pitched y_k (unnormalised)
  const float* U;       // pitched S^p (multiplier of the next stored iterate) or null
  float* a;             // pitched: U * x_k (next iterate), or null
  float* x_dense;       // dense output (last iteration) or null
  double* sc;
  double* partials;     // [2][B][T*gx]
  unsigned* counter;
  unsigned* err;
  int B, T, H, W, Wp, gx;
  float kappa;
  double* tape_bin;     // hot-path tape [B][K][2] (theta_k in x units, n_pos) or null
  int K, k;             // iteration recorded in tape_bin
};

__global__ void __launch_bounds__(kEwThreads) pos_stats_kernel(const __grid_constant__ BinParams P) {
  __shared__ double red[kEwThreads / 32];
  __shared__ int flag;
  const int bt = blockIdx.y;
  const int b = bt / P.T, t = bt - b * P.T;
  const long HWp = (long)P.H * P.Wp;
  double s = 0.0, n = 0.0;
  for (int y = blockIdx.x; y < P.H; y += P.gx)
    for (int x = threadIdx.x; x < P.W; x += kEwThreads) {
      const float v = P.y[(long)bt * HWp + (long)y * P.Wp + x];
      if (v > 0.f) {
        s += (double)v;
        n += 1.0;
      }
    }
  const double ss = block_sum<kEwThreads>(s, red);
  const double nn = block_sum<kEwThreads>(n, red);
  const long nper = (long)P.T * P.gx;
  if (threadIdx.x == 0) {
    P.partials[(long)b * nper + (long)t * P.gx + blockIdx.x] = ss;
    P.partials[(long)(P.B + b) * nper + (long)t * P.gx + blockIdx.x] = nn;
  }
  if (!last_block_arrive(P.counter, gridDim.x * gridDim.y, &flag)) return;
  for (int v = 0; v < P.B; ++v) {
    const double tot = block_sum_array<kEwThreads>(P.partials + (long)v * nper, nper, 1, red);
    const double cnt = block_sum_array<kEwThreads>(P.partials + (long)(P.B + v) * nper, nper, 1, red);
    if (threadIdx.x == 0) {
      P.sc[v * kScal + SC_THETA] = cnt > 0.0 ? tot / cnt : 0.0;
      if (P.tape_bin) {
        double* tb = P.tape_bin + ((long)v * P.K + (P.k - 1)) * 2;
        tb[0] = cnt > 0.0 ? tot / cnt / P.sc[v * kScal + SC_NU] : 0.0;
        tb[1] = cnt;
      }
    }
  }
  if (threadIdx.x == 0) *P.counter = 0u;
}

__global__ void __launch_bounds__(kEwThreads) binarize_kernel(const __grid_constant__ BinParams P) {
  __shared__ double red[kEwThreads / 32];
  __shared__ int flag;
  const int bt = blockIdx.y;
  const int b = bt / P.T, t = bt - b * P.T;
  const long HWp = (long)P.H * P.Wp, HW = (long)P.H * P.W;
  const double nu = P.sc[b * kScal + SC_NU];
  const float inv_nu = (float)(1.0 / nu);
  const float theta = (float)(P.sc[b * kScal + SC_THETA] / nu);
  double acc = 0.0;
  for (int y = blockIdx.x; y < P.H; y += P.gx)
    for (int x = threadIdx.x; x < P.Wp; x += kEwThreads) {
      const long po = (long)bt * HWp + (long)y * P.Wp + x;
      float xv = 0.f;
      if (x < P.W) {
        xv = 1.f / (1.f + expf(-P.kappa * (P.y[po] * inv_nu - theta)));
        acc += (double)xv * (double)xv;
        if (P.x_dense) P.x_dense[(long)bt * HW + (long)y * P.W + x] = xv;
      }
      if (P.a) P.a[po] = P.U ? P.U[po] * xv : xv;
    }
  const double s = block_sum<kEwThreads>(acc, red);
  const long nper = (long)P.T * P.gx;
  if (threadIdx.x == 0) P.partials[(long)b * nper + (long)t * P.gx + blockIdx.x] = s;
  if (!last_block_arrive(P.counter, gridDim.x * gridDim.y, &flag)) return;
  for (int v = 0; v < P.B; ++v) {
    const double tot = block_sum_array<kEwThreads>(P.partials + (long)v * nper, nper, 1, red);
    if (threadIdx.x == 0) {
      P.sc[v * kScal + SC_XNORM] = sqrt(tot);  // ||x_k|| for the next gain
      P.sc[v * kScal + SC_S] = 1.0;            // x_k is the iterate itself (no pending normaliser)
    }
  }
  if (threadIdx.x == 0) *P.counter = 0u;
}

}  // namespace sfseg
