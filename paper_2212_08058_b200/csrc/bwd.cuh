// Backward step epilogue as a streaming kernel (Appendix A of SURVEY.md; the
// operations of spass_kernel<R, SP_BWD>'s epilogue, split from the spatial pass):
//   u = G_xy * v is produced by the tensor-core spatial pass in plain mode;
//   y_bar_k = (x_bar_k - F u_{k-1} cn) / nu_k,  x_{k-1} = F u_{k-2} / nu_{k-1}
//   (x_0 = F or the user's x_0 at k = 1),
//   F_bar += y_bar_k u_{k-1} + x_{k-1} u,  x_bar_{k-1} = F u,
//   c_{k-1} = <x_{k-1}, x_bar_{k-1}> (fixed-order fp64 partials; last block:
//   bwd_finalize -> the next step's cn, 1/nu, 1/nu_prev).
// Soft-binarised iteration k-1 (row f2, reading A21; kappa > 0): its output b_{k-1} =
//   sigma(kappa (x_{k-1} - theta)) is the input of iteration k, so F_bar uses b_{k-1}, and
//   the adjoint F u of b_{k-1} is pulled back through the sigmoid and the centre theta:
//   g = kappa sigma' (F u) is stored, with the partials sum(g) and sum(x g); the finalize
//   turns them into corr = sum(g)/n_pos and c_{k-1} = sum(x g) - theta sum(g), and the
//   next step forms x_bar_{k-1} = g - [x_{k-1} > 0] corr on the fly (tpass, this kernel).
// One float4 per thread per row step, row-parallel like the other streaming kernels.
#pragma once
#include "misc.cuh"
#include "spass.cuh"

namespace sfseg {

struct BwdEpiParams {
  const float* u;    // pitched G_xy * v
  const float* F;    // pitched
  float* xbar;       // pitched, in: x_bar_k, out: x_bar_{k-1}
  const float* u1;   // tape u_{k-1}
  const float* u2;   // tape u_{k-2} (k >= 2) or null
  const float* x0p;  // pitched user x_0 (k == 1) or null (x_0 = F)
  float* Fbar;       // pitched, accumulated
  double* sc;
  const double* tape_nu;
  double* partials;  // [B][T * gx]
  unsigned* counter;
  const double* tape_bin;  // [B][K][2] (theta in x units, n_pos) of the binarised iterations
  float kappa_prev;        // steepness of iteration k-1 (0: not binarised)
  double* loc;             // time slabs: per-volume local sums [B][2] (finalized after the allreduce)
  unsigned* xbmax;         // max |x_bar_{k-1}| per volume (the next tcgen05 backward step's range) or null
  int B, T, H, W, Wp, gx, K, k;
};

__global__ void __launch_bounds__(kEwThreads) bwd_epi_kernel(const __grid_constant__ BwdEpiParams P) {
  __shared__ double red[kEwThreads / 32];
  __shared__ int flag;
  const int bt = blockIdx.y;
  const int b = bt / P.T, t = bt - b * P.T;
  const long HWp = (long)P.H * P.Wp;
  const long W4 = P.Wp / 4;
  const float cn = (float)P.sc[b * kScal + SC_CN];
  const float inv_nu = (float)P.sc[b * kScal + SC_INV_NU];
  const float inv_nu_prev = (float)P.sc[b * kScal + SC_INV_NU_PREV];
  const float corr = (float)P.sc[b * kScal + SC_CORR];
  const float kap = P.kappa_prev;
  const bool bin = kap > 0.f;  // iteration k-1 >= 1 was soft-binarised (then u2 != null)
  const float theta = bin ? (float)P.tape_bin[((long)b * P.K + (P.k - 2)) * 2] : 0.f;
  double acc = 0.0, acc2 = 0.0;
  float xm = 0.f;
  for (int y = blockIdx.x; y < P.H; y += P.gx) {
    for (long x4 = threadIdx.x; x4 < W4; x4 += kEwThreads) {
      const long po = (long)bt * HWp + (long)y * P.Wp + 4 * x4;
      const float4 u4 = __ldcs(reinterpret_cast<const float4*>(P.u + po));
      const float4 f4 = *reinterpret_cast<const float4*>(P.F + po);
      const float4 xb4 = *reinterpret_cast<const float4*>(P.xbar + po);
      const float4 a4 = *reinterpret_cast<const float4*>(P.u1 + po);
      float4 d4 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (P.u2) d4 = *reinterpret_cast<const float4*>(P.u2 + po);
      else if (P.x0p) d4 = *reinterpret_cast<const float4*>(P.x0p + po);
      const float4 fb4 = *reinterpret_cast<const float4*>(P.Fbar + po);
      const float uv[4] = {u4.x, u4.y, u4.z, u4.w}, fv[4] = {f4.x, f4.y, f4.z, f4.w};
      const float xbv[4] = {xb4.x, xb4.y, xb4.z, xb4.w}, u1v[4] = {a4.x, a4.y, a4.z, a4.w};
      const float dv[4] = {d4.x, d4.y, d4.z, d4.w}, fbv[4] = {fb4.x, fb4.y, fb4.z, fb4.w};
      float xo[4], fo[4];
      float s = 0.f, s2 = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool in = 4 * x4 + i < P.W;
        const float f = in ? fv[i] : 0.f;
        const float uu = in ? uv[i] : 0.f;
        // x_{k-1}: the normalised y_{k-1} (from the tape), the user's x_0 or F
        const float xp = P.u2 ? f * dv[i] * inv_nu_prev : (P.x0p ? (in ? dv[i] : 0.f) : f);
        const float fu1 = f * u1v[i];
        const float yb = (xbv[i] - (fu1 > 0.f ? corr : 0.f) - fu1 * cn) * inv_nu;
        if (bin) {
          const float sg = in ? 1.f / (1.f + expf(-kap * (xp - theta))) : 0.f;  // b_{k-1}
          fo[i] = fbv[i] + (yb * u1v[i] + sg * uu);
          xo[i] = kap * sg * (1.f - sg) * (f * uu);  // g = kappa sigma' b_bar
          s = fmaf(xp, xo[i], s);
          s2 += xo[i];
        } else {
          fo[i] = fbv[i] + (yb * u1v[i] + xp * uu);
          xo[i] = f * uu;
          s = fmaf(xp, xo[i], s);
        }
      }
      *reinterpret_cast<float4*>(P.Fbar + po) = make_float4(fo[0], fo[1], fo[2], fo[3]);
      *reinterpret_cast<float4*>(P.xbar + po) = make_float4(xo[0], xo[1], xo[2], xo[3]);
      xm = fmaxf(xm, fmaxf(fmaxf(fabsf(xo[0]), fabsf(xo[1])), fmaxf(fabsf(xo[2]), fabsf(xo[3]))));
      acc += (double)s;
      acc2 += (double)s2;
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
  for (int v = 0; v < P.B; ++v) {
    const double tot = block_sum_array<kEwThreads>(P.partials + (long)v * nper, nper, 1, red);
    if (P.loc) {
      const double sg = bin ? block_sum_array<kEwThreads>(P.partials + (long)(P.B + v) * nper, nper, 1, red) : 0.0;
      if (threadIdx.x == 0) {
        P.loc[2 * v] = tot;
        P.loc[2 * v + 1] = sg;
      }
    } else if (bin) {
      const double sg = block_sum_array<kEwThreads>(P.partials + (long)(P.B + v) * nper, nper, 1, red);
      if (threadIdx.x == 0) {
        const double* tb = P.tape_bin + ((long)v * P.K + (P.k - 2)) * 2;
        bwd_finalize(P.sc + v * kScal, P.tape_nu, P.K, P.k, v, tot - tb[0] * sg, tb[1] > 0.0 ? sg / tb[1] : 0.0);
      }
    } else if (threadIdx.x == 0) {
      bwd_finalize(P.sc + v * kScal, P.tape_nu, P.K, P.k, v, tot);
    }
  }
  if (threadIdx.x == 0) *P.counter = 0u;
}

// Time slabs: the bwd_epi finalize from the allreduced sums glob[B][2].
struct BwdStepFinParams {
  const double* glob;
  double* sc;
  const double* tape_nu;
  const double* tape_bin;
  float kappa_prev;
  int B, K, k;
};
__global__ void bwd_step_finalize_kernel(const __grid_constant__ BwdStepFinParams P) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= P.B) return;
  const double tot = P.glob[2 * v], sg = P.glob[2 * v + 1];
  if (P.kappa_prev > 0.f) {
    const double* tb = P.tape_bin + ((long)v * P.K + (P.k - 2)) * 2;
    bwd_finalize(P.sc + v * kScal, P.tape_nu, P.K, P.k, v, tot - tb[0] * sg, tb[1] > 0.0 ? sg / tb[1] : 0.0);
  } else {
    bwd_finalize(P.sc + v * kScal, P.tape_nu, P.K, P.k, v, tot);
  }
}

}  // namespace sfseg
