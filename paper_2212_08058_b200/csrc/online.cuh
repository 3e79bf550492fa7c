// Online / sub-window mode: the
// warm start of a window from the previous window's solution on the overlap
// frames, rescaled per volume to the L2 norm of F on those frames (reading A20).
// Two small streaming kernels; the windows themselves are ordinary solves.
#pragma once
#include "common.cuh"
#include "misc.cuh"

namespace sfseg {

struct OnlineParams {
  const float* xprev;   // dense [B][q][H][W] previous window solution
  const float* Fw;      // dense [B][q][H][W] F of the current window
  float* x0;            // dense [B][q][H][W] warm start (pre-filled with Fw)
  double* partials;     // [2][B][nov*gx]
  double* factor;       // [B]  (< 0: keep F)
  unsigned* counter;
  long HW;
  int B, q, nov, po, gx;  // overlap: current frames [0, nov) == previous frames [po, po + nov)
};

// grid (gx, B * nov): sums of squares of xprev and F over the overlap frames.
__global__ void __launch_bounds__(kEwThreads) online_norms_kernel(const __grid_constant__ OnlineParams P) {
  __shared__ double red[kEwThreads / 32];
  __shared__ int flag;
  const int b = blockIdx.y / P.nov, t = blockIdx.y % P.nov;
  const float* xp = P.xprev + ((long)b * P.q + P.po + t) * P.HW;
  const float* fw = P.Fw + ((long)b * P.q + t) * P.HW;
  double sx = 0.0, sf = 0.0;
  for (long e = (long)blockIdx.x * kEwThreads + threadIdx.x; e < P.HW; e += (long)P.gx * kEwThreads) {
    const double a = xp[e], c = fw[e];
    sx += a * a;
    sf += c * c;
  }
  const double tx = block_sum<kEwThreads>(sx, red);
  const double tf = block_sum<kEwThreads>(sf, red);
  const long nper = (long)P.nov * P.gx;
  if (threadIdx.x == 0) {
    P.partials[(long)b * nper + (long)t * P.gx + blockIdx.x] = tx;
    P.partials[(long)(P.B + b) * nper + (long)t * P.gx + blockIdx.x] = tf;
  }
  if (!last_block_arrive(P.counter, gridDim.x * gridDim.y, &flag)) return;
  for (int v = 0; v < P.B; ++v) {
    const double nx = block_sum_array<kEwThreads>(P.partials + (long)v * nper, nper, 1, red);
    const double nf = block_sum_array<kEwThreads>(P.partials + (long)(P.B + v) * nper, nper, 1, red);
    if (threadIdx.x == 0) P.factor[v] = nx > 0.0 ? sqrt(nf) / sqrt(nx) : -1.0;
  }
  if (threadIdx.x == 0) *P.counter = 0u;
}

// grid (gx, B * nov): x0[b, t] = factor_b * xprev[b, po + t] on the overlap frames.
__global__ void __launch_bounds__(kEwThreads) online_warm_kernel(const __grid_constant__ OnlineParams P) {
  const int b = blockIdx.y / P.nov, t = blockIdx.y % P.nov;
  const double f = P.factor[b];
  if (f < 0.0) return;  // previous solution zero on the overlap: keep the cold start F
  const float ff = (float)f;
  const float* xp = P.xprev + ((long)b * P.q + P.po + t) * P.HW;
  float* x0 = P.x0 + ((long)b * P.q + t) * P.HW;
  for (long e = (long)blockIdx.x * kEwThreads + threadIdx.x; e < P.HW; e += (long)P.gx * kEwThreads)
    x0[e] = ff * xp[e];
}

}  // namespace sfseg
