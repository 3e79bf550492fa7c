// Learning-loop kernels: the optimizer of Eq.13 and the
// Focal-Dice loss of Eq.12, on the device.
#pragma once
#include "common.cuh"

namespace sfseg {

// Eq.13:  w_t = w_{t-1} - eta_t (alpha m_hat_t / (sqrt(v_hat_t) + eps) + lambda w_{t-1})
// with alpha = 1, eta_t = lr, lambda = weight_decay; "AdamW optimizer with AMSGrad": the
// second moment in the denominator is the running maximum of v_t.  m_hat_t = m_t / (1 - beta1^t),
// v_hat_t = v_max,t / (1 - beta2^t) (reading A22).  One thread per parameter; state = [m | v | v_max].
struct AdamwParams {
  double* w;
  const double* grad;
  double* state;
  int n;
  double lr, beta1, beta2, eps, weight_decay;
  double c1, c2;  // 1 - beta1^t, 1 - beta2^t (host-computed)
  int amsgrad;
};

__global__ void adamw_kernel(const AdamwParams P) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  double* m = P.state;
  double* v = P.state + P.n;
  double* vmax = P.state + 2 * P.n;
  const double g = P.grad[i];
  const double mi = P.beta1 * m[i] + (1.0 - P.beta1) * g;     // first moment
  const double vi = P.beta2 * v[i] + (1.0 - P.beta2) * g * g; // second moment
  m[i] = mi;
  v[i] = vi;
  double vd = vi;
  if (P.amsgrad) {
    vd = fmax(vmax[i], vi);
    vmax[i] = vd;
  }
  const double m_hat = mi / P.c1;
  const double denom = sqrt(vd) / sqrt(P.c2) + P.eps;           // sqrt(v_hat) + eps
  const double w_prev = P.w[i];
  P.w[i] = w_prev - P.lr * (m_hat / denom + P.weight_decay * w_prev);
}

}  // namespace sfseg

namespace sfseg {

// Focal-Dice loss, Eq.12, reading A24: per training frame i (every
// (volume, frame) pair) the soft Dice overlap D_i = 2 sum(x t) / (sum(x) + sum(t)) of the
// prediction x (the soft-binarised output) and the binary ground truth t, and
//   J = sum_i (1 - D_i)^gamma      (gamma = 0.75),
//   dJ/dx = -gamma (1 - D_i)^(gamma - 1) * 2 (t sum_i - inter_i) / sum_i^2,  sum_i = sum(x) + sum(t).
// A frame with sum_i == 0 contributes nothing.  Two launches: per-(frame, block) fp64 partials
// of (inter, sum x, sum t); then every block folds its frame's partials in fixed order, writes
// its rows of dJ/dx, and the last block sums the per-frame losses in frame order.
constexpr int kFdGx = 16;

struct FocalDiceParams {
  const float* x;         // dense [B*T][H*W]
  const uint8_t* t;       // dense [B*T][H*W], 0 / 1
  float* grad;            // dense dJ/dx
  double* part;           // [3][BT][kFdGx]
  double* frame_loss;     // [BT]
  double* loss;           // device scalar J
  unsigned* counter;
  long HW;
  int BT;
  double gamma;
};

__global__ void __launch_bounds__(kEwThreads) focal_dice_sums_kernel(const __grid_constant__ FocalDiceParams P) {
  __shared__ double red[kEwThreads / 32];
  const int bt = blockIdx.y;
  const float* xf = P.x + (long)bt * P.HW;
  const uint8_t* tf = P.t + (long)bt * P.HW;
  double si = 0.0, sx = 0.0, st = 0.0;
  for (long e = (long)blockIdx.x * kEwThreads + threadIdx.x; e < P.HW; e += (long)gridDim.x * kEwThreads) {
    const double xv = (double)__ldg(xf + e);
    const double tv = tf[e] ? 1.0 : 0.0;
    si += xv * tv;
    sx += xv;
    st += tv;
  }
  si = block_sum<kEwThreads>(si, red);
  sx = block_sum<kEwThreads>(sx, red);
  st = block_sum<kEwThreads>(st, red);
  if (threadIdx.x == 0) {
    const long o = (long)bt * kFdGx + blockIdx.x;
    P.part[o] = si;
    P.part[(long)P.BT * kFdGx + o] = sx;
    P.part[2L * P.BT * kFdGx + o] = st;
  }
}

__global__ void __launch_bounds__(kEwThreads) focal_dice_grad_kernel(const __grid_constant__ FocalDiceParams P) {
  __shared__ double red[kEwThreads / 32];
  __shared__ int flag;
  const int bt = blockIdx.y;
  double inter = 0.0, sx = 0.0, st = 0.0;
  for (int i = 0; i < kFdGx; ++i) {  // fixed order: every block of the frame gets identical sums
    const long o = (long)bt * kFdGx + i;
    inter += P.part[o];
    sx += P.part[(long)P.BT * kFdGx + o];
    st += P.part[2L * P.BT * kFdGx + o];
  }
  const double den = sx + st;
  double c_t = 0.0, c_0 = 0.0;  // dJ/dx = c_t * t + c_0
  double lf = 0.0;
  if (den > 0.0) {
    const double D = 2.0 * inter / den;
    lf = pow(fmax(1.0 - D, 0.0), P.gamma);
    if (D < 1.0) {
      const double a = -P.gamma * pow(1.0 - D, P.gamma - 1.0) * 2.0 / (den * den);
      c_t = a * den;
      c_0 = -a * inter;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) P.frame_loss[bt] = lf;
  const float ct = (float)c_t, c0 = (float)c_0;
  const uint8_t* tf = P.t + (long)bt * P.HW;
  float* gf = P.grad + (long)bt * P.HW;
  for (long e = (long)blockIdx.x * kEwThreads + threadIdx.x; e < P.HW; e += (long)gridDim.x * kEwThreads)
    gf[e] = tf[e] ? ct + c0 : c0;
  if (!last_block_arrive(P.counter, gridDim.x * gridDim.y, &flag)) return;
  const double J = block_sum_array<kEwThreads>(P.frame_loss, P.BT, 1, red);
  if (threadIdx.x == 0) {
    *P.loss = J;
    *P.counter = 0u;
  }
}

}  // namespace sfseg
