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
