"""Learning loop -- TEST INFRASTRUCTURE ONLY.

PAPER.md:210-232 (§3.4): the channel weights w (and bias b) of Eq.9 are learned
by minimising a loss of the final segmentation, with the gradient propagated
"through the full spectral algorithm", using AdamW (Eq.13) --
"an AdamW optimizer with AMSGrad"; "We make SFSeg++ trainable by using a
soft-binarization between iterations".  Readings:
A13 -- BASELINE c3's loss: the mean squared error between x_K and the unit-normalised
clean mask; A24 -- the paper's Focal-Dice loss (Eq.12) on the soft-binarised
output, with the soft Dice overlap per training frame and gamma = 0.75;
A22 -- AdamW with AMSGrad in PyTorch's form (decoupled weight decay w <- w - lr*wd*w,
bias-corrected moments, running max of the second moment).
"""
from __future__ import annotations

import math

import numpy as np

from .sfseg_oracle import combine, power_iterate, power_iterate_backward


def mse_loss_grad(x: np.ndarray, mask: np.ndarray):
    """Reading A13: L = mean (x_K - m_hat)^2, m_hat = m / ||m|| (per volume); returns (L, dL/dx)."""
    x = np.asarray(x, np.float64)
    m = np.asarray(mask, np.float64)
    mh = np.empty_like(m)
    for b in range(m.shape[0]):
        n = np.linalg.norm(m[b])
        mh[b] = m[b] / n if n > 0 else m[b]
    d = x - mh
    return float(np.mean(d * d)), 2.0 * d / x.size


def focal_dice_loss_grad(x: np.ndarray, mask: np.ndarray, gamma: float = 0.75):
    """Eq.12, reading A24:  J = sum_i (1 - D_i)^gamma over the training frames i
    (every (volume, frame) pair), with the soft Dice overlap of the prediction X_m (the
    soft-binarised output, values in (0, 1)) and the ground truth X_t:
        D_i = 2 sum(x t) / (sum(x) + sum(t))            (the printed "2 (X_m cap X_t) / (X_m cup X_t)")
    and gamma = 0.75 ("Focal-Dice loss ... with 0.75 coefficient").  A frame with
    sum(x) + sum(t) == 0 contributes 0.  Returns (J, dJ/dx)."""
    x = np.asarray(x, np.float64)
    t = np.asarray(mask, np.float64)
    B, T = x.shape[:2]
    J = 0.0
    g = np.zeros_like(x)
    for b in range(B):
        for f in range(T):
            xi, ti = x[b, f], t[b, f]
            inter = float(np.sum(xi * ti))
            den = float(np.sum(xi)) + float(np.sum(ti))
            if den == 0.0:
                continue
            D = 2.0 * inter / den
            J += (1.0 - D) ** gamma
            # dD/dx = 2 (t den - inter) / den^2 ;  dJ/dx = -gamma (1 - D)^(gamma - 1) dD/dx
            if D < 1.0:
                g[b, f] = -gamma * (1.0 - D) ** (gamma - 1.0) * 2.0 * (ti * den - inter) / (den * den)
    return J, g


class AdamW:
    """Eq.13 with AMSGrad, PyTorch's update order (reading A22)."""

    def __init__(self, n: int, lr: float, betas=(0.9, 0.999), eps: float = 1e-8, weight_decay: float = 0.0,
                 amsgrad: bool = True):
        self.lr, self.b1, self.b2, self.eps, self.wd, self.ams = lr, betas[0], betas[1], eps, weight_decay, amsgrad
        self.m = np.zeros(n)
        self.v = np.zeros(n)
        self.vmax = np.zeros(n)
        self.t = 0

    def step(self, params: np.ndarray, grad: np.ndarray) -> np.ndarray:
        self.t += 1
        p = np.asarray(params, np.float64) * (1.0 - self.lr * self.wd)   # decoupled weight decay
        g = np.asarray(grad, np.float64)
        self.m = self.b1 * self.m + (1.0 - self.b1) * g
        self.v = self.b2 * self.v + (1.0 - self.b2) * g * g
        bc1 = 1.0 - self.b1 ** self.t
        bc2 = 1.0 - self.b2 ** self.t
        if self.ams:
            self.vmax = np.maximum(self.vmax, self.v)
            denom = np.sqrt(self.vmax) / math.sqrt(bc2) + self.eps
        else:
            denom = np.sqrt(self.v) / math.sqrt(bc2) + self.eps
        return p - (self.lr / bc1) * self.m / denom


def train(ch, mask, w0, b0: float, act: int, g_t, g_s, K: int, steps: int, lr: float, weight_decay: float = 0.0,
          loss: str = "mse", binarize=None, gamma: float = 0.75):
    """`steps` AdamW steps on (w, b) of Eq.9; loss "mse" (A13, on x_K) or "focal_dice" (Eq.12, A24,
    on the output of the binarised iteration ``binarize``); returns (w, b, losses)."""
    w = np.asarray(w0, np.float64).copy()
    b = float(b0)
    opt = AdamW(w.size + 1, lr, weight_decay=weight_decay)
    losses = []
    for _ in range(steps):
        F, _ = combine(ch, w, b, act)
        x, _ = power_iterate(F, g_t, g_s, K, binarize=binarize)
        L, g = mse_loss_grad(x, mask) if loss == "mse" else focal_dice_loss_grad(x, mask, gamma)
        losses.append(L)
        dw, db = power_iterate_backward(ch, w, b, act, g_t, g_s, K, g, binarize=binarize)
        pb = opt.step(np.concatenate([w, [b]]), np.concatenate([dw, [db]]))
        w, b = pb[:-1], float(pb[-1])
    return w, b, losses
