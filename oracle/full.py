"""Full SFSeg / SFSeg++ operator -- TEST INFRASTRUCTURE ONLY.

The hot path (sfseg_oracle.py) is the unary-only special case of the paper's
power iteration.  This module transcribes the general step: the unary map S
(exponent p) and the pairwise map F with the first-order Taylor bracket of
Eq.2, in the three-convolution form of Eq.7 / Eq.10
(P:196-203):

    X_crt = S^p (alpha^-1 1 - F^2) G*(S^p X)  -  S^p G*(F^2 S^p X)
            + 2 S^p F G*(F S^p X)
    X_{k+1} = X_crt / ||X_crt||_2                                   (Eq.8 / Eq.11)

with the multi-channel combine of Eq.9 for S_m and F_m, x_0 = S_m
(Alg.1 line 3, "X_m <- S_m").  Eq.7 is Eq.6 divided by alpha (
the overall scale is removed by the normalisation).  Readings:
A18 -- no clamping: Eq.7 is computed as printed; with S, F in [0, 1] and
alpha <= 1 every bracket alpha^-1 - (f_i - f_j)^2 is >= 0 so M is
non-negative (Perron-Frobenius); SPEC's clamp-at-0 is not
applied.  A19 -- S^p with p > 0 on S >= 0 (0^p = 0).
Shares no code with the CUDA path; reuses only the oracle's own
gaussian_taps / combine / gaussian_filter (pinned separately).
"""
from __future__ import annotations

import math

import numpy as np

from .sfseg_oracle import DegenerateError, binarize_kappa, combine, gaussian_filter, soft_binarize


def full_step(U: np.ndarray, F: np.ndarray, alpha: float, x: np.ndarray, g_t, g_y, g_x) -> np.ndarray:
    """One unnormalised Eq.7 step for one volume; U = S^p (already raised), F the pairwise map."""
    U = np.asarray(U, np.float64)
    F = np.asarray(F, np.float64)
    a = U * np.asarray(x, np.float64)                       # S^p . X
    t1 = (1.0 / alpha - F * F) * gaussian_filter(a, g_t, g_y, g_x)
    t2 = gaussian_filter(F * F * a, g_t, g_y, g_x)
    t3 = 2.0 * F * gaussian_filter(F * a, g_t, g_y, g_x)
    return U * (t1 - t2 + t3)


def combine_full(s_ch, ws, bs, act_s, f_ch, wf, bf, act_f, p: float):
    """Eq.9 for both maps; returns (S_m, U = S_m^p, F_m) float64 [B][T][H][W]."""
    S, _ = combine(s_ch, ws, bs, act_s)
    F, _ = combine(f_ch, wf, bf, act_f)
    if np.any(S < 0):
        raise ValueError("S^p needs S >= 0 (reading A19)")
    U = np.power(S, float(p))
    return S, U, F


def power_iterate_full(S: np.ndarray, U: np.ndarray, F: np.ndarray, alpha: float, g_t, g_s, K: int, x0=None,
                       binarize=None):
    """K iterations of Eq.7 + Eq.8 per volume from x_0 = S (Alg.1 line 3) or x0.

    binarize = (n_cont, kappa0, growth): Alg.1 STEP 3 -- after the normalisation of
    iteration k > n_cont the iterate is soft-binarised with kappa_k = kappa0 *
    growth^(k - n_cont - 1) (reading A21, SPEC's geometric schedule); the result is
    then the next iterate as is (not renormalised) and, after the last iteration,
    the output (values in (0, 1)).
    Returns (x_K [B][T][H][W], stats) with stats["nu"][b, k] = ||X_crt_k||,
    stats["gain"][b, k] = nu_k / ||x_{k-1}||, stats["rho"][b, k] = Rayleigh quotient.
    """
    S, U, F = (np.asarray(a, np.float64) for a in (S, U, F))
    g_y = np.asarray(g_s, np.float64)
    B = S.shape[0]
    nus, gains, rhos = np.zeros((B, K)), np.zeros((B, K)), np.zeros((B, K))
    xs = np.empty_like(S)
    for b in range(B):
        x = S[b].copy() if x0 is None else np.asarray(x0[b], np.float64).copy()
        for k in range(K):
            y = full_step(U[b], F[b], alpha, x, g_t, g_y, g_y)
            xx = float(np.sum(x * x))
            nu = math.sqrt(float(np.sum(y * y)))
            if nu == 0.0 or xx == 0.0:
                raise DegenerateError(f"zero norm at iteration {k + 1}, volume {b}")
            nus[b, k] = nu
            gains[b, k] = nu / math.sqrt(xx)
            rhos[b, k] = float(np.sum(x * y)) / xx
            x = y / nu
            kap = binarize_kappa(k + 1, binarize)
            if kap > 0.0:
                x = soft_binarize(x, kap)
        xs[b] = x
    return xs, {"nu": nus, "gain": gains, "rho": rhos}
