"""Explicit dense adjacency matrix for tiny volumes (TEST INFRASTRUCTURE ONLY).

M_ij = s_i s_j [1 - alpha (f_i - f_j)^2] G_ij   (Eq.2) with the
north-star choices p = 1, constant pairwise map (bracket == 1), so
M_ij = F_i F_j G_ij, and G_ij = g_t[dt] g_y[dy] g_x[dx] for |d| <= r on each
axis, 0 otherwise (local connections only, "M is sparse").

Built element by element from voxel coordinates -- it shares nothing with the
stencil code in sfseg_oracle.py except ``gaussian_taps`` (the 1D weights, which
are pinned separately against SPEC S:118).  Used by tests to pin the oracle's
iteration against Eq.4, dense eigh (Eq.3) and
brute-force power iteration.
"""
from __future__ import annotations

import numpy as np


def dense_G(T: int, H: int, W: int, g_t, g_y, g_x) -> np.ndarray:
    """N x N matrix G_ij for an N = T*H*W volume, flattened C-order (t, y, x)."""
    g_t, g_y, g_x = (np.asarray(g, np.float64) for g in (g_t, g_y, g_x))
    rt, ry, rx = (len(g_t) - 1) // 2, (len(g_y) - 1) // 2, (len(g_x) - 1) // 2
    t, y, x = np.meshgrid(np.arange(T), np.arange(H), np.arange(W), indexing="ij")
    t, y, x = t.ravel(), y.ravel(), x.ravel()
    dt = t[:, None] - t[None, :]
    dy = y[:, None] - y[None, :]
    dx = x[:, None] - x[None, :]
    inside = (np.abs(dt) <= rt) & (np.abs(dy) <= ry) & (np.abs(dx) <= rx)
    G = np.zeros(dt.shape, dtype=np.float64)
    G[inside] = (g_t[dt[inside] + rt] * g_y[dy[inside] + ry] * g_x[dx[inside] + rx])
    return G


def dense_M(F: np.ndarray, g_t, g_y, g_x) -> np.ndarray:
    """M = diag(F) G diag(F) for one volume F [T][H][W]."""
    F = np.asarray(F, np.float64)
    T, H, W = F.shape
    G = dense_G(T, H, W, g_t, g_y, g_x)
    f = F.ravel()
    return f[:, None] * G * f[None, :]


def dense_M_taylor(S: np.ndarray, F: np.ndarray, p: float, alpha: float, g_t, g_y, g_x) -> np.ndarray:
    """Eq.2 built entry by entry, divided by alpha (the scale of Eq.7):
    M_ij = s_i^p s_j^p [alpha^-1 - (f_i - f_j)^2] G_ij  for one volume [T][H][W]."""
    S, F = np.asarray(S, np.float64), np.asarray(F, np.float64)
    T, H, W = S.shape
    G = dense_G(T, H, W, g_t, g_y, g_x)
    u = np.power(S.ravel(), float(p))
    f = F.ravel()
    bracket = 1.0 / alpha - (f[:, None] - f[None, :]) ** 2
    return u[:, None] * u[None, :] * bracket * G
