"""Online / sub-window mode -- TEST INFRASTRUCTURE ONLY.

PAPER.md:367-387 (§4.5, Fig. `offline_online` P:377-383): instead of the whole
video, the power iteration runs on smaller sub-windows of q frames that slide
over the video; "we initialize the current solution with the final solution over
the previous sub-window (for the frames that overlap)".
fixes the remaining choices used here:
  * windows start at 0, stride, 2*stride, ... while start + q < T; a last window
    [T - q, T) covers the tail (one window = the offline solve when q >= T);
  * inside a window: the offline iteration (K steps of Eq.4/7/8 on the window,
    zero padding at the window's temporal ends, normalisation per window);
  * per-frame output from the LAST window covering that frame.
Reading A20: the warm start takes the previous window's solution on
the overlap frames rescaled per volume so that its L2 norm equals that of F on
those frames (the eigenvector is unit-norm over a whole window while F -- the
cold start "X_m <- S_m" of Alg.1 line 3 -- is not), and F on the new frames.
"""
from __future__ import annotations

import math

import numpy as np

from .sfseg_oracle import power_iterate


def window_starts(T: int, q: int, stride: int):
    if q >= T:
        return [0]
    starts = []
    s = 0
    while s + q < T:
        starts.append(s)
        s += stride
    if not starts or starts[-1] + q < T:
        starts.append(T - q)
    return starts


def power_iterate_online(F: np.ndarray, g_t, g_s, K: int, q: int, stride: int):
    """F [B][T][H][W] (float64) -> x [B][T][H][W]: per-frame results of the sliding windows."""
    F = np.asarray(F, np.float64)
    B, T = F.shape[:2]
    out = np.zeros_like(F)
    prev = None  # (start, x_window)
    for s in window_starts(T, q, stride):
        e = min(T, s + q)
        Fw = F[:, s:e]
        x0 = Fw.copy()
        if prev is not None:
            ps, px = prev
            ov0, ov1 = s, min(e, ps + px.shape[1])
            if ov1 > ov0:
                for b in range(B):
                    xo = px[b, ov0 - ps:ov1 - ps]
                    fo = F[b, ov0:ov1]
                    nx, nf = math.sqrt(float(np.sum(xo * xo))), math.sqrt(float(np.sum(fo * fo)))
                    x0[b, :ov1 - ov0] = xo * (nf / nx) if nx > 0 else fo
        xw, _ = power_iterate(Fw, g_t, g_s, K, x0=x0)
        out[:, s:e] = xw
        prev = (s, xw)
    return out
