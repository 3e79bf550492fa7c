"""Multi-process driver of the oracle for full-size volumes (TEST INFRASTRUCTURE).

Only ``tests/`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs use
it.  It adds NO arithmetic of its own: it calls ``sfseg_oracle.correlate_axis`` on
independent pieces of the volume, which is the same computation element by
element as the serial ``gaussian_filter`` (P:319's three 1D passes):

  * the T pass (axis 0) of a volume is independent per (y, x): split by rows H;
  * the H and W passes (axes 1, 2) are independent per frame: split by frames T.

Every output element is produced by the identical sequence of float64 operations
as in the serial oracle, so the results are bitwise equal to
``sfseg_oracle.gaussian_filter`` (checked by tests/test_oracle_parallel.py).  The
power iteration and its backward are the serial oracle's steps (Eq.4/7/8,
Appendix A of SURVEY.md) with the filter swapped for this one.
"""
from __future__ import annotations

import math
import multiprocessing as mp
import os
from multiprocessing import shared_memory

import numpy as np

from .sfseg_oracle import DegenerateError, combine, correlate_axis, ACT_IDENTITY

_W = {}  # worker-side attached arrays


def _attach(name_in, name_out, shape):
    a = shared_memory.SharedMemory(name=name_in)
    b = shared_memory.SharedMemory(name=name_out)
    _W["shm"] = (a, b)
    _W["vin"] = np.ndarray(shape, np.float64, buffer=a.buf)
    _W["vout"] = np.ndarray(shape, np.float64, buffer=b.buf)


def _t_chunk(args):
    h0, h1, g_t = args
    _W["vout"][:, h0:h1, :] = correlate_axis(_W["vin"][:, h0:h1, :], g_t, 0)


def _yx_chunk(args):
    t0, t1, g_y, g_x = args
    v = correlate_axis(_W["vin"][t0:t1], g_y, 1)
    _W["vin"][t0:t1] = correlate_axis(v, g_x, 2)  # in place: frames are independent


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class ParallelFilter:
    """G_3D (*) v for volumes of one shape [T][H][W] on ``procs`` worker processes."""

    def __init__(self, shape, procs: int | None = None):
        self.shape = tuple(int(s) for s in shape)
        self.procs = max(1, int(procs or host_cores()))
        n = int(np.prod(self.shape)) * 8
        self._a = shared_memory.SharedMemory(create=True, size=n)
        self._b = shared_memory.SharedMemory(create=True, size=n)
        self.vin = np.ndarray(self.shape, np.float64, buffer=self._a.buf)
        self.vout = np.ndarray(self.shape, np.float64, buffer=self._b.buf)
        ctx = mp.get_context("spawn")   # no fork of a multi-threaded (CUDA) parent
        self.pool = ctx.Pool(self.procs, initializer=_attach, initargs=(self._a.name, self._b.name, self.shape))

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()
            self.pool = None
            del self.vin, self.vout
            self._a.close(); self._a.unlink()
            self._b.close(); self._b.unlink()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __call__(self, v, g_t, g_y, g_x) -> np.ndarray:
        T, H, W = self.shape
        g_t, g_y, g_x = (np.asarray(g, np.float64) for g in (g_t, g_y, g_x))
        self.vin[...] = v
        nh = max(1, min(H, 4 * self.procs))
        hs = [H * i // nh for i in range(nh + 1)]
        self.pool.map(_t_chunk, [(hs[i], hs[i + 1], g_t) for i in range(nh) if hs[i] < hs[i + 1]])
        self.vin[...] = self.vout   # T-pass output becomes the spatial passes' input
        nt = max(1, min(T, 4 * self.procs))
        ts = [T * i // nt for i in range(nt + 1)]
        self.pool.map(_yx_chunk, [(ts[i], ts[i + 1], g_y, g_x) for i in range(nt) if ts[i] < ts[i + 1]])
        return self.vin.copy()


def power_iterate(F, g_t, g_s, K: int, x0=None, procs: int | None = None, iters: int | None = None):
    """sfseg_oracle.power_iterate (Eq.4/7/8) with the parallel filter.
    ``iters`` < K stops early (bounded CPU-baseline samples).  Returns (x, stats)."""
    F = np.asarray(F, np.float64)
    B = F.shape[0]
    K_run = K if iters is None else int(iters)
    stats = {"gain": np.zeros((B, K_run)), "rho": np.zeros((B, K_run)), "nu": np.zeros((B, K_run))}
    xs = np.empty_like(F)
    with ParallelFilter(F.shape[1:], procs) as filt:
        for b in range(B):
            x = F[b].copy() if x0 is None else np.asarray(x0[b], np.float64).copy()
            for k in range(K_run):
                y = F[b] * filt(F[b] * x, g_t, g_s, g_s)
                xx = float(np.sum(x * x))
                nu = math.sqrt(float(np.sum(y * y)))
                if nu == 0.0 or xx == 0.0:
                    raise DegenerateError(f"zero norm at iteration {k + 1}, volume {b}")
                stats["gain"][b, k] = nu / math.sqrt(xx)
                stats["rho"][b, k] = float(np.sum(x * y)) / xx
                stats["nu"][b, k] = nu
                x = y / nu
            xs[b] = x
    return xs, stats


def power_iterate_backward(ch, w, b, act, g_t, g_s, K: int, dL_dx, x0=None, procs: int | None = None):
    """sfseg_oracle.power_iterate_backward
    with the parallel filter.  Returns (dw [C], db)."""
    ch = np.asarray(ch, np.float64)
    F, z = combine(ch, w, b, act)
    dL_dx = np.asarray(dL_dx, np.float64)
    B = F.shape[0]
    F_bar = np.zeros_like(F)
    with ParallelFilter(F.shape[1:], procs) as filt:
        for bb in range(B):
            Fb = F[bb]
            x = Fb.copy() if x0 is None else np.asarray(x0[bb], np.float64).copy()
            xs, us, nus = [x], [], []
            for k in range(K):
                u = filt(Fb * x, g_t, g_s, g_s)
                y = Fb * u
                nu = math.sqrt(float(np.sum(y * y)))
                if nu == 0.0:
                    raise DegenerateError("zero norm")
                x = y / nu
                us.append(u)
                nus.append(nu)
                xs.append(x)
            xbar = dL_dx[bb].copy()
            for k in range(K, 0, -1):
                c = float(np.sum(xs[k] * xbar))
                ybar = (xbar - xs[k] * c) / nus[k - 1]
                v = filt(Fb * ybar, g_t, g_s, g_s)
                F_bar[bb] += ybar * us[k - 1] + xs[k - 1] * v
                xbar = Fb * v
            if x0 is None:
                F_bar[bb] += xbar
    if act == ACT_IDENTITY:
        dphi = np.ones_like(z)
    else:
        s = 1.0 / (1.0 + np.exp(-z))
        dphi = s * (1.0 - s)
    z_bar = F_bar * dphi
    dw = np.array([float(np.sum(z_bar * ch[:, c])) for c in range(ch.shape[1])])
    return dw, float(np.sum(z_bar))
