"""Plain float64 CPU oracle of the SFSeg power-iteration hot path.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  Shares no code with the
CUDA path.  Every function cites the passage of /root/reference/PAPER.md
("P:<lines>") or SPEC.md ("S:<lines>") it transcribes; readings of ambiguous
passages are the SURVEY.md §8(c) readings A1-A17, listed in DESIGN.md.

Hot path (BASELINE.json north_star): x <- F * (G (*) (F * x)), then L2
normalisation -- the unary-only case of Eq.7 / Eq.10
with exponent p = 1 and a constant pairwise map, i.e. M_ij = F_i F_j G(i - j).
Arrays are float64 numpy, layout [B][T][H][W] (C-order, W fastest); channel
stacks are [B][C][T][H][W].
"""
from __future__ import annotations

import math

import numpy as np

ACT_IDENTITY = 0
ACT_SIGMOID = 1
THR_PER_FRAME_MAX = 0
THR_GLOBAL_MAX = 1
THR_ABSOLUTE = 2


class DegenerateError(ValueError):
    """Zero-norm iterate (normalize_l2 of an all-zero vector is an error)."""


# --------------------------------------------------------------------------- O1
def gaussian_taps(sigma: float, radius: int) -> np.ndarray:
    """1D Gaussian taps g[k] = exp(-k^2 / (2 sigma^2)) / sum, k = -r..r.

    G_3D is the separable Gaussian of Eq.1's  e^{-beta dist^2}  term
    ("G_{i,j}"; separability P:319).  Per-axis normalisation to sum 1
    is reading A6; radius = ceil(3 sigma) is reading A5.
    """
    if not (sigma > 0):
        raise ValueError("sigma must be > 0 (S:113)")
    if radius < 0:
        raise ValueError("radius must be >= 0")
    k = np.arange(-radius, radius + 1, dtype=np.float64)
    g = np.exp(-(k * k) / (2.0 * sigma * sigma))
    return g / g.sum()


# --------------------------------------------------------------------------- O2
def combine(ch: np.ndarray, w, b: float = 0.0, act: int = ACT_IDENTITY):
    """Channel combine, Eq.9 / Alg.1 lines 1-2.

    z = sum_c w_c ch_c + b ;  F = z (identity: the single-channel case "without
    the sigmoid", reading A2) or F = 1 / (1 + e^{-z}) (sigmoid; the
    printed 1/(1+e^{x}) is a typo, reading A1 / S:252).
    ch: [B][C][T][H][W].  Returns (F, z), both float64 [B][T][H][W].
    """
    ch = np.asarray(ch, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64).reshape(-1)
    if ch.ndim != 5 or ch.shape[1] != w.shape[0]:
        raise ValueError("ch must be [B][C][T][H][W] with C == len(w)")
    z = np.full(ch.shape[:1] + ch.shape[2:], float(b), dtype=np.float64)
    for c in range(w.shape[0]):
        z += w[c] * ch[:, c]
    if act == ACT_IDENTITY:
        F = z.copy()
    elif act == ACT_SIGMOID:
        with np.errstate(over="ignore"):
            F = 1.0 / (1.0 + np.exp(-z))
    else:
        raise ValueError("unknown activation")
    return F, z


# --------------------------------------------------------------------------- O4 pieces
def correlate_axis(v: np.ndarray, g: np.ndarray, axis: int) -> np.ndarray:
    """Zero-padded 1D correlation along ``axis``: out[i] = sum_k g[k+r] v[i+k].

    One of the "three vector-wise convolutions" of P:319; zero padding is
    reading A8 (missing neighbours contribute nothing to Eq.4's sum).
    The kernel is symmetric so correlation == convolution.  Written as one
    shifted add per tap.
    """
    r = (len(g) - 1) // 2
    n = v.shape[axis]
    out = np.zeros_like(v, dtype=np.float64)
    for k in range(-r, r + 1):
        lo, hi = max(0, -k), min(n, n - k)
        if lo >= hi:
            continue
        dst = [slice(None)] * v.ndim
        src = [slice(None)] * v.ndim
        dst[axis] = slice(lo, hi)
        src[axis] = slice(lo + k, hi + k)
        out[tuple(dst)] += g[k + r] * v[tuple(src)]
    return out


def gaussian_filter(v: np.ndarray, g_t, g_y, g_x) -> np.ndarray:
    """G_3D (*) v for one volume [T][H][W]: T pass, then H, then W."""
    v = np.asarray(v, dtype=np.float64)
    out = correlate_axis(v, np.asarray(g_t, np.float64), 0)
    out = correlate_axis(out, np.asarray(g_y, np.float64), 1)
    return correlate_axis(out, np.asarray(g_x, np.float64), 2)


def apply_M(F: np.ndarray, x: np.ndarray, g_t, g_y, g_x) -> np.ndarray:
    """y = M x with M_ij = F_i F_j G_ij, one volume.

    Eq.7 with S^p = F (p = 1, reading A3) and a constant pairwise
    map, whose bracket [alpha^-1 - F^2 ...] collapses to alpha^-1, and
    alpha = 1:  X_crt = S . G_3D * (S . X).
    """
    return F * gaussian_filter(F * x, g_t, g_y, g_x)


def normalize_l2(y: np.ndarray) -> np.ndarray:
    """Eq.8: X <- X / ||X||_2 over the whole volume (reading A9)."""
    n = math.sqrt(float(np.sum(np.asarray(y, np.float64) ** 2)))
    if n == 0.0:
        raise DegenerateError("zero-norm iterate")
    return y / n


# --------------------------------------------------------------------------- row f2
def soft_binarize(x: np.ndarray, kappa: float) -> np.ndarray:
    """Alg.1 STEP 3: X_m <- sigma(X_m), "a sigmoid function (controlled by a
    parameter)".  Reading A21: sigma(kappa (x - theta)) with
    theta = mean of the strictly positive entries of x (0 if there are none)."""
    x = np.asarray(x, np.float64)
    pos = x[x > 0]
    theta = float(pos.mean()) if pos.size else 0.0
    with np.errstate(over="ignore"):
        return 1.0 / (1.0 + np.exp(-kappa * (x - theta)))


def binarize_kappa(k: int, binarize) -> float:
    """Steepness of iteration k (1-based) under binarize = (n_cont, kappa0, growth), or 0
    when iteration k is not binarised: Alg.1 STEP 3 runs after the N_cont continuous
    iterations ("gradually"); SPEC's geometric schedule (S:224,
    S:251: start kappa0, times growth per iteration) -- reading A21."""
    if binarize is None or k <= binarize[0]:
        return 0.0
    return float(binarize[1]) * float(binarize[2]) ** (k - binarize[0] - 1)


# --------------------------------------------------------------------------- O3/O4
def power_iterate(F: np.ndarray, g_t, g_s, K: int, x0=None, g_x=None,
                  keep_iterates: bool = False, binarize=None):
    """K power iterations of Eq.4 in the filtering form of Eq.7/8.

    F: [B][T][H][W].  x_0 = F (Alg.1 line 3, "X_m <- S_m"; reading A10:
    x_0 is not normalised) unless ``x0`` is given.  For k = 1..K, per volume:
        y_k   = F * G(F * x_{k-1})                         (Eq.7, p = 1)
        nu_k  = ||y_k||_2
        gain_k = nu_k / ||x_{k-1}||_2                      (n_k, reading A10)
        rho_k = <x_{k-1}, y_k> / ||x_{k-1}||^2             (Rayleigh quotient, Eq.3)
        x_k   = y_k / nu_k                                  (Eq.8)
    ``g_s`` is used for both spatial axes unless ``g_x`` is given.
    binarize = (n_cont, kappa0, growth): after the normalisation of every iteration
    k > n_cont the iterate is soft-binarised, x_k <- soft_binarize(x_k, kappa_k)
    (Alg.1 STEP 3; reading A21) and is the next iterate as is; the output is
    then the last binarised iterate (values in (0, 1)).
    Returns (x_K float64 [B][T][H][W], stats) with stats arrays of shape [B][K].
    """
    F = np.asarray(F, dtype=np.float64)
    if F.ndim != 4:
        raise ValueError("F must be [B][T][H][W]")
    g_y = np.asarray(g_s, np.float64)
    g_x = g_y if g_x is None else np.asarray(g_x, np.float64)
    B = F.shape[0]
    gains = np.zeros((B, K))
    rhos = np.zeros((B, K))
    nus = np.zeros((B, K))
    xs = np.empty_like(F)
    iterates = []
    for b in range(B):
        x = F[b].copy() if x0 is None else np.asarray(x0[b], np.float64).copy()
        it_b = [x.copy()] if keep_iterates else None
        for k in range(K):
            y = apply_M(F[b], x, g_t, g_y, g_x)
            xx = float(np.sum(x * x))
            nu = math.sqrt(float(np.sum(y * y)))
            if nu == 0.0 or xx == 0.0:
                raise DegenerateError(f"zero norm at iteration {k + 1}, volume {b}")
            gains[b, k] = nu / math.sqrt(xx)
            rhos[b, k] = float(np.sum(x * y)) / xx
            nus[b, k] = nu
            x = y / nu
            kap = binarize_kappa(k + 1, binarize)
            if kap > 0.0:
                x = soft_binarize(x, kap)
            if keep_iterates:
                it_b.append(x.copy())
        xs[b] = x
        if keep_iterates:
            iterates.append(it_b)
    stats = {"gain": gains, "rho": rhos, "nu": nus}
    if keep_iterates:
        stats["iterates"] = iterates
    return xs, stats


# --------------------------------------------------------------------------- O5
def threshold(x: np.ndarray, tau: float, mode: int = THR_PER_FRAME_MAX) -> np.ndarray:
    """Hard threshold of the eigenvector, "simply obtained by thresholding",
    "we apply a hard threshold".

    Reading A12: PER_FRAME_MAX rescales each frame by its max before comparing,
    mask = x / max_frame(x) > tau (strict); a frame whose max is <= 0 gives an
    all-zero mask.  GLOBAL_MAX uses the per-volume max; ABSOLUTE compares x > tau.
    x: [B][T][H][W] -> uint8 mask.
    """
    x = np.asarray(x, dtype=np.float64)
    if mode == THR_ABSOLUTE:
        return (x > tau).astype(np.uint8)
    if mode == THR_PER_FRAME_MAX:
        m = x.max(axis=(2, 3), keepdims=True)
    elif mode == THR_GLOBAL_MAX:
        m = x.max(axis=(1, 2, 3), keepdims=True)
    else:
        raise ValueError("unknown threshold mode")
    out = np.zeros(x.shape, dtype=np.uint8)
    pos = np.broadcast_to(m > 0, x.shape)
    safe = np.where(m > 0, m, 1.0)
    out[pos] = ((x / safe) > tau)[pos]
    return out


# --------------------------------------------------------------------------- O6
def power_iterate_backward(ch, w, b, act, g_t, g_s, K: int, dL_dx, x0=None, binarize=None):
    """Gradient of L(x_K) w.r.t. the channel weights w and bias b, through the
    K unrolled iterations ("gradient ... through the full spectral algorithm",
    P:42).  SURVEY.md Appendix A recursion, per volume:

        x_bar_K = dL/dx_K
        for k = K..1:
            c_k     = <x_k, x_bar_k>
            y_bar_k = (x_bar_k - x_k c_k) / nu_k                   (through Eq.8)
            v_k     = G(F * y_bar_k)                               (G symmetric)
            F_bar  += y_bar_k * u_{k-1} + x_{k-1} * v_k            (u_{k-1} = G(F x_{k-1}))
            x_bar_{k-1} = F * v_k
        F_bar += x_bar_0                (x_0 = F, Alg.1 line 3; skipped if x0 given)
        z_bar = F_bar * phi'(z);  dw_c = <z_bar, ch_c>;  db = sum z_bar   (Eq.9)

    With binarize (row f2), iteration k > n_cont ends with b_k = sigma(kappa_k (x_k -
    theta_k)), theta_k = mean of the positive entries of x_k (A21), and b_k is the next
    iterate; its adjoint is first pulled back through the sigmoid and the centre:
        g = kappa_k sigma'(z) b_bar ;  x_bar_k = g - [x_k > 0] sum(g) / n_pos
    (d theta / d x_j = [x_j > 0] / n_pos), then through Eq.8 as above.

    Returns (dw float64 [C], db float64), summed over volumes.
    """
    ch = np.asarray(ch, np.float64)
    F, z = combine(ch, w, b, act)
    g_y = np.asarray(g_s, np.float64)
    dL_dx = np.asarray(dL_dx, np.float64)
    B = F.shape[0]
    F_bar = np.zeros_like(F)
    for bb in range(B):
        Fb = F[bb]
        x = Fb.copy() if x0 is None else np.asarray(x0[bb], np.float64).copy()
        xs, xn, us, nus = [x], [None], [], []   # xs[k]: input of iteration k+1; xn[k]: y_k / nu_k
        for k in range(K):
            u = gaussian_filter(Fb * x, g_t, g_y, g_y)
            y = Fb * u
            nu = math.sqrt(float(np.sum(y * y)))
            if nu == 0.0:
                raise DegenerateError("zero norm")
            x = y / nu
            xn.append(x)
            kap = binarize_kappa(k + 1, binarize)
            if kap > 0.0:
                x = soft_binarize(x, kap)
            us.append(u)
            nus.append(nu)
            xs.append(x)
        xbar = dL_dx[bb].copy()
        for k in range(K, 0, -1):
            kap = binarize_kappa(k, binarize)
            if kap > 0.0:   # xbar is the adjoint of b_k: pull it back to x_k = y_k / nu_k
                s = xs[k] * (1.0 - xs[k])          # sigma'(z) = b (1 - b)
                g = kap * s * xbar
                pos = xn[k] > 0
                xbar = g - pos * (float(np.sum(g)) / max(int(pos.sum()), 1))
            c = float(np.sum(xn[k] * xbar))
            ybar = (xbar - xn[k] * c) / nus[k - 1]
            v = gaussian_filter(Fb * ybar, g_t, g_y, g_y)
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
    db = float(np.sum(z_bar))
    return dw, db
