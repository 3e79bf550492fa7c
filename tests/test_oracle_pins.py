"""Pins of the CPU oracle against things other than itself.

CPU only (no GPU marker).  Each test names the pin and the passage it fixes.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
from oracle.dense import dense_M
import workloads as WL

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


# ----------------------------------------------------------------- P8: SPEC worked values
def test_p8_taps_spec_values():
    g = _gold("spec_examples.json")
    e = g["taps_r1_sigma1"]
    np.testing.assert_allclose(O.gaussian_taps(e["sigma"], e["radius"]), e["expected"], atol=e["atol"])
    e = g["taps_r0"]
    assert O.gaussian_taps(e["sigma"], e["radius"]).tolist() == e["expected"]
    e = g["taps_r2_sigma10_ratio"]
    t = O.gaussian_taps(e["sigma"], e["radius"])
    assert t.max() / t.min() < e["max_ratio"]
    with pytest.raises(ValueError):
        O.gaussian_taps(0.0, 3)


def test_taps_closed_form():
    """Ratios g[k]/g[0] = exp(-k^2/(2 sigma^2)) and unit sum (Eq.1 beta dist^2 term, A6)."""
    for sigma, r in [(1.0, 3), (2.0, 6), (8.0, 24), (12.0, 36), (1.5, 5), (0.5, 1)]:
        g = O.gaussian_taps(sigma, r)
        assert len(g) == 2 * r + 1
        assert abs(g.sum() - 1.0) < 1e-14
        k = np.arange(-r, r + 1)
        np.testing.assert_allclose(g / g[r], np.exp(-k * k / (2 * sigma * sigma)), rtol=1e-14)
        np.testing.assert_array_equal(g, g[::-1])


def test_p8_combine_spec_values():
    g = _gold("spec_examples.json")
    e = g["sigmoid_w2m1_b05"]
    ch = np.ones((1, 2, 2, 3, 3))
    F, _ = O.combine(ch, e["w"], e["b"], O.ACT_SIGMOID)
    np.testing.assert_allclose(F, e["expected"], atol=e["atol"])
    e = g["sigmoid_w0"]
    F, _ = O.combine(np.random.default_rng(1).random((1, 1, 2, 3, 3)), e["w"], e["b"], O.ACT_SIGMOID)
    np.testing.assert_allclose(F, e["expected"], atol=0)
    # saturation: w = [1000] on a binary channel -> the channel itself
    binary = (np.random.default_rng(2).random((1, 1, 3, 4, 4)) > 0.5).astype(np.float64) * 2 - 1
    F, _ = O.combine(binary, [1000.0], 0.0, O.ACT_SIGMOID)
    np.testing.assert_allclose(F, (binary[:, 0] > 0).astype(float), atol=1e-9)
    # identity combine is the plain weighted sum (A2)
    ch = np.random.default_rng(3).random((2, 3, 2, 4, 5))
    F, z = O.combine(ch, [0.2, -0.5, 1.5], 0.25, O.ACT_IDENTITY)
    np.testing.assert_allclose(F, 0.2 * ch[:, 0] - 0.5 * ch[:, 1] + 1.5 * ch[:, 2] + 0.25, rtol=1e-15)


def test_p8_normalize_spec_values():
    g = _gold("spec_examples.json")
    e = g["normalize_34"]
    np.testing.assert_allclose(O.normalize_l2(np.array(e["input"])), e["expected"], rtol=1e-15)
    with pytest.raises(O.DegenerateError):
        O.normalize_l2(np.zeros(5))


def test_p8_swap_matrix():
    """2-node swap graph -> v = [1,1]/sqrt2, lambda = 1.  A 1x1x2 volume with
    F = 1 and x-taps [1, 0, 1] (un-normalised, centre 0) is exactly that matrix."""
    F = np.ones((1, 1, 1, 2))
    lam = _gold("spec_examples.json")["swap_matrix"]["lambda"]
    x2, st2 = O.power_iterate(F, [1.0], [1.0], 3, g_x=np.array([1.0, 0.0, 1.0]),
                              x0=np.array([[[[1.0, 1.0]]]]))
    np.testing.assert_allclose(x2.ravel(), [1 / math.sqrt(2)] * 2, rtol=1e-15)
    np.testing.assert_allclose(st2["rho"][0], lam, rtol=1e-15)
    np.testing.assert_allclose(st2["gain"][0], lam, rtol=1e-15)


# ----------------------------------------------------------------- P1: separable == direct
def _direct_conv(v, gt, gy, gx):
    """Brute-force triple loop with the tensor-product kernel."""
    T, H, W = v.shape
    rt, ry, rx = len(gt) // 2, len(gy) // 2, len(gx) // 2
    out = np.zeros_like(v)
    for t in range(T):
        for y in range(H):
            for x in range(W):
                s = 0.0
                for a in range(-rt, rt + 1):
                    if not 0 <= t + a < T:
                        continue
                    for b in range(-ry, ry + 1):
                        if not 0 <= y + b < H:
                            continue
                        for c in range(-rx, rx + 1):
                            if 0 <= x + c < W:
                                s += gt[a + rt] * gy[b + ry] * gx[c + rx] * v[t + a, y + b, x + c]
                out[t, y, x] = s
    return out


@pytest.mark.parametrize("shape,radii", [((5, 9, 9), (2, 3, 3)), ((6, 12, 12), (1, 3, 2))])
def test_p1_separable_equals_direct(shape, radii):
    v = np.random.default_rng(7).random(shape)
    gt, gy, gx = (O.gaussian_taps(s, r) for s, r in zip((1.0, 1.7, 1.2), radii))
    sep = O.correlate_axis(O.correlate_axis(O.correlate_axis(v, gt, 0), gy, 1), gx, 2)
    ref = _direct_conv(v, gt, gy, gx)
    assert _rel(sep, ref) < 1e-13
    # gaussian_filter uses the same (t, y, x) pipeline
    assert _rel(O.gaussian_filter(v, gt, gy, gx), ref) < 1e-13


def test_p9_impulse_and_zero():
    """Impulse -> tensor-product kernel; zero -> zero; linearity."""
    gt, gs = O.gaussian_taps(1.0, 2), O.gaussian_taps(2.0, 4)
    v = np.zeros((7, 11, 13))
    v[3, 5, 6] = 1.0
    out = O.gaussian_filter(v, gt, gs, gs)
    k3 = gt[:, None, None] * gs[None, :, None] * gs[None, None, :]
    np.testing.assert_allclose(out[1:6, 1:10, 2:11], k3, rtol=1e-15, atol=0)
    assert out.sum() == pytest.approx(1.0, abs=1e-14)
    assert not O.gaussian_filter(np.zeros((3, 4, 5)), gt, gs, gs).any()
    a, b = np.random.default_rng(1).random((2, 4, 9, 9))
    lhs = O.gaussian_filter(2.0 * a - 3.0 * b, gt, gs, gs)
    rhs = 2.0 * O.gaussian_filter(a, gt, gs, gs) - 3.0 * O.gaussian_filter(b, gt, gs, gs)
    np.testing.assert_allclose(lhs, rhs, atol=1e-14)


def test_p9_closed_forms():
    """r = 0 on 1x1x1: y = F^2 x (S:197 with alpha = 1).  F == c and x constant:
    y = c^2 x at voxels >= r from every border (kernel sums to 1)."""
    F = np.array([[[[0.7]]]])
    x, st = O.power_iterate(F, [1.0], [1.0], 1, x0=np.array([[[[0.3]]]]))
    assert st["nu"][0, 0] == pytest.approx(0.49 * 0.3, rel=1e-15)
    assert x.ravel()[0] == pytest.approx(1.0, rel=1e-15)
    c = 0.6
    gt, gs = O.gaussian_taps(1.0, 2), O.gaussian_taps(1.5, 3)
    Fv = np.full((9, 12, 14), c)
    y = O.apply_M(Fv, np.full_like(Fv, 2.0), gt, gs, gs)
    np.testing.assert_allclose(y[2:-2, 3:-3, 3:-3], c * c * 2.0, rtol=1e-14)
    assert (y[0] < c * c * 2.0).all()   # zero padding attenuates the border frames


# ----------------------------------------------------------------- c1 dense pins P2-P7
@pytest.fixture(scope="module")
def c1_dense():
    wl = WL.generate("c1")
    cfg = wl.cfg
    F, _ = O.combine(wl.ch, wl.w, wl.b, O.ACT_IDENTITY)
    gt = O.gaussian_taps(cfg.sigma_t, cfg.radius_t)
    gs = O.gaussian_taps(cfg.sigma_s, cfg.radius_s)
    M = dense_M(F[0], gt, gs, gs)
    lam, V = np.linalg.eigh(M)
    return dict(cfg=cfg, F=F, gt=gt, gs=gs, M=M, lam=lam, V=V)


def test_p2_operator_equals_dense_matrix(c1_dense):
    d = c1_dense
    rng = np.random.default_rng(11)
    for x in (d["F"][0], rng.random(d["F"][0].shape)):
        y = O.apply_M(d["F"][0], x, d["gt"], d["gs"], d["gs"])
        ym = d["M"] @ x.ravel()
        assert _rel(y.ravel(), ym) < 1e-13
    assert np.allclose(d["M"], d["M"].T, atol=0)       # symmetric
    assert (d["M"] >= 0).all()                          # non-negative


def test_p3_p4_closed_form_and_brute_force(c1_dense):
    d = c1_dense
    K = d["cfg"].K
    x_orc, st = O.power_iterate(d["F"], d["gt"], d["gs"], K)
    # P3: x_K proportional to V Lambda^K V^T x_0
    x0 = d["F"][0].ravel()
    xc = d["V"] @ (d["lam"] ** K * (d["V"].T @ x0))
    xc /= np.linalg.norm(xc)
    assert _rel(x_orc.ravel(), xc) < 1e-12
    # P4: dense brute-force power iteration with normalisation
    x = x0.copy()
    for _ in range(K):
        x = d["M"] @ x
        x /= np.linalg.norm(x)
    assert _rel(x_orc.ravel(), x) < 1e-13
    # per-iteration gains against the dense operator
    x = x0.copy()
    for k in range(K):
        y = d["M"] @ x
        assert st["gain"][0, k] == pytest.approx(np.linalg.norm(y) / np.linalg.norm(x), rel=1e-13)
        assert st["rho"][0, k] == pytest.approx(x @ y / (x @ x), rel=1e-13)
        x = y / np.linalg.norm(y)


def test_p5_perron_frobenius(c1_dense):
    d = c1_dense
    lam, V = d["lam"], d["V"]
    v = V[:, -1] * np.sign(V[:, -1].sum())
    assert (v > 0).all()                      # F > 0 everywhere in c1 -> irreducible, strictly positive
    assert lam[-1] > abs(lam[0])
    assert lam[-1] > lam[-2]
    _, st = O.power_iterate(d["F"], d["gt"], d["gs"], d["cfg"].K, keep_iterates=True)
    for it in st["iterates"][0]:
        assert (it >= 0).all()


def test_p6_monotone_gain(c1_dense):
    d = c1_dense
    _, st = O.power_iterate(d["F"], d["gt"], d["gs"], 30)
    gain, rho = st["gain"][0], st["rho"][0]
    assert (np.diff(gain) >= -1e-15 * gain[1:]).all()        # exact for symmetric M
    assert (np.diff(rho) >= -1e-12 * np.abs(rho[1:])).all()  # A11 tolerance (M slightly indefinite)
    assert rho[-1] <= d["lam"][-1] + 1e-15


def test_p7_eigenvalue_matches_solver(c1_dense):
    d = c1_dense
    v = d["V"][:, -1] * np.sign(d["V"][:, -1].sum())
    x, st = O.power_iterate(d["F"], d["gt"], d["gs"], 900)
    assert abs(st["rho"][0, -1] - d["lam"][-1]) < 1e-10 * d["lam"][-1]
    assert abs(st["gain"][0, -1] - d["lam"][-1]) < 1e-9 * d["lam"][-1]
    assert _rel(x.ravel(), v) < 1e-6


def test_p10_misinitialised_convergence():
    """Fig. approx: from a start 70 deg away from the eigenvector (in the
    non-negative cone) the angle shrinks to ~0."""
    rng = np.random.default_rng(5)
    F = np.clip(rng.random((1, 4, 8, 8)) * 0.4 + 0.6, 0, 1)
    F[0, :, 2:6, 2:6] = 1.0
    gt, gs = O.gaussian_taps(1.0, 2), O.gaussian_taps(1.5, 3)
    M = dense_M(F[0], gt, gs, gs)
    lam, V = np.linalg.eigh(M)
    v = V[:, -1] * np.sign(V[:, -1].sum())
    e = np.zeros_like(v)
    e[0] = 1.0                                     # a corner voxel indicator

    def ang(a, b):
        return math.degrees(math.acos(min(1.0, a @ b / np.linalg.norm(a) / np.linalg.norm(b))))
    lo, hi = 0.0, 1e6
    for _ in range(200):                          # bisection on x0 = v + s e to get 70 deg
        mid = 0.5 * (lo + hi)
        lo, hi = (mid, hi) if ang(v + mid * e, v) < 70.0 else (lo, mid)
    x0 = (v + lo * e).reshape(F.shape)
    assert abs(ang(x0.ravel(), v) - 70.0) < 1e-6
    angles = []
    x = x0
    for _ in range(60):
        x, _ = O.power_iterate(F, gt, gs, 1, x0=x)
        angles.append(ang(x.ravel(), v))
    assert all(a2 <= a1 + 1e-9 for a1, a2 in zip(angles[3:], angles[4:]))
    assert angles[-1] < 0.5


# ----------------------------------------------------------------- P11: equivariances
def test_p11_equivariances():
    wl = WL.generate("c1")
    F, _ = O.combine(wl.ch, wl.w, wl.b)
    gt, gs = O.gaussian_taps(1.0, 3), O.gaussian_taps(2.0, 6)
    x, st = O.power_iterate(F, gt, gs, 6)
    for ax in (1, 2, 3):
        xm, stm = O.power_iterate(np.flip(F, ax), gt, gs, 6)
        np.testing.assert_allclose(np.flip(xm, ax), x, atol=1e-14)
        np.testing.assert_allclose(stm["gain"], st["gain"], rtol=1e-13)
    xs, sts = O.power_iterate(3.7 * F, gt, gs, 6)
    np.testing.assert_allclose(xs, x, atol=1e-14)
    np.testing.assert_allclose(sts["gain"], 3.7 ** 2 * st["gain"], rtol=1e-13)
    ch = np.random.default_rng(4).random((1, 3, 4, 6, 7))
    w = np.array([0.2, 0.3, 0.5])
    perm = [2, 0, 1]
    Fa, _ = O.combine(ch, w, 0.1, O.ACT_SIGMOID)
    Fb, _ = O.combine(ch[:, perm], w[perm], 0.1, O.ACT_SIGMOID)
    np.testing.assert_allclose(Fa, Fb, rtol=1e-15)


# ----------------------------------------------------------------- P12: gradient
def _loss_and_grad_x(x, m):
    """A13: L = mean (x - m_hat)^2, m_hat = m / ||m||.  Returns L, dL/dx."""
    mh = m / np.linalg.norm(m)
    d = x - mh
    return float(np.mean(d * d)), 2.0 * d / d.size


def _loss(ch, w, b, act, gt, gs, K, m):
    F, _ = O.combine(ch, w, b, act)
    x, _ = O.power_iterate(F, gt, gs, K)
    return _loss_and_grad_x(x, m)


@pytest.mark.parametrize("act,b", [(O.ACT_IDENTITY, 0.0), (O.ACT_SIGMOID, 0.3)])
def test_p12_gradient_vs_finite_differences(act, b):
    rng = np.random.default_rng(9)
    ch = rng.random((1, 3, 6, 12, 12))
    m = (rng.random((1, 6, 12, 12)) > 0.6).astype(np.float64)
    w = np.array([0.5, 0.3, 0.8])
    gt, gs = O.gaussian_taps(1.0, 2), O.gaussian_taps(1.5, 4)
    K = 5
    F, _ = O.combine(ch, w, b, act)
    x, _ = O.power_iterate(F, gt, gs, K)
    _, g = _loss_and_grad_x(x, m)
    dw, db = O.power_iterate_backward(ch, w, b, act, gt, gs, K, g)
    fd = np.zeros(3)
    for c in range(3):
        h = 1e-6 * abs(w[c])
        wp, wm = w.copy(), w.copy()
        wp[c] += h
        wm[c] -= h
        fd[c] = (_loss(ch, wp, b, act, gt, gs, K, m)[0] - _loss(ch, wm, b, act, gt, gs, K, m)[0]) / (2 * h)
    h = 1e-6
    fdb = (_loss(ch, w, b + h, act, gt, gs, K, m)[0] - _loss(ch, w, b - h, act, gt, gs, K, m)[0]) / (2 * h)
    assert _rel(dw, fd) < 1e-6
    assert abs(db - fdb) < 1e-6 * max(abs(fdb), np.abs(fd).max())
    if act == O.ACT_IDENTITY and b == 0.0:
        # Euler identity: F linear in w and x_K scale-invariant -> w . dL/dw = 0
        assert abs(w @ dw) < 1e-12 * np.linalg.norm(w) * np.linalg.norm(dw)


def test_p12_single_channel_zero_gradient():
    rng = np.random.default_rng(10)
    ch = rng.random((2, 1, 4, 8, 8))
    gt, gs = O.gaussian_taps(1.0, 2), O.gaussian_taps(1.5, 3)
    g = rng.normal(size=(2, 4, 8, 8))
    dw, _ = O.power_iterate_backward(ch, [0.7], 0.0, O.ACT_IDENTITY, gt, gs, 4, g)
    F, _ = O.combine(ch, [0.7], 0.0)
    dw_scale = O.power_iterate_backward(ch, [1.0], 0.0, O.ACT_IDENTITY, gt, gs, 4, g)[0]
    assert abs(dw[0]) < 1e-12 * np.abs(g).sum() * F.max()
    assert abs(dw_scale[0]) < 1e-12 * np.abs(g).sum()


def test_p12_user_x0_gradient_fd():
    """With a given x_0 the recursion omits the x_bar_0 term; check by FD."""
    rng = np.random.default_rng(12)
    ch = rng.random((1, 2, 4, 6, 7))
    x0 = rng.random((1, 4, 6, 7))
    w = np.array([0.6, 0.9])
    gt, gs = O.gaussian_taps(1.0, 2), O.gaussian_taps(1.2, 2)
    g = rng.normal(size=(1, 4, 6, 7))

    def L(wv):
        F, _ = O.combine(ch, wv, 0.1, O.ACT_SIGMOID)
        x, _ = O.power_iterate(F, gt, gs, 3, x0=x0)
        return float(np.sum(g * x))
    dw, _ = O.power_iterate_backward(ch, w, 0.1, O.ACT_SIGMOID, gt, gs, 3, g, x0=x0)
    fd = [(L(w + h * e) - L(w - h * e)) / (2 * h) for e, h in ((np.eye(2)[i], 1e-6) for i in range(2))]
    assert _rel(dw, fd) < 1e-6


# ----------------------------------------------------------------- threshold (definitional)
def test_threshold_definition():
    d = _gold("threshold_tiny.json")
    x = np.array(d["x"])
    assert O.threshold(x, d["tau"], O.THR_PER_FRAME_MAX).tolist() == d["per_frame_max"]
    assert O.threshold(x, d["tau"], O.THR_GLOBAL_MAX).tolist() == d["global_max"]
    assert O.threshold(x, d["tau"], O.THR_ABSOLUTE).tolist() == d["absolute"]


# ----------------------------------------------------------------- degenerate
def test_degenerate_zero_F():
    with pytest.raises(O.DegenerateError):
        O.power_iterate(np.zeros((1, 2, 3, 4)), [1.0], [1.0], 2)
