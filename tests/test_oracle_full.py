"""Pins of the full SFSeg operator oracle (oracle/full.py).

Each pin checks the Eq.7 three-convolution form against something other than
itself: the entry-by-entry Eq.2 adjacency matrix, SPEC's closed forms, the
hot-path oracle it must reduce to, and the symmetry / Perron-Frobenius
properties the paper states.
"""
import math

import numpy as np
import pytest

import oracle as O


def _taps(rt, rs):
    return O.gaussian_taps(max(rt, 1) / 2.0, rt), O.gaussian_taps(max(rs, 1) / 2.0, rs)


@pytest.mark.parametrize("shape,rt,rs,p,alpha", [
    ((3, 5, 6), 1, 2, 1.0, 1.0),
    ((4, 6, 5), 2, 1, 0.2, 1.0),
    ((2, 7, 7), 1, 3, 0.1, 0.5),
    ((5, 4, 4), 3, 2, 0.5, 2.0),      # alpha > 1: brackets may go negative; still Eq.2 exactly
])
def test_full_step_equals_taylor_matrix(shape, rt, rs, p, alpha):
    """Eq.7 (three convolutions) == Eq.2 matrix (entry by entry) times x, P:119-125 / P:166-173."""
    rng = np.random.default_rng(sum(shape) + rt + rs)
    S, F, x = rng.random(shape), rng.random(shape), rng.random(shape)
    gt, gs = _taps(rt, rs)
    M = O.dense_M_taylor(S, F, p, alpha, gt, gs, gs)
    ref = (M @ x.ravel()).reshape(shape)
    got = O.full_step(np.power(S, p), F, alpha, x, gt, gs, gs)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_full_step_closed_forms_spec():
    """1x1x1, radius 0: s^{2p} alpha^-1 x (the F terms cancel);
    S:197 -- S == 1, F constant: alpha^-1 G*X (pure Gaussian smoothing)."""
    g0 = np.array([1.0])
    s, f, x, p, alpha = 0.7, 0.3, 2.5, 0.2, 0.8
    y = O.full_step(np.full((1, 1, 1), s ** p), np.full((1, 1, 1), f), alpha, np.full((1, 1, 1), x), g0, g0, g0)
    assert abs(y.item() - s ** (2 * p) / alpha * x) <= 1e-15
    rng = np.random.default_rng(1)
    X = rng.random((4, 9, 8))
    gt, gs = _taps(1, 3)
    y = O.full_step(np.ones_like(X), np.full_like(X, 0.6), alpha, X, gt, gs, gs)
    ref = O.gaussian_filter(X, gt, gs, gs) / alpha
    assert np.abs(y - ref).max() <= 1e-14


def test_full_reduces_to_hot_path():
    """F == 0, alpha = 1, p = 1: M_ij = s_i s_j G_ij, the north-star operator (reading A3)."""
    rng = np.random.default_rng(2)
    S = rng.random((1, 5, 10, 12))
    gt, gs = _taps(2, 3)
    xf, stf = O.power_iterate_full(S, S, np.zeros_like(S), 1.0, gt, gs, 6)
    xh, sth = O.power_iterate(S, gt, gs, 6)
    assert np.abs(xf - xh).max() <= 1e-14
    np.testing.assert_allclose(stf["gain"], sth["gain"], rtol=1e-13)


def test_full_operator_symmetric():
    """<a, M b> == <M a, b> for the Eq.7 operator (M symmetric)."""
    rng = np.random.default_rng(3)
    U, F = rng.random((4, 8, 9)), rng.random((4, 8, 9))
    a, b = rng.normal(size=(4, 8, 9)), rng.normal(size=(4, 8, 9))
    gt, gs = _taps(2, 3)
    l = float(np.sum(a * O.full_step(U, F, 0.9, b, gt, gs, gs)))
    r = float(np.sum(O.full_step(U, F, 0.9, a, gt, gs, gs) * b))
    assert abs(l - r) <= 1e-12 * max(abs(l), 1.0)


def test_full_power_iteration_matches_dense_and_perron_frobenius():
    """K iterations == dense brute force (Eq.4); S,F in [0,1], alpha <= 1 -> non-negative
    iterates and a non-negative principal eigenvector; the gain rises (symmetric M)."""
    rng = np.random.default_rng(4)
    shape = (3, 6, 7)
    S, F = rng.random(shape) * 0.9 + 0.05, rng.random(shape)
    p, alpha, K = 0.2, 1.0, 8
    gt, gs = _taps(1, 2)
    U = np.power(S, p)
    xs, st = O.power_iterate_full(S[None], U[None], F[None], alpha, gt, gs, K)
    M = O.dense_M_taylor(S, F, p, alpha, gt, gs, gs)
    assert (M >= 0).all()
    x = S.ravel().copy()
    for _ in range(K):
        y = M @ x
        x = y / np.linalg.norm(y)
    assert np.abs(xs[0].ravel() - x).max() <= 1e-13
    assert (xs >= 0).all()
    g = st["gain"][0]
    assert (np.diff(g[1:]) >= -1e-12).all()
    w, V = np.linalg.eigh(M)
    v = V[:, -1] * np.sign(V[:, -1].sum())
    assert (v >= -1e-12).all() and w[-1] >= abs(w[0])


def test_combine_full_maps_and_power():
    """Eq.9 for both maps (sigmoid, S:189 worked value) and U = S^p (reading A19)."""
    ones = np.ones((1, 2, 1, 2, 2))
    S, U, F = O.combine_full(ones, [2.0, -1.0], 0.5, 1, ones[:, :1], [0.0], 0.0, 1, 0.5)
    assert abs(S.max() - 1.0 / (1.0 + math.exp(-1.5))) <= 1e-15
    assert abs(F.max() - 0.5) <= 1e-15
    assert np.allclose(U, np.sqrt(S), rtol=0, atol=1e-15)


# --------------------------------------------------------------------------- row f2
def test_soft_binarize_spec_values():
    """x = theta -> 0.5; kappa 4, x - theta = 0.25 -> sigma(1); saturation to {0, 1};
    the map is monotone (order preserving)."""
    x = np.array([0.25, 0.75])          # theta = mean of positives = 0.5
    y = O.soft_binarize(x, 4.0)
    assert abs(y[1] - 1.0 / (1.0 + math.exp(-1.0))) <= 1e-15
    assert abs(O.soft_binarize(np.array([0.5, 0.5]), 7.0)[0] - 0.5) <= 1e-15
    z = O.soft_binarize(np.array([0.1, 0.9]), 1e4)
    assert abs(z[0]) <= 1e-6 and abs(z[1] - 1.0) <= 1e-6
    r = np.random.default_rng(0).random(50)
    assert (np.argsort(O.soft_binarize(r, 3.0), kind="stable") == np.argsort(r, kind="stable")).all()


def test_binarized_iteration_follows_alg1():
    """With binarize=(n_cont, k0, g): iterations <= n_cont are the plain Eq.7/8 steps; after each
    later iteration the normalised iterate is soft-binarised with the geometric kappa."""
    rng = np.random.default_rng(5)
    S, F = rng.random((1, 3, 6, 7)), rng.random((1, 3, 6, 7))
    gt, gs = _taps(1, 2)
    U = np.power(S, 0.5)
    xb, stb = O.power_iterate_full(S, U, F, 1.0, gt, gs, 5, binarize=(3, 4.0, 2.0))
    x = S[0].copy()
    for k in range(5):
        y = O.full_step(U[0], F[0], 1.0, x, gt, gs, gs)
        x = y / np.linalg.norm(y)
        if k + 1 > 3:
            x = O.soft_binarize(x, 4.0 * 2.0 ** (k - 3))
    assert np.abs(xb[0] - x).max() <= 1e-14
    assert 0.0 < xb.min() and xb.max() < 1.0
