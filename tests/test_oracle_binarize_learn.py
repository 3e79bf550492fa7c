"""Pins of the SURVEY.md §8(f) rows f2 (soft-binarisation on the hot path, forward and
backward) and f4 (Focal-Dice loss, Eq.12) in the oracle, each with a committed seeded
mutation that the pin must catch (tests/_mutation.py)."""
import math

import numpy as np
import pytest

import oracle as O
from oracle import learn as OL
from oracle import online as OO
from oracle import sfseg_oracle as OS
from _mutation import mutant

ID = np.array([1.0])   # radius-0 taps: G is the identity, so y = F^2 x voxelwise (P:144 with G = I)


def _logit(p):
    return math.log(p / (1.0 - p))


def _observed_kappa(out, xn):
    """kappa seen in a binarised output: out = sigma(kappa (xn - theta)), theta = mean of xn > 0."""
    theta = float(xn[xn > 0].mean())
    i = int(np.argmax(np.abs(xn - theta)))
    return _logit(float(out[i])) / float(xn[i] - theta)


def _kappa_pin(power_iterate):
    """SPEC S:224 / S:251 defaults (start 4, growth 2 per iteration, first binarised iteration
    n_cont + 1), observed in outputs of a two-voxel volume with G = I."""
    F = np.array([0.5, 0.8]).reshape(1, 1, 1, 2)
    f = F.ravel()
    bz = (1, 4.0, 2.0)
    out1, _ = power_iterate(F, ID, ID, 1, binarize=bz)       # iteration 1 <= n_cont: continuous
    x1 = f ** 3 / np.linalg.norm(f ** 3)                      # x_1 = M F / ||M F||, M = diag(F^2)
    if np.abs(out1.ravel() - x1).max() > 1e-14:
        return False
    out2, _ = power_iterate(F, ID, ID, 2, binarize=bz)
    xn2 = f ** 5 / np.linalg.norm(f ** 5)                     # normalised y_2, before binarisation
    if abs(_observed_kappa(out2.ravel(), xn2) - 4.0) > 1e-9:
        return False
    out3, _ = power_iterate(F, ID, ID, 3, binarize=bz)
    y3 = f ** 2 * out2.ravel()                                # iteration 3 starts from b_2 as is
    xn3 = y3 / np.linalg.norm(y3)
    return abs(_observed_kappa(out3.ravel(), xn3) - 8.0) <= 1e-9


def test_kappa_schedule_pinned_by_observed_outputs():
    assert _kappa_pin(O.power_iterate)


@pytest.mark.parametrize("old,new", [
    ("** (k - binarize[0] - 1)", "** (k - binarize[0])"),     # schedule one step late
    ("k <= binarize[0]", "k < binarize[0]"),                   # binarises iteration n_cont too
])
def test_kappa_pin_catches_mutations(old, new):
    bad_kappa = mutant(OS.binarize_kappa, old, new)
    ns_pi = mutant(OS.power_iterate, "kap = binarize_kappa(k + 1, binarize)",
                   "kap = _bk(k + 1, binarize)")
    ns_pi.__globals__["_bk"] = bad_kappa
    assert not _kappa_pin(ns_pi)


# --------------------------------------------------------------------------- backward through f2
def _fd_case():
    rng = np.random.default_rng(7)
    ch = rng.random((1, 2, 5, 9, 11)) * 0.8 + 0.1
    w, b, act = np.array([0.7, -0.4]), 0.3, O.ACT_SIGMOID
    gt, gs = O.gaussian_taps(1.0, 2), O.gaussian_taps(1.5, 4)
    r = rng.normal(size=(1, 5, 9, 11))
    return ch, w, b, act, gt, gs, r


def _fd_rel_err(backward, binarize, K=4):
    ch, w, b, act, gt, gs, r = _fd_case()

    def loss(wv, bv):
        F, _ = O.combine(ch, wv, bv, act)
        x, _ = O.power_iterate(F, gt, gs, K, binarize=binarize)
        return float(np.sum(r * x))

    dw, db = backward(ch, w, b, act, gt, gs, K, r, binarize=binarize)
    h = 1e-6
    fd = []
    for c in range(len(w)):
        e = np.zeros_like(w)
        e[c] = h
        fd.append((loss(w + e, b) - loss(w - e, b)) / (2 * h))
    fdb = (loss(w, b + h) - loss(w, b - h)) / (2 * h)
    g, gf = np.append(dw, db), np.append(fd, fdb)
    return float(np.linalg.norm(g - gf) / np.linalg.norm(gf))


def test_binarized_backward_matches_finite_differences():
    """training through the soft-binarised iterations; the adjoint of
    sigma(kappa (x - theta(x))) (theta = mean of the positive entries) against central FD."""
    assert _fd_rel_err(O.power_iterate_backward, (2, 3.0, 1.5)) <= 1e-6
    assert _fd_rel_err(O.power_iterate_backward, (0, 2.0, 2.0), K=3) <= 1e-6   # every iteration binarised


@pytest.mark.parametrize("old,new", [
    ("xbar = g - pos * (float(np.sum(g)) / max(int(pos.sum()), 1))", "xbar = g"),   # theta treated as constant
    ("s = xs[k] * (1.0 - xs[k])", "s = xs[k]"),                                        # wrong sigmoid derivative
    ("c = float(np.sum(xn[k] * xbar))", "c = float(np.sum(xs[k] * xbar))"),            # b_k used for x_k
])
def test_binarized_backward_pin_catches_mutations(old, new):
    bad = mutant(OS.power_iterate_backward, old, new)
    assert _fd_rel_err(bad, (2, 3.0, 1.5)) > 1e-4


def test_binarized_backward_euler_identity():
    """Identity combine with b = 0: F is linear in w and the binarised output is scale
    invariant in w (the normalisation precedes the sigmoid), so w . dL/dw = 0."""
    rng = np.random.default_rng(9)
    ch = rng.random((1, 3, 4, 8, 9)) + 0.1
    w = np.array([0.5, 0.2, 0.9])
    gt, gs = O.gaussian_taps(1.0, 2), O.gaussian_taps(1.0, 3)
    dw, _ = O.power_iterate_backward(ch, w, 0.0, 0, gt, gs, 4, rng.normal(size=(1, 4, 8, 9)),
                                     binarize=(1, 4.0, 2.0))
    assert abs(float(np.dot(w, dw))) <= 1e-12 * np.linalg.norm(w) * np.linalg.norm(dw)


# --------------------------------------------------------------------------- f4: Focal-Dice (Eq.12)
def test_focal_dice_values():
    """Eq.12 with the soft Dice (A24): perfect overlap -> 0; disjoint binary frames -> 1 each;
    x = [0.5, 0.5], t = [1, 0] -> D = 2*0.5/2 = 0.5, J = 0.5^0.75 (P:603's 0.75)."""
    t = np.zeros((1, 2, 2, 3))
    t[0, 0, 0, :2] = 1
    t[0, 1, 1, 2] = 1
    J, g = O.focal_dice_loss_grad(t, t)
    assert J == 0.0 and np.abs(g).max() == 0.0
    J, _ = O.focal_dice_loss_grad(1.0 - t, t)
    assert abs(J - 2.0) <= 1e-15
    J, _ = O.focal_dice_loss_grad(np.array([0.5, 0.5]).reshape(1, 1, 1, 2), np.array([1.0, 0.0]).reshape(1, 1, 1, 2))
    assert abs(J - 0.5 ** 0.75) <= 1e-15
    J1, _ = O.focal_dice_loss_grad(np.array([0.5, 0.5]).reshape(1, 1, 1, 2), np.array([1.0, 0.0]).reshape(1, 1, 1, 2),
                                   gamma=1.0)
    assert abs(J1 - 0.5) <= 1e-15   # gamma = 1: the plain Dice loss 1 - D


def _focal_fd_err(lossfn):
    rng = np.random.default_rng(3)
    x = rng.random((2, 3, 4, 5)) * 0.9 + 0.05
    t = (rng.random((2, 3, 4, 5)) > 0.6).astype(np.float64)
    J, g = lossfn(x, t)
    h = 1e-7
    err = 0.0
    for idx in [(0, 0, 0, 0), (1, 2, 3, 4), (0, 1, 2, 3), (1, 0, 1, 1)]:
        xp, xm = x.copy(), x.copy()
        xp[idx] += h
        xm[idx] -= h
        fd = (lossfn(xp, t)[0] - lossfn(xm, t)[0]) / (2 * h)
        err = max(err, abs(fd - g[idx]) / max(abs(fd), 1e-12))
    return err


def test_focal_dice_gradient_matches_finite_differences():
    assert _focal_fd_err(O.focal_dice_loss_grad) <= 1e-6


@pytest.mark.parametrize("old,new", [
    ("2.0 * (ti * den - inter) / (den * den)", "2.0 * ti / den"),          # quotient rule dropped
    ("(1.0 - D) ** (gamma - 1.0)", "(1.0 - D) ** gamma"),                 # focal exponent
])
def test_focal_dice_pin_catches_mutations(old, new):
    assert _focal_fd_err(mutant(OL.focal_dice_loss_grad, old, new)) > 1e-3


# --------------------------------------------------------------------------- f3: online warm start
def _moving_blob(T=9, H=16, W=20):
    rng = np.random.default_rng(11)
    F = np.full((1, T, H, W), 0.1) + 0.02 * rng.random((1, T, H, W))
    for t in range(T):
        F[0, t, 4:10, 2 + 2 * t:7 + 2 * t] = 0.9     # moves 2 px / frame
    return F


def _online_pin(online):
    """q = T - 1, stride 1: two windows [0, T-1) and [1, T).  The second window's x_0
    ("initialize the current solution with the final solution over the previous
    sub-window (for the frames that overlap)") is built here from the first window's
    offline solve: its frames 1..T-2, rescaled to the L2 norm of F there (reading A20),
    and F on the new frame T-1; the online output on frames 1..T-1 must be that window's
    solve from this x_0.  K = 2 keeps the warm start visible in the result."""
    F = _moving_blob()
    T = F.shape[1]
    gt, gs = O.gaussian_taps(1.0, 2), O.gaussian_taps(1.5, 4)
    K = 2
    x_first, _ = O.power_iterate(F[:, :T - 1], gt, gs, K)
    x0 = F[:, 1:].copy()
    ov = x_first[:, 1:]
    x0[:, :T - 2] = ov * (np.linalg.norm(F[:, 1:T - 1]) / np.linalg.norm(ov))
    x_second, _ = O.power_iterate(F[:, 1:], gt, gs, K, x0=x0)
    got = online(F, gt, gs, K, T - 1, 1)
    return (np.abs(got[:, 1:] - x_second).max() <= 1e-12 and
            np.abs(got[:, :1] - x_first[:, :1]).max() <= 1e-12)


def test_online_warm_start_second_window():
    assert _online_pin(O.power_iterate_online)


@pytest.mark.parametrize("old,new", [
    ("xo = px[b, ov0 - ps:ov1 - ps]", "xo = px[b, ov0 - ps + 1:ov1 - ps + 1] if ov1 - ps + 1 <= px.shape[1] "
                                      "else px[b, ov0 - ps - 1:ov1 - ps - 1]"),     # overlap off by one frame
    ("x0[b, :ov1 - ov0] = xo * (nf / nx) if nx > 0 else fo", "x0[b, :ov1 - ov0] = xo"),   # no rescale
    ("x0[b, :ov1 - ov0] = xo * (nf / nx) if nx > 0 else fo", "x0[b, :ov1 - ov0] = xo * (nx / nf)"),  # inverted
])
def test_online_pin_catches_mutations(old, new):
    assert not _online_pin(mutant(OO.power_iterate_online, old, new))
