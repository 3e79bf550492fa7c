"""Pins of the learning-loop oracle (oracle/learn.py)."""
import math

import numpy as np

import oracle as O


def test_adamw_first_step_closed_form():
    """Step 1 of Adam: m_hat = g, v_hat = g^2 -> update = lr * g / (|g| + eps) (sign step), plus
    the decoupled decay w * (1 - lr * wd) (Eq.13)."""
    w = np.array([0.5, -1.0, 2.0])
    g = np.array([0.1, -3.0, 0.0])
    opt = O.AdamW(3, lr=0.01, eps=1e-8, weight_decay=0.1)
    new = opt.step(w, g)
    ref = w * (1 - 0.01 * 0.1) - 0.01 * g / (np.abs(g) + 1e-8)
    assert np.abs(new - ref).max() <= 1e-15


def test_amsgrad_keeps_the_running_max():
    """AMSGrad: the denominator uses max_t v_t, so a small gradient after a large
    one takes a smaller step than plain Adam would."""
    a, b = O.AdamW(1, 0.1, amsgrad=True), O.AdamW(1, 0.1, amsgrad=False)
    p = np.zeros(1)
    for g in (10.0, 0.01, 0.01):
        pa, pb = a.step(p, np.array([g])), b.step(p, np.array([g]))
    assert abs(pa[0]) < abs(pb[0])
    assert a.vmax[0] == max(a.vmax[0], a.v[0]) and a.vmax[0] > a.v[0]


def test_mse_grad_matches_finite_difference():
    rng = np.random.default_rng(0)
    x = rng.random((1, 2, 3, 4))
    m = rng.random((1, 2, 3, 4)) > 0.5
    L, g = O.mse_loss_grad(x, m)
    h = 1e-6
    for idx in [(0, 0, 0, 0), (0, 1, 2, 3), (0, 1, 0, 2)]:
        xp, xm = x.copy(), x.copy()
        xp[idx] += h
        xm[idx] -= h
        fd = (O.mse_loss_grad(xp, m)[0] - O.mse_loss_grad(xm, m)[0]) / (2 * h)
        assert abs(fd - g[idx]) <= 1e-8


def test_training_reduces_the_loss_and_prefers_clean_channels():
    """Fig. learned_weights: learning favours clean, strong channels.  Three
    channels = clean mask + increasing noise; after training the clean channel has the
    largest weight and the loss has gone down."""
    rng = np.random.default_rng(1)
    T, H, W = 4, 12, 14
    m = np.zeros((1, T, H, W), bool)
    m[:, :, 3:9, 4:10] = True
    base = m.astype(np.float64)
    ch = np.stack([base, np.clip(base + rng.normal(0, 0.3, base.shape), 0, 1),
                   np.clip(rng.random(base.shape), 0, 1)], axis=1)
    gt, gs = O.gaussian_taps(1.0, 2), O.gaussian_taps(1.0, 3)
    w, b, losses = O.train(ch, m, [0.3, 0.3, 0.3], 0.0, 0, gt, gs, 4, 25, 0.05)
    assert losses[-1] < losses[0]
    assert w[0] > w[1] > w[2]
