"""GPU parity of SURVEY.md §8(f) rows f2 (soft-binarisation on the hot path, forward and
backward through it) and f4 (Focal-Dice loss on the device, training through the binarised
iterations) against the f64 oracle (tests/test_oracle_binarize_learn.py pins the oracle)."""
import numpy as np
import pytest

import oracle as O
import workloads as WL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2212_08058_b200 as m
    m.lib()
    return m


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


# steepness scaled to the unit-norm iterate (theta ~ N^-1/2): kappa0 * theta ~ 2
def _kappa0(shape):
    return 2.0 * np.sqrt(np.prod(shape))


@pytest.mark.parametrize("radii,algo", [((6, 24), "auto"), ((3, 6), "auto"), ((6, 24), "fp32")])
def test_binarized_forward_matches_oracle(sf, radii, algo):
    r_t, r_s = radii
    wl = WL.generate("c3", cfg=WL.get_config("c3", T=10, H=60, W=140))
    B, C, T, H, W = wl.ch.shape
    bz = (3, _kappa0((T, H, W)), 1.5)
    K = 6
    g = sf.Gauss(max(r_t, 1) / 3.0, r_s / 3.0, r_t, r_s)
    s = sf.Solver((B, T, H, W), C, g, K, binarize=bz,
                  algo=sf.ALGO_TWO_PASS_FP32 if algo == "fp32" else sf.ALGO_AUTO)
    x = s.forward(torch.from_numpy(wl.ch).cuda(), wl.w).cpu().numpy()
    F, _ = O.combine(wl.ch, wl.w)
    xo, sto = O.power_iterate(F, O.gaussian_taps(g.sigma_t, r_t), O.gaussian_taps(g.sigma_s, r_s), K, binarize=bz)
    assert 0.0 < x.min() and x.max() < 1.0
    assert np.abs(x - xo).max() <= 1e-4, np.abs(x - xo).max()
    assert _rel(x, xo) <= 1e-5
    np.testing.assert_allclose(s.stats.cpu().numpy()[..., 1], sto["gain"], rtol=1e-5)


@pytest.mark.parametrize("radii,act", [((6, 24), 1), ((3, 6), 1), ((6, 24), 0)])
def test_binarized_backward_focal_dice_matches_oracle(sf, radii, act):
    """dL/dw through the soft-binarised iterations for the Focal-Dice loss (Eq.12) computed on
    the device, against the oracle's loss and adjoint (both f64-pinned)."""
    r_t, r_s = radii
    wl = WL.generate("c3", cfg=WL.get_config("c3", T=8, H=56, W=120))
    B, C, T, H, W = wl.ch.shape
    w = wl.w if act == 0 else np.array([0.5, -0.3, 0.8, 0.1, 0.6, -0.2], np.float32)
    b = 0.0 if act == 0 else 0.2
    bz = (2, _kappa0((T, H, W)), 1.5)
    K = 5
    g = sf.Gauss(max(r_t, 1) / 3.0, r_s / 3.0, r_t, r_s)
    gt, gs = O.gaussian_taps(g.sigma_t, r_t), O.gaussian_taps(g.sigma_s, r_s)
    dev = torch.device("cuda")
    s = sf.Solver((B, T, H, W), C, g, K, want_tape=True, binarize=bz)
    cht = torch.from_numpy(wl.ch).to(dev)
    x = s.forward(cht, w, b, act)
    fd = sf.FocalDice((B, T, H, W))
    mask = torch.from_numpy(wl.mask.astype(np.uint8)).to(dev)
    L, grad = fd(x, mask)
    F, _ = O.combine(wl.ch, w, b, act)
    xo, _ = O.power_iterate(F, gt, gs, K, binarize=bz)
    Lo, go = O.focal_dice_loss_grad(xo, wl.mask)
    assert abs(float(L.item()) - Lo) <= 1e-5 * max(1.0, abs(Lo))
    # the device loss gradient of the device x, against the oracle's Eq.12 gradient of the same x
    Lx, gx = O.focal_dice_loss_grad(x.cpu().numpy(), wl.mask)
    assert _rel(grad.cpu().numpy(), gx) <= 1e-5
    dw, db = s.backward(cht, w, grad, b, act)
    dwo, dbo = O.power_iterate_backward(wl.ch, w, b, act, gt, gs, K, go, binarize=bz)
    assert _rel(dw, dwo) <= 1e-3, (dw, dwo)
    assert abs(db - dbo) <= 1e-3 * max(abs(dbo), np.abs(dwo).max())
    if act == 0:   # scale invariance survives the binarisation (oracle pin): w . dL/dw = 0
        assert abs(float(np.dot(w, dw))) <= 1e-3 * np.linalg.norm(w) * np.linalg.norm(dw)


def test_focal_dice_kernel_edge_frames(sf):
    """Empty frames (no mask, x = 0) contribute nothing; a perfect frame has loss 0 and zero
    gradient; ragged H*W (not a multiple of 4)."""
    rng = np.random.default_rng(2)
    x = rng.random((2, 3, 7, 9)).astype(np.float32)
    t = (rng.random((2, 3, 7, 9)) > 0.5).astype(np.uint8)
    x[0, 1] = 0.0
    t[0, 1] = 0
    x[1, 2] = t[1, 2]
    fd = sf.FocalDice(x.shape)
    L, g = fd(torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda())
    Lo, go = O.focal_dice_loss_grad(x, t)
    assert abs(float(L.item()) - Lo) <= 1e-12 * max(1.0, Lo)
    gg = g.cpu().numpy()
    assert np.abs(gg[0, 1]).max() == 0.0 and np.abs(gg[1, 2]).max() == 0.0
    np.testing.assert_allclose(gg, go, rtol=1e-6, atol=1e-9)


def test_train_focal_dice_through_binarisation(sf):
    """f4 end to end on the device (forward with binarisation + Focal-Dice + backward + AdamW)
    against the oracle's loop (same losses and weights), and the learned ordering of Fig.
    learned_weights: clean > noisy > random channel."""
    rng = np.random.default_rng(1)
    T, H, W = 6, 40, 60
    m = np.zeros((1, T, H, W), bool)
    m[:, :, 10:28, 15:40] = True
    base = m.astype(np.float32)
    ch = np.stack([base, np.clip(base + rng.normal(0, 0.3, base.shape), 0, 1),
                   rng.random(base.shape)], axis=1).astype(np.float32)
    g = sf.Gauss(1.0, 2.0, 3, 6)
    bz = (2, _kappa0((T, H, W)), 1.5)
    dev = torch.device("cuda")
    w_g, b_g, l_g = sf.train_weights(torch.from_numpy(ch).to(dev), torch.from_numpy(m).to(dev), [0.3, 0.3, 0.3], 0.0,
                                     1, g, 5, 12, 0.05, loss="focal_dice", binarize=bz)
    w_o, b_o, l_o = O.train(ch, m, [0.3, 0.3, 0.3], 0.0, 1, O.gaussian_taps(1.0, 3), O.gaussian_taps(2.0, 6), 5, 12,
                            0.05, loss="focal_dice", binarize=bz)
    np.testing.assert_allclose(l_g, l_o, rtol=1e-4)
    np.testing.assert_allclose(w_g, w_o, rtol=0, atol=1e-4)
    assert l_g[-1] < l_g[0]
    assert w_g[0] > w_g[1] > w_g[2]
