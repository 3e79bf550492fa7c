"""GPU parity of the full SFSeg operator against the f64 oracle.

sfseg_power_iterate_full (Eq.7 / Eq.10 with unary exponent p, pairwise map F and
alpha; Eq.9 for both maps) vs oracle.power_iterate_full.  Tolerances as the hot
path: x_K relative L2 <= 1e-4, per-iteration norms / gains <= 1e-5 relative.
"""
import numpy as np
import pytest

import oracle as O
import workloads as WL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

X_TOL = 1e-4
NU_TOL = 1e-5


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


def _check(sf, s_ch, ws, f_ch, wf, p, alpha, sig_t, sig_s, r_t, r_s, K, bs=0.0, act_s=0, bf=0.0, act_f=0, x0=None):
    dev = torch.device("cuda")
    B, Cs, T, H, W = s_ch.shape
    Cf = f_ch.shape[1]
    solver = sf.FullSolver((B, T, H, W), Cs, Cf, sf.Gauss(sig_t, sig_s, r_t, r_s), K)
    x0t = None if x0 is None else torch.from_numpy(np.ascontiguousarray(x0, np.float32)).to(dev)
    xg = solver.forward(torch.from_numpy(np.ascontiguousarray(s_ch)).to(dev), ws,
                        torch.from_numpy(np.ascontiguousarray(f_ch)).to(dev), wf, p, alpha, bs, act_s, bf, act_f,
                        x0=x0t).cpu().numpy()
    stg = solver.stats.cpu().numpy()
    S, U, F = O.combine_full(s_ch, ws, bs, act_s, f_ch, wf, bf, act_f, p)
    gt, gs = O.gaussian_taps(sig_t, r_t), O.gaussian_taps(sig_s, r_s)
    xo, sto = O.power_iterate_full(S, U, F, alpha, gt, gs, K, x0=None if x0 is None else np.asarray(x0, np.float64))
    assert np.isfinite(xg).all()
    for b in range(B):
        assert _rel(xg[b], xo[b]) <= X_TOL, f"volume {b}: x rel err {_rel(xg[b], xo[b]):.3e}"
        assert abs(np.linalg.norm(xg[b].astype(np.float64)) - 1.0) < 1e-5
    np.testing.assert_allclose(stg[..., 0], sto["nu"], rtol=NU_TOL)
    np.testing.assert_allclose(stg[..., 1], sto["gain"], rtol=NU_TOL)
    return xg, xo


@pytest.mark.parametrize("shape,radii,p,alpha", [
    ((1, 6, 40, 70), (2, 6), 0.2, 1.0),
    ((2, 5, 33, 150), (1, 3), 0.1, 0.8),     # B > 1, ragged strips / blocks, small radii
    ((1, 9, 70, 130), (6, 24), 1.0, 1.0),    # config-2 radii across several strips
    ((2, 5, 40, 150), (3, 9), 0.5, 1.2),     # B > 1 on the tensor-core plan (fused combination)
])
def test_full_random(sf, shape, radii, p, alpha):
    B, T, H, W = shape
    rng = np.random.default_rng(sum(shape))
    s_ch = (rng.random((B, 1, T, H, W)) * 0.9 + 0.05).astype(np.float32)
    f_ch = rng.random((B, 1, T, H, W)).astype(np.float32)
    r_t, r_s = radii
    _check(sf, s_ch, [1.0], f_ch, [1.0], p, alpha, max(r_t, 1) / 3.0, max(r_s, 1) / 3.0, r_t, r_s, 6)


def test_full_multichannel_sigmoid_and_x0(sf):
    """SFSeg++ form: both maps by the sigmoid combine of Eq.9, a user x0."""
    rng = np.random.default_rng(7)
    s_ch = rng.normal(size=(1, 3, 6, 36, 90)).astype(np.float32)
    f_ch = rng.normal(size=(1, 2, 6, 36, 90)).astype(np.float32)
    x0 = rng.random((1, 6, 36, 90)).astype(np.float32)
    _check(sf, s_ch, [0.7, -0.4, 0.9], f_ch, [1.1, 0.6], 0.3, 1.0, 1.0, 3.0, 3, 9, 5, bs=0.2, act_s=1, bf=-0.1,
           act_f=1, x0=x0)


def test_full_c2f_recipe_crop(sf):
    cfg = WL.get_config("c2f", T=12, H=100, W=220)
    wl = WL.generate("c2f", cfg=cfg)
    e = wl.extra
    _check(sf, wl.ch, wl.w, e["f_ch"], e["wf"], e["p"], e["alpha"], cfg.sigma_t, cfg.sigma_s, cfg.radius_t,
           cfg.radius_s, cfg.K)


def test_full_reduces_to_hot_path_gpu(sf):
    """F == 0, p = 1, alpha = 1: the full operator is the hot path's M = D_S G D_S."""
    rng = np.random.default_rng(9)
    s_ch = (rng.random((1, 1, 8, 50, 120)) * 0.8 + 0.1).astype(np.float32)
    f_ch = np.zeros_like(s_ch)
    dev = torch.device("cuda")
    g = sf.Gauss(1.0, 3.0, 3, 9)
    xf = sf.FullSolver((1, 8, 50, 120), 1, 1, g, 5).forward(torch.from_numpy(s_ch).to(dev), [1.0],
                                                             torch.from_numpy(f_ch).to(dev), [1.0], 1.0, 1.0)
    xh = sf.Solver((1, 8, 50, 120), 1, g, 5).forward(torch.from_numpy(s_ch).to(dev), [1.0])
    assert _rel(xf.cpu().numpy(), xh.cpu().numpy()) <= 1e-5


def test_full_invalid_arguments(sf):
    dev = torch.device("cuda")
    s = torch.rand((1, 1, 4, 16, 16), device=dev)
    solver = sf.FullSolver((1, 4, 16, 16), 1, 1, sf.Gauss(1.0, 1.0, 3, 3), 2)
    for p, alpha in ((0.0, 1.0), (-1.0, 1.0), (1.0, 0.0), (float("nan"), 1.0)):
        with pytest.raises(RuntimeError):
            solver.forward(s, [1.0], s, [1.0], p, alpha)


# --------------------------------------------------------------------------- row f2
@pytest.mark.parametrize("n_cont,K", [(3, 6), (0, 3), (5, 5)])
def test_full_soft_binarisation(sf, n_cont, K):
    """Alg.1 STEP 3: soft-binarisation after n_cont continuous iterations (reading A21).
    Output values in (0,1) when K > n_cont; per-iteration norms and gains (the gain after a
    binarised iteration uses ||x_k|| of the binarised iterate) match the oracle."""
    rng = np.random.default_rng(13 + n_cont)
    B, T, H, W = 2, 6, 40, 90
    s_ch = (rng.random((B, 1, T, H, W)) * 0.9 + 0.05).astype(np.float32)
    f_ch = rng.random((B, 1, T, H, W)).astype(np.float32)
    dev = torch.device("cuda")
    g = sf.Gauss(1.0, 3.0, 3, 9)
    solver = sf.FullSolver((B, T, H, W), 1, 1, g, K)
    xg = solver.forward(torch.from_numpy(s_ch).to(dev), [1.0], torch.from_numpy(f_ch).to(dev), [1.0], 0.5, 1.0,
                        binarize=(n_cont, 4.0, 2.0)).cpu().numpy()
    S, U, F = O.combine_full(s_ch, [1.0], 0.0, 0, f_ch, [1.0], 0.0, 0, 0.5)
    xo, sto = O.power_iterate_full(S, U, F, 1.0, O.gaussian_taps(1.0, 3), O.gaussian_taps(3.0, 9), K,
                                   binarize=(n_cont, 4.0, 2.0))
    for b in range(B):
        assert _rel(xg[b], xo[b]) <= X_TOL, f"volume {b}: rel err {_rel(xg[b], xo[b]):.3e}"
    stg = solver.stats.cpu().numpy()
    np.testing.assert_allclose(stg[..., 0], sto["nu"], rtol=NU_TOL)
    np.testing.assert_allclose(stg[..., 1], sto["gain"], rtol=NU_TOL)
    if K > n_cont:
        assert xg.min() > 0.0 and xg.max() < 1.0
        mask = sf.threshold(torch.from_numpy(xg).to(dev), 0.5, sf.THR_ABSOLUTE).cpu().numpy()
        ref = O.threshold(xo, 0.5, O.THR_ABSOLUTE)
        band = np.abs(xo - 0.5) > 1e-4
        assert (mask[band] == ref[band]).all()
