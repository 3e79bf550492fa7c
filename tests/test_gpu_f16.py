"""The two-plane fp16 spatial pass (SFSEG_ALGO_TWO_PASS_MMA_F16; spass_tc.cuh FMT = 1,
DESIGN.md reading A25): three products per tap, per-volume power-of-two range scaling from
the temporal pass's max |v| (SC_VMAX).  Against the f64 oracle: every compiled radius,
ragged strips / blocks, B > 1 with volumes 12 orders of magnitude apart (the per-volume
scale), the Rayleigh / tape epilogue and the backward on its tape, soft-binarised
iterations, time slabs, and its error next to the FP32-FMA pass's on a c2 crop."""
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


def _frame_err(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    d = np.abs(a - b).reshape(b.shape[0], -1).max(-1)
    m = np.abs(b).reshape(b.shape[0], -1).max(-1)
    ok = m > 0
    return float((d[ok] / m[ok]).max())


def _solve(sf, ch, w, g, K, rayleigh=False, algo=None, **kw):
    B, C, T, H, W = ch.shape
    s = sf.Solver((B, T, H, W), C, g, K, algo=sf.ALGO_TWO_PASS_MMA_F16 if algo is None else algo, **kw)
    x = s.forward(torch.from_numpy(ch).cuda(), w, want_rayleigh=rayleigh).cpu().numpy()
    return x, s.stats.cpu().numpy()


@pytest.mark.parametrize("r_s,shape", [
    (24, (1, 6, 70, 300)),     # 3 strips (128 + 128 + 44), ragged 32-row blocks
    (8, (2, 5, 33, 130)),
    (9, (1, 4, 40, 81)),
    (12, (1, 3, 97, 71)),
    (16, (1, 3, 64, 128)),
    (18, (2, 4, 50, 170)),
    (32, (1, 3, 80, 200)),
    (36, (1, 2, 90, 140)),
    (48, (1, 2, 100, 260)),
    (24, (1, 2, 1, 300)),      # H = 1
    (24, (1, 1, 5, 5)),        # tiny
])
def test_f16_spatial_radii(sf, r_s, shape):
    B, T, H, W = shape
    rng = np.random.default_rng(200 + r_s)
    ch = (rng.random((B, 1, T, H, W)) * 0.8 + 0.1).astype(np.float32)
    g = sf.Gauss(1.0, r_s / 3.0, 2, r_s)
    assert sf.forward_path((B, T, H, W), g, sf.ALGO_TWO_PASS_MMA_F16)[0] == sf.PATH_TWO_PASS_TC_F16
    x, st = _solve(sf, ch, [1.0], g, 5, rayleigh=True)
    F, _ = O.combine(ch, [1.0])
    xo, sto = O.power_iterate(F, O.gaussian_taps(1.0, 2), O.gaussian_taps(r_s / 3.0, r_s), 5)
    for b in range(B):
        assert _rel(x[b], xo[b]) <= 1e-6, _rel(x[b], xo[b])
        assert _frame_err(x[b], xo[b]) <= 1e-5
    np.testing.assert_allclose(st[..., 0], sto["nu"], rtol=1e-6)
    np.testing.assert_allclose(st[..., 2], sto["rho"], rtol=1e-6)


def test_f16_per_volume_scale(sf):
    """Volumes of one batch 1e-6 and 1e+6 in magnitude: each is scaled into fp16's range on
    its own (fp16 itself spans 2^-24 .. 65504), and x_0 = a user iterate with a third scale."""
    rng = np.random.default_rng(7)
    B, T, H, W = 3, 5, 60, 150
    ch = (rng.random((B, 1, T, H, W)) * 0.8 + 0.1)
    ch[0] *= 1e-6
    ch[2] *= 1e6
    ch = ch.astype(np.float32)
    x0 = (rng.random((B, T, H, W)) * 1e3).astype(np.float32)
    g = sf.Gauss(2.0, 8.0, 6, 24)
    s = sf.Solver((B, T, H, W), 1, g, 6, algo=sf.ALGO_TWO_PASS_MMA_F16)
    x = s.forward(torch.from_numpy(ch).cuda(), [1.0], x0=torch.from_numpy(x0).cuda()).cpu().numpy()
    F, _ = O.combine(ch, [1.0])
    xo, sto = O.power_iterate(F, O.gaussian_taps(2.0, 6), O.gaussian_taps(8.0, 24), 6, x0=x0)
    for b in range(B):
        assert _rel(x[b], xo[b]) <= 1e-6 and _frame_err(x[b], xo[b]) <= 1e-5, b
    np.testing.assert_allclose(s.stats.cpu().numpy()[..., 1], sto["gain"], rtol=1e-5)


def test_f16_c2_crop_error_vs_fp32_and_backward(sf):
    """c2 recipe crop: the fp16 pass's x_K error is within 2x the FP32-FMA pass's (the
    fp32-class bar of reading A23); c3 crop backward on the fp16 forward's tape."""
    wl = WL.generate("c2", cfg=WL.get_config("c2", T=16, H=150, W=300))
    g = sf.Gauss(2.0, 8.0, 6, 24)
    F, _ = O.combine(wl.ch, wl.w)
    xo, _ = O.power_iterate(F, O.gaussian_taps(2.0, 6), O.gaussian_taps(8.0, 24), 15)
    x16, _ = _solve(sf, wl.ch, wl.w, g, 15)
    x32, _ = _solve(sf, wl.ch, wl.w, g, 15, algo=sf.ALGO_TWO_PASS_FP32)
    e16, e32 = _rel(x16, xo), _rel(x32, xo)
    assert e16 <= 2.0 * e32 + 1e-9, (e16, e32)
    assert _frame_err(x16[0], xo[0]) <= 1e-5
    wl = WL.generate("c3", cfg=WL.get_config("c3", T=12, H=72, W=150))
    w = np.array([0.5, -0.3, 0.8, 0.1, 0.6, -0.2], np.float32)
    B, C, T, H, W = wl.ch.shape
    K = 8
    s = sf.Solver((B, T, H, W), C, g, K, want_tape=True, algo=sf.ALGO_TWO_PASS_MMA_F16)
    cht = torch.from_numpy(wl.ch).cuda()
    s.forward(cht, w, 0.2, 1, want_rayleigh=True)
    gr = np.random.default_rng(0).normal(size=(B, T, H, W)).astype(np.float32)
    dw, db = s.backward(cht, w, torch.from_numpy(gr).cuda(), 0.2, 1)
    dwo, dbo = O.power_iterate_backward(wl.ch, w, 0.2, 1, O.gaussian_taps(2.0, 6), O.gaussian_taps(8.0, 24), K,
                                        gr.astype(np.float64))
    assert _rel(dw, dwo) <= 1e-3


def test_f16_binarized(sf):
    """Soft-binarised iterations (row f2): the binarised iterate (values in (0,1), scale 1)
    feeds the next temporal pass, whose max |v| re-ranges the fp16 pass."""
    wl = WL.generate("c3", cfg=WL.get_config("c3", T=10, H=60, W=140))
    B, C, T, H, W = wl.ch.shape
    g = sf.Gauss(2.0, 8.0, 6, 24)
    bz = (3, 2.0 * np.sqrt(T * H * W), 1.5)   # kappa0 * theta ~ 2 (tests/test_gpu_binarize.py)
    x, _ = _solve(sf, wl.ch, wl.w, g, 6, binarize=bz)
    F, _ = O.combine(wl.ch, wl.w)
    xo, _ = O.power_iterate(F, O.gaussian_taps(2.0, 6), O.gaussian_taps(8.0, 24), 6, binarize=bz)
    assert 0.0 < x.min() and x.max() < 1.0
    assert np.abs(x - xo).max() <= 1e-4
    assert _rel(x, xo) <= 1e-5


def test_f16_slabs(sf):
    cfg = WL.get_config("c2", T=26, H=70, W=150)
    wl = WL.generate("c2", cfg=cfg)
    g = sf.Gauss(2.0, 8.0, 6, 24)
    ch = torch.from_numpy(wl.ch).cuda()
    xs, _ = sf.power_iterate_slabs(ch, wl.w, g, 6, 3, algo=sf.ALGO_TWO_PASS_MMA_F16)[:2]
    F, _ = O.combine(wl.ch, wl.w)
    xo, _ = O.power_iterate(F, O.gaussian_taps(2.0, 6), O.gaussian_taps(8.0, 24), 6)
    assert _rel(xs.cpu().numpy(), xo) <= 1e-6


def test_f16_deterministic(sf):
    wl = WL.generate("c2", cfg=WL.get_config("c2", T=8, H=96, W=240))
    a, _ = _solve(sf, wl.ch, wl.w, sf.Gauss(2.0, 8.0, 6, 24), 6)
    b, _ = _solve(sf, wl.ch, wl.w, sf.Gauss(2.0, 8.0, 6, 24), 6)
    assert np.array_equal(a, b)


def test_f16_wide_dynamic_range(sf):
    """Entries spread over 20 decades inside one volume (log-uniform F): the power-of-two
    range scaling keeps the large entries exact to 2^-22 and the entries below ~2^-24 of the
    volume's max lose relative precision only (A25); the L2 and per-frame criteria hold, and
    the error stays within 2x the FP32-FMA pass's."""
    rng = np.random.default_rng(11)
    B, T, H, W = 1, 6, 64, 150
    ch = (10.0 ** rng.uniform(-20, 0, size=(B, 1, T, H, W))).astype(np.float32)
    g = sf.Gauss(2.0, 8.0, 6, 24)
    F, _ = O.combine(ch, [1.0])
    xo, sto = O.power_iterate(F, O.gaussian_taps(2.0, 6), O.gaussian_taps(8.0, 24), 6)
    x16, st16 = _solve(sf, ch, [1.0], g, 6)
    x32, _ = _solve(sf, ch, [1.0], g, 6, algo=sf.ALGO_TWO_PASS_FP32)
    assert np.isfinite(x16).all()
    e16, e32 = _rel(x16, xo), _rel(x32, xo)
    assert e16 <= 1e-6 and e16 <= 2.0 * e32 + 1e-9, (e16, e32)
    assert _frame_err(x16[0], xo[0]) <= 1e-5
    np.testing.assert_allclose(st16[..., 1], sto["gain"], rtol=1e-5)
