"""The tcgen05 / TMEM spatial pass (spass_tc6.cuh: UTCHMMA with dense-rate shapes, x-pass
operands from the TMA box of the fp16 planes the temporal pass writes, y-pass A operand in
tensor memory) against the f64 oracle: every compiled radius, ragged strips (128-column
strips: W not a multiple of 128) and 64-row blocks, B > 1, H = 1, segments spanning many
x-blocks (more units than CTAs), the Rayleigh / tape epilogue, and the backward of a
tcgen05 forward (plain mma.sync pass)."""
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


def _solve(sf, ch, w, g, K, rayleigh=False):
    B, C, T, H, W = ch.shape
    s = sf.Solver((B, T, H, W), C, g, K, algo=sf.ALGO_TWO_PASS_TCGEN05)
    x = s.forward(torch.from_numpy(ch).cuda(), w, want_rayleigh=rayleigh).cpu().numpy()
    return x, s.stats.cpu().numpy()


@pytest.mark.parametrize("r_s,shape", [
    (24, (1, 6, 70, 300)),     # 3 strips (128 + 128 + 44), ragged 64-row blocks
    (8, (2, 5, 33, 130)),      # B = 2, two columns in the last strip
    (9, (1, 4, 40, 129)),      # one live column in the last strip
    (12, (1, 3, 97, 71)),      # W < one strip
    (16, (1, 3, 128, 256)),    # exact strips and blocks
    (18, (2, 4, 200, 170)),
    (24, (1, 2, 1, 300)),      # H = 1
    (24, (1, 1, 5, 5)),        # tiny: pure padding around one partial block
    (24, (1, 20, 480, 260)),   # 960 units > 148 CTAs: segments of several y-blocks, Q ring wraps
    (32, (1, 3, 150, 300)),    # 12 x-pass k steps (three full boxes)
    (36, (1, 3, 150, 300)),    # c5's radius: four TMA boxes, chunk origin 64 rows above the segment
    (36, (2, 12, 300, 200)),   # r_s = 36 with many units per CTA (segments of several y-blocks)
])
def test_tcgen05_spatial_radii(sf, r_s, shape):
    B, T, H, W = shape
    rng = np.random.default_rng(100 + r_s)
    ch = (rng.random((B, 1, T, H, W)) * 0.8 + 0.1).astype(np.float32)
    g = sf.Gauss(1.0, r_s / 3.0, 2, r_s)
    assert sf.forward_path((B, T, H, W), g, sf.ALGO_TWO_PASS_TCGEN05)[0] == sf.PATH_TWO_PASS_TCGEN05
    x, st = _solve(sf, ch, [1.0], g, 5, rayleigh=True)
    F, _ = O.combine(ch, [1.0])
    xo, sto = O.power_iterate(F, O.gaussian_taps(1.0, 2), O.gaussian_taps(r_s / 3.0, r_s), 5)
    for b in range(B):
        assert _rel(x[b], xo[b]) <= 1e-6, _rel(x[b], xo[b])
        assert _frame_err(x[b], xo[b]) <= 1e-5
    np.testing.assert_allclose(st[..., 0], sto["nu"], rtol=1e-6)
    np.testing.assert_allclose(st[..., 2], sto["rho"], rtol=1e-6)


def test_tcgen05_c2_crop_and_backward(sf):
    """c2 recipe crop (several strips, ragged) forward; c3 crop backward (plain tcgen05 pass +
    streaming epilogue) against the oracle's dL/dw."""
    wl = WL.generate("c2", cfg=WL.get_config("c2", T=16, H=150, W=300))
    x, _ = _solve(sf, wl.ch, wl.w, sf.Gauss(2.0, 8.0, 6, 24), 15)
    F, _ = O.combine(wl.ch, wl.w)
    xo, _ = O.power_iterate(F, O.gaussian_taps(2.0, 6), O.gaussian_taps(8.0, 24), 15)
    assert _rel(x, xo) <= 1e-6 and _frame_err(x[0], xo[0]) <= 1e-5
    wl = WL.generate("c3", cfg=WL.get_config("c3", T=12, H=72, W=150))
    w = np.array([0.5, -0.3, 0.8, 0.1, 0.6, -0.2], np.float32)
    B, C, T, H, W = wl.ch.shape
    K = 8
    g = sf.Gauss(2.0, 8.0, 6, 24)
    s = sf.Solver((B, T, H, W), C, g, K, want_tape=True, algo=sf.ALGO_TWO_PASS_TCGEN05)
    cht = torch.from_numpy(wl.ch).cuda()
    s.forward(cht, w, 0.2, 1)
    rng = np.random.default_rng(0)
    gr = rng.normal(size=(B, T, H, W)).astype(np.float32)
    dw, db = s.backward(cht, w, torch.from_numpy(gr).cuda(), 0.2, 1)
    dwo, dbo = O.power_iterate_backward(wl.ch, w, 0.2, 1, O.gaussian_taps(2.0, 6), O.gaussian_taps(8.0, 24), K,
                                        gr.astype(np.float64))
    assert _rel(dw, dwo) <= 1e-3


def test_tcgen05_deterministic(sf):
    wl = WL.generate("c2", cfg=WL.get_config("c2", T=8, H=96, W=240))
    a, _ = _solve(sf, wl.ch, wl.w, sf.Gauss(2.0, 8.0, 6, 24), 6)
    b, _ = _solve(sf, wl.ch, wl.w, sf.Gauss(2.0, 8.0, 6, 24), 6)
    assert np.array_equal(a, b)
