"""Full BASELINE.json sizes in the launch configuration bench.py times, against the
multi-process f64 oracle (oracle/parallel.py: the serial oracle split into independent
pieces, bitwise equal to it -- tests/test_oracle_parallel.py).  Elementwise bounds: the
volume-wide relative L2 (north star: 1e-4) AND a per-frame bound max|x - x_orc| / max|x_orc|
per frame (<= 1e-4), so a local error in one strip, border frame or ragged tail is caught.
The tensor-core spatial pass (six bf16 products, A23) must stay within 2x of
the FP32-FMA pass's own error against the oracle (fp32-class arithmetic)."""
import numpy as np
import pytest

import oracle as O
from oracle import parallel as OP
import workloads as WL

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

X_TOL = 1e-4
FRAME_TOL = 1e-4
G_TOL = 1e-3


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


def _taps(c):
    return O.gaussian_taps(c.sigma_t, c.radius_t), O.gaussian_taps(c.sigma_s, c.radius_s)


def _gauss(sf, c):
    return sf.Gauss(c.sigma_t, c.sigma_s, c.radius_t, c.radius_s)


@pytest.fixture(scope="module")
def c2(sf):
    wl = WL.generate("c2")
    c = wl.cfg
    F, _ = O.combine(wl.ch, wl.w)
    xo, sto = OP.power_iterate(F, *_taps(c), c.K)
    return wl, xo, sto


def test_c2_full_size_tensor_core_and_fp32(sf, c2):
    """configs[1], every spatial pass, at 1x70x480x854: rel L2, per-frame bound, gains, and
    every tensor-core pass's error <= 2x the FP32-FMA path's (the default tcgen05 pass and the
    mma.sync fp16 pass: two fp16 planes; the mma.sync bf16 pass: three planes; measured
    round 2: fp16 mma.sync 2.1e-7, bf16 1.8e-7, FP32-FMA 1.25e-7; profiles/f16a/precision.json)."""
    wl, xo, sto = c2
    c = wl.cfg
    ch = torch.from_numpy(wl.ch).cuda()
    errs = {}
    for algo in (sf.ALGO_AUTO, sf.ALGO_TWO_PASS_MMA_F16, sf.ALGO_TWO_PASS_MMA_SYNC, sf.ALGO_TWO_PASS_FP32):
        s = sf.Solver((c.B, c.T, c.H, c.W), c.C, _gauss(sf, c), c.K, algo=algo)
        x = s.forward(ch, wl.w).cpu().numpy()
        st = s.stats.cpu().numpy()
        for b in range(c.B):
            assert _rel(x[b], xo[b]) <= X_TOL
            assert _frame_err(x[b], xo[b]) <= FRAME_TOL
        np.testing.assert_allclose(st[..., 1], sto["gain"], rtol=1e-5)
        assert (x >= 0).all()
        errs[algo] = _rel(x, xo)
    assert errs[sf.ALGO_AUTO] <= 2.0 * errs[sf.ALGO_TWO_PASS_FP32] + 1e-8, errs
    assert errs[sf.ALGO_TWO_PASS_MMA_SYNC] <= 2.0 * errs[sf.ALGO_TWO_PASS_FP32] + 1e-8, errs
    assert errs[sf.ALGO_TWO_PASS_MMA_F16] <= 2.0 * errs[sf.ALGO_TWO_PASS_FP32] + 1e-8, errs


def test_c2_full_size_masks(sf, c2):
    """The per-frame threshold (tau = 0.5, reading A12) at full size: bit-exact wherever the
    oracle's rescaled value is farther than 1e-4 from tau."""
    wl, xo, _ = c2
    c = wl.cfg
    s = sf.Solver((c.B, c.T, c.H, c.W), c.C, _gauss(sf, c), c.K)
    x = s.forward(torch.from_numpy(wl.ch).cuda(), wl.w)
    mg = s.threshold(x, c.tau).cpu().numpy()
    mo = O.threshold(xo, c.tau)
    xhat = xo / xo.max(axis=(2, 3), keepdims=True)
    far = np.abs(xhat - c.tau) > 1e-4
    assert far.mean() > 0.99
    assert (mg[far] == mo[far]).all()


def test_combine_and_F_out_vs_oracle(sf):
    """sfseg_combine_channels and the solve's F_out against oracle.combine (Eq.9) on the full
    c3 ensemble (C = 6) and a sigmoid combine with bias."""
    wl = WL.generate("c3", with_mask=False)
    c = wl.cfg
    ch = torch.from_numpy(wl.ch).cuda()
    Fo, _ = O.combine(wl.ch, wl.w)
    F = sf.combine_channels(ch, wl.w).cpu().numpy()
    assert np.abs(F - Fo).max() <= 1e-6 * np.abs(Fo).max()
    w2, b2 = np.array([0.5, -0.3, 0.8, 0.1, 0.6, -0.2], np.float32), 0.2
    Fo2, _ = O.combine(wl.ch, w2, b2, O.ACT_SIGMOID)
    F2 = sf.combine_channels(ch, w2, b2, sf.ACT_SIGMOID).cpu().numpy()
    assert np.abs(F2 - Fo2).max() <= 1e-6
    s = sf.Solver((c.B, c.T, c.H, c.W), c.C, _gauss(sf, c), 2)
    F_out = torch.empty((c.B, c.T, c.H, c.W), dtype=torch.float32, device="cuda")
    s.forward(ch, w2, b2, sf.ACT_SIGMOID, F_out=F_out)
    assert np.abs(F_out.cpu().numpy() - Fo2).max() <= 1e-6


def test_c3_full_size_forward_backward(sf):
    """configs[2] at full size (1x6x70x480x854): forward x_K and dL/dw (MSE of reading A13)
    through the 15 unrolled iterations, against the multi-process oracle backward."""
    wl = WL.generate("c3")
    c = wl.cfg
    gt, gs = _taps(c)
    F, _ = O.combine(wl.ch, wl.w)
    xo, _ = OP.power_iterate(F, gt, gs, c.K)
    m = wl.mask.astype(np.float64)
    g = (2.0 * (xo - m / np.linalg.norm(m)) / xo.size).astype(np.float32)
    dwo, dbo = OP.power_iterate_backward(wl.ch, wl.w, 0.0, 0, gt, gs, c.K, g.astype(np.float64))
    dev = torch.device("cuda")
    s = sf.Solver((c.B, c.T, c.H, c.W), c.C, _gauss(sf, c), c.K, want_tape=True)
    ch = torch.from_numpy(wl.ch).to(dev)
    x = s.forward(ch, wl.w).cpu().numpy()
    assert _rel(x, xo) <= X_TOL and _frame_err(x[0], xo[0]) <= FRAME_TOL
    dw, db = s.backward(ch, wl.w, torch.from_numpy(g).to(dev))
    assert _rel(dw, dwo) <= G_TOL, (dw, dwo)
    assert abs(db - dbo) <= G_TOL * max(abs(dbo), np.abs(dwo).max())
    # Euler identity: identity combine, b = 0 -> w . dL/dw = 0
    assert abs(float(np.dot(wl.w, dw))) <= 1e-4 * np.linalg.norm(wl.w) * np.linalg.norm(dw)


def test_c4_full_size_all_volumes(sf):
    """configs[3] at full size: all 64 volumes of 32x256x256 (C = 4) in one batched solve,
    every volume against the oracle (per-volume norms)."""
    wl = WL.generate("c4", with_mask=False)
    c = wl.cfg
    s = sf.Solver((c.B, c.T, c.H, c.W), c.C, _gauss(sf, c), c.K)
    x = s.forward(torch.from_numpy(wl.ch).cuda(), wl.w).cpu().numpy()
    gains = s.stats.cpu().numpy()[..., 1]
    F, _ = O.combine(wl.ch, wl.w)
    xo, sto = OP.power_iterate(F, *_taps(c), c.K)
    for v in range(c.B):
        assert _rel(x[v], xo[v]) <= X_TOL, f"volume {v}: {_rel(x[v], xo[v]):.3e}"
        assert _frame_err(x[v], xo[v]) <= FRAME_TOL, f"volume {v}"
    np.testing.assert_allclose(gains, sto["gain"], rtol=1e-5)


def test_c5_full_resolution_T64_crop(sf):
    """configs[4] recipe at full 1080x1920 resolution on a T = 64 crop (132.7 M voxels,
    r = (9, 36), K = 20) against the multi-process oracle; plus the full T = 512 solve by
    properties (unit norm, non-negativity, monotone gain, time-reversal equivariance)."""
    c = WL.get_config("c5")
    cfg = WL.get_config("c5", T=64)
    crop = WL.generate("c5", cfg=cfg, with_mask=False)
    s = sf.Solver((1, 64, c.H, c.W), c.C, _gauss(sf, c), c.K)
    x = s.forward(torch.from_numpy(crop.ch).cuda(), crop.w).cpu().numpy()
    st = s.stats.cpu().numpy()
    del s
    F, _ = O.combine(crop.ch, crop.w)
    xo, sto = OP.power_iterate(F, *_taps(c), c.K)
    assert _rel(x, xo) <= X_TOL and _frame_err(x[0], xo[0]) <= FRAME_TOL
    np.testing.assert_allclose(st[..., 1], sto["gain"], rtol=1e-5)
    del x, xo, F, crop
    torch.cuda.empty_cache()
    wl = WL.generate("c5", with_mask=False)
    s = sf.Solver((c.B, c.T, c.H, c.W), c.C, _gauss(sf, c), c.K)
    ch = torch.from_numpy(wl.ch).cuda()
    x = s.forward(ch, wl.w)
    gains = s.stats.cpu().numpy()[0, :, 1]
    assert abs(float(torch.linalg.vector_norm(x.double())) - 1.0) < 1e-5
    assert float(x.min()) >= 0.0
    assert (np.diff(gains) >= -1e-6 * gains[1:]).all()
    xr = s.forward(torch.flip(ch, dims=[2]).contiguous(), wl.w)
    assert float(torch.linalg.vector_norm((torch.flip(xr, dims=[1]) - x).double())) <= 1e-4
