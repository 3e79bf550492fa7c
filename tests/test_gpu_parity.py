"""GPU parity: the CUDA path (through the C ABI) against the f64 oracle.

Tolerances (BASELINE.json north_star):
  x_K relative L2 <= 1e-4;  dL/dw relative <= 1e-3;  masks bit-exact wherever
  |x_hat - tau| > 1e-4;  per-iteration gains within 1e-5 relative.
"""
import math

import numpy as np
import pytest

import oracle as O
import workloads as WL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

X_TOL = 1e-4
G_TOL = 1e-3
GAIN_TOL = 1e-5


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


def _gpu_solve(sf, ch, w, gauss, K, b=0.0, act=0, x0=None, rayleigh=True, algo=0):
    dev = torch.device("cuda")
    cht = torch.from_numpy(np.ascontiguousarray(ch)).to(dev)
    B, C, T, H, W = ch.shape
    s = sf.Solver((B, T, H, W), C, gauss, K, algo=algo)
    x0t = None if x0 is None else torch.from_numpy(np.ascontiguousarray(x0, dtype=np.float32)).to(dev)
    x = s.forward(cht, w, b, act, x0=x0t, want_rayleigh=rayleigh)
    return x.cpu().numpy(), s.stats.cpu().numpy(), s


def _oracle_solve(ch, w, gauss_vals, K, b=0.0, act=0, x0=None):
    sig_t, sig_s, r_t, r_s = gauss_vals
    F, _ = O.combine(ch, w, b, act)
    gt, gs = O.gaussian_taps(sig_t, r_t), O.gaussian_taps(sig_s, r_s)
    return O.power_iterate(F, gt, gs, K, x0=None if x0 is None else np.asarray(x0, np.float64))


def _frame_err(a, b):
    """Per-frame bound: max over frames of max|a - b| / max|b| in that frame (a local error
    in one strip, border frame or ragged tail cannot hide in a volume-wide norm)."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    d = np.abs(a - b).reshape(b.shape[0], -1).max(-1)
    m = np.abs(b).reshape(b.shape[0], -1).max(-1)
    ok = m > 0
    return float((d[ok] / m[ok]).max()) if ok.any() else float(d.max())


FRAME_TOL = 1e-4


def _check_forward(sf, ch, w, sig_t, sig_s, r_t, r_s, K, b=0.0, act=0, x0=None, algo=0):
    gauss = sf.Gauss(sig_t, sig_s, r_t, r_s)
    xg, stg, _ = _gpu_solve(sf, ch, w, gauss, K, b, act, x0, algo=algo)
    xo, sto = _oracle_solve(ch, w, (sig_t, sig_s, r_t, r_s), K, b, act, x0)
    assert np.isfinite(xg).all()
    for bb in range(ch.shape[0]):
        assert _rel(xg[bb], xo[bb]) <= X_TOL, f"volume {bb}: x rel err {_rel(xg[bb], xo[bb]):.3e}"
        assert _frame_err(xg[bb], xo[bb]) <= FRAME_TOL, f"volume {bb}: frame err {_frame_err(xg[bb], xo[bb]):.3e}"
    np.testing.assert_allclose(stg[..., 0], sto["nu"], rtol=GAIN_TOL)
    np.testing.assert_allclose(stg[..., 1], sto["gain"], rtol=GAIN_TOL)
    np.testing.assert_allclose(stg[..., 2], sto["rho"], rtol=GAIN_TOL)
    # unit norm per volume
    for bb in range(ch.shape[0]):
        assert abs(np.linalg.norm(xg[bb].astype(np.float64)) - 1.0) < 1e-5
    return xg, xo, stg


# --------------------------------------------------------------------------- configs
def test_c1_full(sf):
    wl = WL.generate("c1")
    c = wl.cfg
    _check_forward(sf, wl.ch, wl.w, c.sigma_t, c.sigma_s, c.radius_t, c.radius_s, c.K)


def test_c2_recipe_several_strips_ragged(sf):
    cfg = WL.get_config("c2", T=16, H=150, W=300)   # 3 strips (128+128+44), 150 rows: ragged blocks
    wl = WL.generate("c2", cfg=cfg)
    _check_forward(sf, wl.ch, wl.w, 2.0, 8.0, 6, 24, 15)


def test_c3_recipe_forward(sf):
    cfg = WL.get_config("c3", T=14, H=100, W=200)
    wl = WL.generate("c3", cfg=cfg)
    _check_forward(sf, wl.ch, wl.w, 2.0, 8.0, 6, 24, 15)


def test_c4_recipe_batched(sf):
    cfg = WL.get_config("c4", B=3, T=12, H=64, W=96)
    wl = WL.generate("c4", cfg=cfg)
    _check_forward(sf, wl.ch, wl.w, 1.5, 6.0, 5, 18, 10)


def test_c5_recipe_crop(sf):
    cfg = WL.get_config("c5", T=24, H=90, W=260)
    wl = WL.generate("c5", cfg=cfg)
    _check_forward(sf, wl.ch, wl.w, 3.0, 12.0, 9, 36, 6)


def test_probe_small_radius(sf):
    cfg = WL.get_config("c2", T=10, H=64, W=140)
    wl = WL.generate("c2", cfg=cfg)
    _check_forward(sf, wl.ch, wl.w, 0.5, 1.0, 1, 3, 15)


@pytest.mark.parametrize("case", ["c1", "probe", "edge", "c2", "c4"])
def test_two_pass_path(sf, case):
    """Small radii run the fused single-pass 3D kernel by default; the two-pass (one
    temporal + one spatial launch per iteration) path must give the same result."""
    A = sf.ALGO_TWO_PASS
    if case == "c1":
        wl = WL.generate("c1")
        c = wl.cfg
        _check_forward(sf, wl.ch, wl.w, c.sigma_t, c.sigma_s, c.radius_t, c.radius_s, c.K, algo=A)
    elif case == "probe":
        cfg = WL.get_config("c2", T=10, H=64, W=140)
        wl = WL.generate("c2", cfg=cfg)
        _check_forward(sf, wl.ch, wl.w, 0.5, 1.0, 1, 3, 15, algo=A)
    elif case == "c2":
        cfg = WL.get_config("c2", T=16, H=150, W=300)
        wl = WL.generate("c2", cfg=cfg)
        _check_forward(sf, wl.ch, wl.w, 2.0, 8.0, 6, 24, 15, algo=A)
    elif case == "c4":
        cfg = WL.get_config("c4", B=3, T=12, H=64, W=96)
        wl = WL.generate("c4", cfg=cfg)
        _check_forward(sf, wl.ch, wl.w, 1.5, 6.0, 5, 18, 10, algo=A)
    else:
        rng = np.random.default_rng(11)
        ch = (rng.random((2, 1, 7, 45, 150)) * 0.8 + 0.1).astype(np.float32)
        _check_forward(sf, ch, [1.0], 1.0, 2.0, 3, 6, 4, algo=A)


@pytest.mark.parametrize("case", ["c2", "c4", "c5", "edge"])
def test_fp32_spatial_pass_path(sf, case):
    """ALGO_TWO_PASS_FP32: the two-pass iteration with the FP32-FMA spatial pass
    (the default two-pass forward runs the spatial pass on the bf16 tensor pipe)."""
    A = sf.ALGO_TWO_PASS_FP32
    if case == "c2":
        wl = WL.generate("c2", cfg=WL.get_config("c2", T=16, H=150, W=300))
        _check_forward(sf, wl.ch, wl.w, 2.0, 8.0, 6, 24, 15, algo=A)
    elif case == "c4":
        wl = WL.generate("c4", cfg=WL.get_config("c4", B=3, T=12, H=64, W=96))
        _check_forward(sf, wl.ch, wl.w, 1.5, 6.0, 5, 18, 10, algo=A)
    elif case == "c5":
        wl = WL.generate("c5", cfg=WL.get_config("c5", T=24, H=90, W=260))
        _check_forward(sf, wl.ch, wl.w, 3.0, 12.0, 9, 36, 6, algo=A)
    else:
        rng = np.random.default_rng(12)
        ch = (rng.random((2, 1, 7, 45, 150)) * 0.8 + 0.1).astype(np.float32)
        _check_forward(sf, ch, [1.0], 1.0, 4.0, 3, 12, 4, algo=A)


@pytest.mark.parametrize("seed", range(6))
def test_tensor_core_random_shapes(sf, seed):
    """Seeded random shapes / radii / weights through the default (tensor-core) path:
    ragged strips and blocks, B > 1, sigmoid combine, both against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    B = int(rng.integers(1, 3))
    T = int(rng.integers(1, 9))
    H = int(rng.integers(1, 110))
    W = int(rng.integers(1, 200))
    C = int(rng.integers(1, 4))
    r_s = int(rng.choice([8, 9, 12, 16, 18, 24]))
    r_t = int(rng.integers(0, 7))
    ch = (rng.random((B, C, T, H, W)) * 0.8 + 0.1).astype(np.float32)
    w = (rng.random(C) + 0.2).astype(np.float32)
    act = int(rng.integers(0, 2))
    _check_forward(sf, ch, w, max(r_t, 1) / 3.0, r_s / 3.0, r_t, r_s, 4, b=0.1 * act, act=act)


@pytest.mark.parametrize("r_s,shape", [
    (8, (2, 5, 70, 200)),      # NKX = 2, one-slot prologue
    (9, (1, 6, 33, 130)),      # radius not a multiple of 4: box offset D = 3
    (12, (1, 4, 97, 71)),      # W < 2 strips, ragged 32-row blocks
    (16, (1, 3, 64, 129)),     # one live column in the last strip
    (32, (1, 3, 50, 300)),     # four-slot ring
    (48, (1, 2, 130, 190)),    # largest compiled radius (box 168 columns)
    (12, (1, 3, 5, 5)),        # W, H << radius: one partial strip, two dead warps, pure padding
    (16, (2, 2, 1, 300)),      # H = 1: every window is zero padding but one row
    (8, (1, 1, 40, 9)),        # T = 1, W = 9 (pitch 16)
])
def test_tensor_core_spatial_radii(sf, r_s, shape):
    """Every compiled radius of the tensor-core spatial pass, on ragged shapes,
    against the oracle (x_K 1e-4, gains 1e-5) and against the FP32 spatial pass."""
    B, T, H, W = shape
    rng = np.random.default_rng(r_s)
    ch = (rng.random((B, 1, T, H, W)) * 0.8 + 0.1).astype(np.float32)
    sig_s = r_s / 3.0
    xg, xo, _ = _check_forward(sf, ch, [1.0], 1.0, sig_s, 2, r_s, 5)
    x32, _, _ = _gpu_solve(sf, ch, [1.0], sf.Gauss(1.0, sig_s, 2, r_s), 5, algo=sf.ALGO_TWO_PASS_FP32)
    for bb in range(B):
        # fp32-class arithmetic on both paths (six bf16 products vs fp32 FMAs)
        assert _rel(xg[bb], x32[bb]) <= 2e-6
        assert _rel(x32[bb], xo[bb]) <= 1e-6
        assert _rel(xg[bb], xo[bb]) <= 1e-6


def test_fused_probe_ragged_tiles_and_runs(sf):
    """Fused path: tiles ragged in x and y (W=300, H=61 with 24-row tiles), T long
    enough that CTA ranges split a tile's frames into several runs."""
    cfg = WL.get_config("c2", T=37, H=61, W=300)
    wl = WL.generate("c2", cfg=cfg)
    _check_forward(sf, wl.ch, wl.w, 0.5, 1.0, 1, 3, 7)


@pytest.mark.parametrize("shape,radii", [
    ((1, 1, 1, 1), (0, 1)),          # single voxel: y = F^2 x
    ((1, 1, 5, 7), (2, 3)),          # T = 1 (temporal radius > T)
    ((2, 3, 1, 9), (1, 2)),          # H = 1
    ((1, 4, 6, 1), (2, 2)),          # W = 1
    ((1, 5, 33, 854), (2, 4)),       # DAVIS width: pitch 856, 7 strips
    ((1, 3, 20, 20), (9, 36)),       # radii >= every dimension: pure zero padding
    ((2, 9, 40, 130), (4, 9)),       # B > 1 across strips
])
def test_edge_shapes(sf, shape, radii):
    B, T, H, W = shape
    rng = np.random.default_rng(sum(shape))
    ch = (rng.random((B, 1, T, H, W)) * 0.8 + 0.1).astype(np.float32)
    r_t, r_s = radii
    _check_forward(sf, ch, [1.0], max(r_t, 1) / 3.0, max(r_s, 1) / 3.0, r_t, r_s, 4)


def test_sigmoid_combine_and_bias(sf):
    rng = np.random.default_rng(3)
    ch = rng.normal(size=(2, 3, 6, 40, 70)).astype(np.float32)
    _check_forward(sf, ch, [0.5, -1.0, 0.7], 1.0, 3.0, 3, 9, 5, b=0.3, act=1)


def test_user_x0(sf):
    rng = np.random.default_rng(4)
    ch = rng.random((1, 1, 8, 50, 60)).astype(np.float32)
    x0 = rng.random((1, 8, 50, 60)).astype(np.float32)
    _check_forward(sf, ch, [1.0], 1.0, 2.0, 3, 6, 6, x0=x0)


# --------------------------------------------------------------------------- device errors / validation
def test_degenerate_and_nonfinite(sf):
    dev = torch.device("cuda")
    g = sf.Gauss(1.0, 2.0)
    s = sf.Solver((1, 4, 16, 16), 1, g, 3)
    with pytest.raises(sf.SfsegError) as e:
        s.forward(torch.zeros((1, 1, 4, 16, 16), device=dev), [1.0])
    assert e.value.status == 4
    ch = torch.rand((1, 1, 4, 16, 16), device=dev)
    ch[0, 0, 2, 5, 5] = float("nan")
    with pytest.raises(sf.SfsegError) as e:
        s.forward(ch, [1.0])
    assert e.value.status == 5
    # error word is cleared: a good solve afterwards succeeds
    s.forward(torch.rand((1, 1, 4, 16, 16), device=dev), [1.0])


def test_workspace_too_small(sf):
    import ctypes as C
    dev = torch.device("cuda")
    L = sf.lib()
    ch = torch.rand((1, 1, 4, 16, 16), device=dev)
    x = torch.empty((1, 4, 16, 16), device=dev)
    ws = torch.empty(1024, dtype=torch.uint8, device=dev)
    st = L.sfseg_power_iterate(C.c_void_p(ch.data_ptr()), 1, (C.c_float * 1)(1.0), 0.0, 0, sf.Shape(1, 4, 16, 16),
                               sf.Gauss(1.0, 2.0).c(), 3, None, C.c_void_p(x.data_ptr()), None, None, 0, None,
                               C.c_void_p(ws.data_ptr()), 1024, None, sf._stream())
    assert st == 3
    st = L.sfseg_power_iterate(C.c_void_p(ch.data_ptr()), 1, (C.c_float * 1)(1.0), 0.0, 0, sf.Shape(1, 4, 16, 16),
                               sf.Gauss(1.0, 2.0).c(), 3, None, C.c_void_p(x.data_ptr()), None, None, 0, None,
                               C.c_void_p(ws.data_ptr() + 8), 1000, None, sf._stream())
    assert st == 3


def test_deterministic_bitwise(sf):
    cfg = WL.get_config("c2", T=12, H=120, W=300)
    wl = WL.generate("c2", cfg=cfg)
    g = sf.Gauss(2.0, 8.0, 6, 24)
    a, sa, _ = _gpu_solve(sf, wl.ch, wl.w, g, 8)
    b, sb, _ = _gpu_solve(sf, wl.ch, wl.w, g, 8)
    assert np.array_equal(a, b) and np.array_equal(sa, sb)


@pytest.mark.parametrize("radii", [(6, 24), (1, 3)])
def test_cuda_graph_capture_and_replay(sf, radii):
    """The forward + threshold (every kernel, no host sync) captured into one CUDA graph
    and replayed gives bitwise the stream-launched result (bench.py --graph 1)."""
    r_t, r_s = radii
    cfg = WL.get_config("c2", T=10, H=70, W=140)
    wl = WL.generate("c2", cfg=cfg)
    dev = torch.device("cuda")
    B, C, T, H, W = wl.ch.shape
    s = sf.Solver((B, T, H, W), C, sf.Gauss(r_t / 3.0, r_s / 3.0, r_t, r_s), 6)
    ch = torch.from_numpy(wl.ch).to(dev)
    x = torch.empty((B, T, H, W), dtype=torch.float32, device=dev)
    m = torch.empty((B, T, H, W), dtype=torch.uint8, device=dev)

    def step():
        s.forward(ch, wl.w, 0.0, 0, x_out=x, check=False)
        s.threshold(x, 0.5, sf.THR_PER_FRAME_MAX, mask=m)

    step()
    s.sync()
    x_ref, m_ref = x.clone(), m.clone()
    x.zero_()
    m.zero_()
    graph = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(dev)
    cap.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(cap):
        with torch.cuda.graph(graph, stream=cap):
            step()
    torch.cuda.current_stream(dev).wait_stream(cap)
    torch.cuda.synchronize(dev)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize(dev)
    assert torch.equal(x, x_ref) and torch.equal(m, m_ref)
    xo, _ = _oracle_solve(wl.ch, wl.w, (r_t / 3.0, r_s / 3.0, r_t, r_s), 6)
    assert _rel(x.cpu().numpy(), xo) <= X_TOL


# --------------------------------------------------------------------------- invariants
def test_invariants_nonneg_monotone_mirror(sf):
    cfg = WL.get_config("c2", T=12, H=96, W=200)
    wl = WL.generate("c2", cfg=cfg)
    g = sf.Gauss(2.0, 8.0, 6, 24)
    x, st, _ = _gpu_solve(sf, wl.ch, wl.w, g, 10)
    assert (x >= 0).all()
    gain = st[0, :, 1]
    assert (np.diff(gain) >= -1e-6 * gain[1:]).all()
    for ax in (2, 3, 4):
        xm, _, _ = _gpu_solve(sf, np.ascontiguousarray(np.flip(wl.ch, ax)), wl.w, g, 10)
        assert _rel(np.flip(xm, ax - 1), x) < 1e-5
    xs, _, _ = _gpu_solve(sf, wl.ch * np.float32(2.0), wl.w, g, 10)
    assert _rel(xs, x) < 1e-5


# --------------------------------------------------------------------------- threshold
def test_threshold_parity(sf):
    cfg = WL.get_config("c2", T=10, H=80, W=150)
    wl = WL.generate("c2", cfg=cfg)
    g = sf.Gauss(2.0, 8.0, 6, 24)
    xg, _, _ = _gpu_solve(sf, wl.ch, wl.w, g, 15)
    xo, _ = _oracle_solve(wl.ch, wl.w, (2.0, 8.0, 6, 24), 15)
    xt = torch.from_numpy(xg).cuda()
    for mode, tau in ((sf.THR_PER_FRAME_MAX, 0.5), (sf.THR_PER_FRAME_MAX, 0.1), (sf.THR_GLOBAL_MAX, 0.3),
                      (sf.THR_ABSOLUTE, float(np.median(xg)))):
        mg = sf.threshold(xt, tau, mode).cpu().numpy()
        # same fp32 x: the decision is exact except where x / max is within rounding of tau
        mo_same = O.threshold(xg, tau, mode)
        if mode == sf.THR_ABSOLUTE:
            xh = xg.astype(np.float64)
            band_scale = 1.0
        else:
            m = xg.max(axis=(2, 3), keepdims=True) if mode == sf.THR_PER_FRAME_MAX else \
                xg.max(axis=(1, 2, 3), keepdims=True)
            xh = xg / m
            band_scale = 1.0
        sure = np.abs(xh - tau) > 1e-6 * band_scale
        assert np.array_equal(mg[sure], mo_same[sure])
        # against the oracle's own x_K: bit-exact outside the 1e-4 band (north star)
        mo = O.threshold(xo, tau, mode)
        if mode == sf.THR_ABSOLUTE:
            xho = xo
        else:
            mm = xo.max(axis=(2, 3), keepdims=True) if mode == sf.THR_PER_FRAME_MAX else \
                xo.max(axis=(1, 2, 3), keepdims=True)
            xho = xo / mm
        band = np.abs(xho - tau) > (1e-4 if mode != sf.THR_ABSOLUTE else 1e-4 * np.abs(xo).max())
        assert np.array_equal(mg[band], mo[band])


def test_threshold_zero_frame(sf):
    x = torch.zeros((1, 3, 4, 5), device="cuda")
    x[0, 1, 2, 3] = 1.0
    m = sf.threshold(x, 0.5).cpu().numpy()
    assert m.sum() == 1 and m[0, 1, 2, 3] == 1


# --------------------------------------------------------------------------- backward
def _mse_grad(x, mask):
    m = mask.astype(np.float64)
    mh = m / np.linalg.norm(m)
    return 2.0 * (x - mh) / x.size


@pytest.mark.parametrize("act,b,algo", [(0, 0.0, "auto"), (1, 0.2, "auto"), (1, 0.2, "fp32")])
def test_backward_c3_recipe(sf, act, b, algo):
    """dL/dw through the unrolled iterations; "auto" records the tape with the
    tensor-core forward spatial pass, "fp32" with the FP32-FMA one (the backward
    passes are FP32 in both)."""
    _backward_c3_case(sf, act, b, sf.ALGO_TWO_PASS_FP32 if algo == "fp32" else sf.ALGO_AUTO)


def _backward_c3_case(sf, act, b, algo=0):
    cfg = WL.get_config("c3", T=12, H=72, W=150)
    wl = WL.generate("c3", cfg=cfg)
    w = wl.w if act == 0 else np.array([0.5, -0.3, 0.8, 0.1, 0.6, -0.2], np.float32)
    K = 15
    xo, _ = _oracle_solve(wl.ch, w, (2.0, 8.0, 6, 24), K, b, act)
    g = _mse_grad(xo, wl.mask).astype(np.float32)
    dwo, dbo = O.power_iterate_backward(wl.ch, w, b, act, O.gaussian_taps(2.0, 6), O.gaussian_taps(8.0, 24), K,
                                        g.astype(np.float64))
    dev = torch.device("cuda")
    B, C, T, H, W = wl.ch.shape
    s = sf.Solver((B, T, H, W), C, sf.Gauss(2.0, 8.0, 6, 24), K, want_tape=True, algo=algo)
    cht = torch.from_numpy(wl.ch).to(dev)
    s.forward(cht, w, b, act)
    dw, db = s.backward(cht, w, torch.from_numpy(g).to(dev), b, act)
    assert _rel(dw, dwo) <= G_TOL, f"dw rel err {_rel(dw, dwo):.3e}"
    assert abs(db - dbo) <= G_TOL * max(abs(dbo), np.abs(dwo).max())
    if act == 0:
        # Euler identity: w . dL/dw = 0 for identity combine, b = 0
        assert abs(float(np.dot(w, dw))) <= 1e-4 * np.linalg.norm(w) * np.linalg.norm(dw)


def test_backward_user_x0(sf):
    rng = np.random.default_rng(8)
    ch = rng.random((2, 2, 6, 40, 50)).astype(np.float32)
    x0 = rng.random((2, 6, 40, 50)).astype(np.float32)
    g = rng.normal(size=(2, 6, 40, 50)).astype(np.float32)
    w = np.array([0.6, 0.9], np.float32)
    gt, gs = O.gaussian_taps(1.0, 3), O.gaussian_taps(2.0, 6)
    dwo, dbo = O.power_iterate_backward(ch, w, 0.1, 1, gt, gs, 5, g.astype(np.float64), x0=x0)
    dev = torch.device("cuda")
    s = sf.Solver((2, 6, 40, 50), 2, sf.Gauss(1.0, 2.0, 3, 6), 5, want_tape=True)
    cht = torch.from_numpy(ch).to(dev)
    x0t = torch.from_numpy(x0).to(dev)
    s.forward(cht, w, 0.1, 1, x0=x0t)
    dw, db = s.backward(cht, w, torch.from_numpy(g).to(dev), 0.1, 1, x0=x0t)
    assert _rel(dw, dwo) <= G_TOL
    assert abs(db - dbo) <= G_TOL * max(abs(dbo), np.abs(dwo).max())


@pytest.mark.parametrize("algo,radii,expect", [
    ("auto", (6, 24), "t6"), ("auto", (1, 3), "f3d"), ("fp32", (6, 24), "fp32"), ("two", (1, 3), "fp32"),
    ("mma", (6, 24), "tc"), ("f16", (6, 24), "f16"),
])
def test_reported_path_is_the_launched_path(sf, algo, radii, expect):
    """sfseg_forward_path's answer matches the kernels that actually run (per-category
    launch counts of a caller-owned sfseg_profiler passed in the call's options)."""
    r_t, r_s = radii
    g = sf.Gauss(r_t / 3.0 if r_t > 1 else 0.5, r_s / 3.0, r_t, r_s)
    shape = (1, 14, 64, 140)
    sel = {"auto": sf.ALGO_AUTO, "fp32": sf.ALGO_TWO_PASS_FP32, "two": sf.ALGO_TWO_PASS,
           "mma": sf.ALGO_TWO_PASS_MMA_SYNC, "f16": sf.ALGO_TWO_PASS_MMA_F16}[algo]
    path = sf.forward_path(shape, g, sel)[0]
    want = {"tc": sf.PATH_TWO_PASS_TC, "f16": sf.PATH_TWO_PASS_TC_F16, "f3d": sf.PATH_FUSED_3D,
            "fp32": sf.PATH_TWO_PASS_FP32, "t6": sf.PATH_TWO_PASS_TCGEN05}[expect]
    assert path == want
    rng = np.random.default_rng(3)
    ch = torch.from_numpy((rng.random((1, 1) + shape[1:]) * 0.8 + 0.1).astype(np.float32)).cuda()
    s0 = sf.Solver(shape, 1, g, 3, algo=sel)        # no profiler: nothing recorded
    s0.forward(ch, [1.0])
    prof = sf.Profiler()
    s = sf.Solver(shape, 1, g, 3, algo=sel, profiler=prof)
    s.forward(ch, [1.0])
    n = {k: v[1] for k, v in prof.read().items()}
    prof.close()
    if expect in ("tc", "f16", "fp32", "t6"):
        assert n["tpass"] == 3 and n["spass"] == 3 and n["f3d"] == 0
    else:
        assert n["f3d"] == 3 and n["spass"] == 0 and n["tpass"] == 0
