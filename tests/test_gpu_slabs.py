"""GPU: the time-slab decomposition (multi-GPU path's per-rank phases, emulated
on one device: halo copies + rank-ordered norm reduction) matches the single-GPU
solve and the oracle, including uneven slabs and B > 1."""
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
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


@pytest.mark.parametrize("name,shape,nslabs,K", [
    ("c2", dict(T=26, H=70, W=150), 1, 6),
    ("c2", dict(T=26, H=70, W=150), 2, 6),
    ("c2", dict(T=26, H=70, W=150), 4, 6),      # uneven: 6,7,6,7 frames, r_t = 6
    ("c5", dict(T=40, H=64, W=140), 3, 5),      # r_t = 9, r_s = 36
    ("c5", dict(T=40, H=200, W=300), 2, 4),     # several y-blocks and strips per frame-range launch (tcgen05 pass)
    ("c4", dict(B=2, T=23, H=48, W=70), 2, 5),  # B > 1
])
def test_slabs_match_single_gpu_and_oracle(sf, name, shape, nslabs, K):
    cfg = WL.get_config(name, **shape)
    wl = WL.generate(name, cfg=cfg)
    g = sf.Gauss(cfg.sigma_t, cfg.sigma_s, cfg.radius_t, cfg.radius_s)
    ch = torch.from_numpy(wl.ch).cuda()
    xs, sts = sf.power_iterate_slabs(ch, wl.w, g, K, nslabs, want_rayleigh=True)
    B, C, T, H, W = wl.ch.shape
    solver = sf.Solver((B, T, H, W), C, g, K)
    x1 = solver.forward(ch, wl.w, want_rayleigh=True)
    xs, x1 = xs.cpu().numpy(), x1.cpu().numpy()
    for b in range(B):
        assert _rel(xs[b], x1[b].astype(np.float64)) < 1e-6
    np.testing.assert_allclose(sts.cpu().numpy(), solver.stats.cpu().numpy(), rtol=1e-6)
    F, _ = O.combine(wl.ch, wl.w)
    xo, sto = O.power_iterate(F, O.gaussian_taps(cfg.sigma_t, cfg.radius_t),
                              O.gaussian_taps(cfg.sigma_s, cfg.radius_s), K)
    for b in range(B):
        assert _rel(xs[b], xo[b]) <= 1e-4
    np.testing.assert_allclose(sts.cpu().numpy()[..., 1], sto["gain"], rtol=1e-5)


def test_slab_fp16_range_covers_halo_frames(sf):
    """tcgen05 path in slabs: the temporal pass writes v as fp16 planes scaled by 2^e, e from
    max |p_{k-1}| over the frames it READS -- the neighbour's halo frames included.  A dim slab
    (1e-4 x the brightness of its neighbour) would overflow fp16 on its boundary frames if only
    its own maximum set the range."""
    cfg = WL.get_config("c2", T=28, H=70, W=150)
    wl = WL.generate("c2", cfg=cfg)
    chn = wl.ch.copy()
    chn[:, :, :14] *= 1e-4          # slab 0 of 2 is dim, slab 1 bright
    g = sf.Gauss(cfg.sigma_t, cfg.sigma_s, cfg.radius_t, cfg.radius_s)
    B, C, T, H, W = chn.shape
    assert sf.forward_path((B, T // 2, H, W), g, sf.ALGO_AUTO)[0] == sf.PATH_TWO_PASS_TCGEN05
    ch = torch.from_numpy(chn).cuda()
    K = 4
    xs, sts = sf.power_iterate_slabs(ch, wl.w, g, K, 2, want_rayleigh=True)
    xs = xs.cpu().numpy()
    assert np.isfinite(xs).all()
    F, _ = O.combine(chn, wl.w)
    xo, sto = O.power_iterate(F, O.gaussian_taps(cfg.sigma_t, cfg.radius_t),
                              O.gaussian_taps(cfg.sigma_s, cfg.radius_s), K)
    assert _rel(xs[0], xo[0]) <= 1e-4
    # the dim slab's frames next to the bright one are where an overflow would show
    fr = slice(14 - cfg.radius_t, 14)
    assert _rel(xs[0][fr], xo[0][fr]) <= 1e-4
    np.testing.assert_allclose(sts.cpu().numpy()[..., 1], sto["gain"], rtol=1e-5)


def test_slab_too_thin_rejected(sf):
    ch = torch.rand((1, 1, 8, 20, 20), device="cuda")
    with pytest.raises(sf.SfsegError) as e:
        sf.power_iterate_slabs(ch, [1.0], sf.Gauss(2.0, 2.0, 6, 6), 3, 4)   # 2-frame slabs < r_t = 6
    assert e.value.status == 2


def test_nccl_single_rank_dist_path(sf):
    """The NCCL-driven per-rank path (sfseg_comm + dist) with one rank: exercises
    dlopen'd NCCL (unique id, comm init, fp64 allreduce) and the dist finalize."""
    import ctypes as C
    from paper_2212_08058_b200.dist import Comm, SlabSolver
    raw = (C.c_uint8 * 128)()
    st = sf.lib().sfseg_get_unique_id(raw)
    if st == 8:
        pytest.skip("NCCL not loadable")
    assert st == 0
    comm = Comm(1, 0, torch.cuda.current_device(), bytes(raw))
    try:
        cfg = WL.get_config("c2", T=12, H=60, W=100)
        wl = WL.generate("c2", cfg=cfg)
        g = sf.Gauss(2.0, 8.0, 6, 24)
        ch = torch.from_numpy(wl.ch).cuda()
        s = SlabSolver(comm, (1, 12, 60, 100), 12, 0, 1, g, 6)
        xd = s.forward(ch, wl.w).cpu().numpy()
        ref = sf.Solver((1, 12, 60, 100), 1, g, 6)
        x1 = ref.forward(ch, wl.w).cpu().numpy()
        assert _rel(xd, x1.astype(np.float64)) < 1e-6
        np.testing.assert_allclose(s.stats.cpu().numpy(), ref.stats.cpu().numpy(), rtol=1e-6)
        # the NCCL backward path (agreement, bwd phases, allreduces) with one rank
        sb = SlabSolver(comm, (1, 12, 60, 100), 12, 0, 1, g, 6, want_tape=True)
        sb.forward(ch, [1.3], 0.1, 1)
        gr = torch.from_numpy(np.random.default_rng(2).normal(size=(1, 12, 60, 100)).astype(np.float32)).cuda()
        dwd, dbd = sb.backward(ch, [1.3], gr, 0.1, 1)
        _, dw1, db1 = sf.power_iterate_backward(ch, [1.3], g, 6, gr, 0.1, 1)
        # the slab forward's lagged normalisation rounds u differently from the single-GPU forward
        scale = max(abs(dw1[0]), abs(db1))
        assert abs(dwd[0] - dw1[0]) <= 1e-4 * scale and abs(dbd - db1) <= 1e-4 * scale
        # a bad argument on a rank is agreed on before any data-path collective (returns, no hang)
        with pytest.raises(sf.SfsegError):
            sb.backward(ch, [float("nan")], gr, 0.1, 1)
    finally:
        comm.close()


@pytest.mark.parametrize("name,shape,nslabs,act", [
    ("c3", dict(T=26, H=56, W=120), 2, 1),
    ("c3", dict(T=26, H=56, W=120), 4, 0),     # uneven slabs 6,7,6,7 with r_t = 6
    ("c4", dict(B=2, T=23, H=48, W=70), 3, 1), # B > 1, r_t = 5
])
def test_slab_backward_matches_single_gpu_and_oracle(sf, name, shape, nslabs, act):
    """Time-slab backward (per step: halo of F y_bar_k with the neighbour slabs, allreduce of
    <x_{k-1}, x_bar_{k-1}>; final allreduce of dw, db) on the slab forward's tapes == the
    single-GPU backward and the oracle's dL/dw."""
    cfg = WL.get_config(name, **shape)
    wl = WL.generate(name, cfg=cfg)
    B, C, T, H, W = wl.ch.shape
    w = wl.w if act == 0 else (np.arange(C, dtype=np.float32) * 0.3 - 0.2)
    b = 0.0 if act == 0 else 0.15
    K = 5
    g = sf.Gauss(cfg.sigma_t, cfg.sigma_s, cfg.radius_t, cfg.radius_s)
    ch = torch.from_numpy(wl.ch).cuda()
    rng = np.random.default_rng(9)
    gr = rng.normal(size=(B, T, H, W)).astype(np.float32)
    grt = torch.from_numpy(gr).cuda()
    xs, _, tape = sf.power_iterate_slabs(ch, w, g, K, nslabs, b, act, want_tape=True)
    dws, dbs = sf.power_iterate_slabs_backward(ch, w, g, K, nslabs, tape, grt, b, act)
    x1, dw1, db1 = sf.power_iterate_backward(ch, w, g, K, grt, b, act)
    dwo, dbo = O.power_iterate_backward(wl.ch, w, b, act, O.gaussian_taps(cfg.sigma_t, cfg.radius_t),
                                        O.gaussian_taps(cfg.sigma_s, cfg.radius_s), K, gr.astype(np.float64))
    assert _rel(dws, np.array(dwo)) <= 1e-3
    assert _rel(dws, np.array(dw1)) <= 1e-4     # lagged normalisation + reduction order
    assert abs(dbs - dbo) <= 1e-3 * max(abs(dbo), np.abs(dwo).max())
    assert _rel(xs.cpu().numpy(), x1.cpu().numpy()) <= 1e-6


@pytest.mark.parametrize("name,shape,nslabs,algo", [
    ("c2", dict(T=40, H=70, W=150), 3, "auto"),    # 13/14-frame slabs, r_t = 6: boundary + 1-2 interior frames
    ("c2", dict(T=26, H=70, W=150), 4, "auto"),    # middle slabs too thin to split: one launch
    ("c5", dict(T=40, H=64, W=140), 2, "fp32"),    # r_t = 9, FP32-FMA spatial pass
    ("c4", dict(B=2, T=30, H=48, W=70), 2, "mma"),  # B > 1, bf16 three-plane pass
])
def test_slab_overlapped_schedule_bitwise_equals_serial(sf, name, shape, nslabs, algo):
    """The overlapped time-slab schedule (boundary frames first, halo copies under the interior
    frames and the norm reduction under the next temporal pass, on a second stream) gives
    bitwise the serial schedule's x, stats and tape; both match the single-GPU solve."""
    cfg = WL.get_config(name, **shape)
    wl = WL.generate(name, cfg=cfg)
    g = sf.Gauss(cfg.sigma_t, cfg.sigma_s, cfg.radius_t, cfg.radius_s)
    A = {"auto": sf.ALGO_AUTO, "fp32": sf.ALGO_TWO_PASS_FP32, "mma": sf.ALGO_TWO_PASS_MMA_SYNC}[algo]
    ch = torch.from_numpy(wl.ch).cuda()
    K = 6
    res = {}
    for sched in (sf.SLAB_OVERLAP, sf.SLAB_SERIAL):
        x, st, tape = sf.power_iterate_slabs(ch, wl.w, g, K, nslabs, want_rayleigh=True, algo=A, want_tape=True,
                                             slab_schedule=sched)
        torch.cuda.synchronize()
        res[sched] = (x.cpu().numpy(), st.cpu().numpy(), tape.cpu().numpy())
    for a, b in zip(res[sf.SLAB_OVERLAP], res[sf.SLAB_SERIAL]):
        assert np.array_equal(a, b)
    B, C, T, H, W = wl.ch.shape
    s1 = sf.Solver((B, T, H, W), C, g, K, algo=A)
    x1 = s1.forward(ch, wl.w, want_rayleigh=True).cpu().numpy()
    for b in range(B):
        assert _rel(res[sf.SLAB_OVERLAP][0][b], x1[b].astype(np.float64)) < 1e-6
    np.testing.assert_allclose(res[sf.SLAB_OVERLAP][1], s1.stats.cpu().numpy(), rtol=1e-6)
