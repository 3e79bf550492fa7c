"""GPU parity of the online / sub-window mode against the oracle."""
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


@pytest.mark.parametrize("shape,q,stride,radii,K", [
    ((1, 20, 40, 70), 7, 3, (2, 6), 6),      # overlapping windows, ragged last window
    ((2, 21, 33, 90), 7, 7, (3, 6), 5),      # disjoint windows, B > 1
    ((1, 12, 48, 64), 20, 4, (1, 3), 8),     # q >= T: the offline solve
    ((1, 30, 60, 150), 14, 5, (6, 24), 5),   # config-2 radii
])
def test_online_matches_oracle(sf, shape, q, stride, radii, K):
    B, T, H, W = shape
    rng = np.random.default_rng(sum(shape) + q)
    ch = (rng.random((B, 1, T, H, W)) * 0.8 + 0.1).astype(np.float32)
    r_t, r_s = radii
    st, ss = max(r_t, 1) / 3.0, max(r_s, 1) / 3.0
    x = sf.power_iterate_online(torch.from_numpy(ch).to("cuda"), [1.0], sf.Gauss(st, ss, r_t, r_s), K, q,
                                stride).cpu().numpy()
    F, _ = O.combine(ch, [1.0])
    xo = O.power_iterate_online(F, O.gaussian_taps(st, r_t), O.gaussian_taps(ss, r_s), K, q, stride)
    for b in range(B):
        assert _rel(x[b], xo[b]) <= 1e-4, f"volume {b}: {_rel(x[b], xo[b]):.3e}"


def test_online_c2_recipe_multichannel(sf):
    """c3 recipe crop (6 channels, softmax weights): F combined once, windows of 14 by 7."""
    cfg = WL.get_config("c3", T=30, H=64, W=120)
    wl = WL.generate("c3", cfg=cfg)
    g = sf.Gauss(2.0, 8.0, 6, 24)
    x = sf.power_iterate_online(torch.from_numpy(wl.ch).to("cuda"), wl.w, g, 6, 14, 7).cpu().numpy()
    F, _ = O.combine(wl.ch, wl.w)
    xo = O.power_iterate_online(F, O.gaussian_taps(2.0, 6), O.gaussian_taps(8.0, 24), 6, 14, 7)
    assert _rel(x, xo) <= 1e-4


def test_online_zero_window_error_is_not_wiped(sf):
    """an all-zero F window in the MIDDLE of the video (stride == q, so windows
    are disjoint) makes that window's solve degenerate; later windows must not clear the
    workspace's error word (sticky until sfseg_sync_status), so the call reports it."""
    rng = np.random.default_rng(5)
    ch = (rng.random((1, 1, 15, 20, 30)) * 0.8 + 0.1).astype(np.float32)
    ch[:, :, 5:10] = 0.0   # window [5, 10) is all zero
    with pytest.raises(sf.SfsegError) as e:
        sf.power_iterate_online(torch.from_numpy(ch).cuda(), [1.0], sf.Gauss(1.0, 2.0, 2, 6), 4, 5, 5)
    assert e.value.status == 4   # SFSEG_ERR_DEGENERATE


def test_sticky_error_survives_later_solves(sf):
    """Two solves on one workspace, the first degenerate (F == 0), the second fine: the
    error is reported at the sync after the second (sticky), then cleared."""
    g = sf.Gauss(1.0, 2.0, 2, 6)
    s = sf.Solver((1, 4, 16, 24), 1, g, 3)
    z = torch.zeros((1, 1, 4, 16, 24), dtype=torch.float32, device="cuda")
    ok = torch.rand((1, 1, 4, 16, 24), dtype=torch.float32, device="cuda") + 0.1
    s.forward(z, [1.0], check=False)
    s.forward(ok, [1.0], check=False)
    with pytest.raises(sf.SfsegError) as e:
        s.sync()
    assert e.value.status == 4
    s.forward(ok, [1.0])   # cleared by the sync that reported it
