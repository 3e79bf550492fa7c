"""GPU learning loop against the oracle's loop."""
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


def test_training_trajectory_matches_oracle(sf):
    """Five AdamW steps on the c3 recipe crop: the GPU loop (forward + backward through the
    C ABI) and the f64 oracle loop give the same losses and weights."""
    cfg = WL.get_config("c3", T=8, H=48, W=80)
    wl = WL.generate("c3", cfg=cfg)
    g = sf.Gauss(2.0, 8.0, 6, 24)
    dev = torch.device("cuda")
    w_g, b_g, l_g = sf.train_weights(torch.from_numpy(wl.ch).to(dev), torch.from_numpy(wl.mask).to(dev),
                                     wl.w, 0.0, 1, g, 6, 5, 0.05)
    w_o, b_o, l_o = O.train(wl.ch, wl.mask, wl.w, 0.0, 1, O.gaussian_taps(2.0, 6), O.gaussian_taps(8.0, 24), 6, 5,
                            0.05)
    np.testing.assert_allclose(l_g, l_o, rtol=1e-4)
    np.testing.assert_allclose(w_g, w_o, rtol=0, atol=1e-4)
    assert abs(b_g - b_o) <= 1e-4
    assert l_g[-1] < l_g[0]


def test_training_prefers_clean_channels(sf):
    """Fig. learned_weights on a synthetic three-channel stack (clean, noisy, random)."""
    rng = np.random.default_rng(1)
    T, H, W = 6, 40, 60
    m = np.zeros((1, T, H, W), bool)
    m[:, :, 10:28, 15:40] = True
    base = m.astype(np.float32)
    ch = np.stack([base, np.clip(base + rng.normal(0, 0.3, base.shape), 0, 1),
                   rng.random(base.shape)], axis=1).astype(np.float32)
    dev = torch.device("cuda")
    # SFSeg++ form: sigmoid combine (Eq.9); the identity combine with b = 0 is scale invariant
    # in w (w . dL/dw = 0), which leaves the ordering of weak channels loose
    w, b, losses = sf.train_weights(torch.from_numpy(ch).to(dev), torch.from_numpy(m).to(dev), [0.3, 0.3, 0.3], 0.0,
                                    1, sf.Gauss(1.0, 2.0, 3, 6), 5, 30, 0.05)
    assert losses[-1] < losses[0]
    assert w[0] > w[1] > w[2]
