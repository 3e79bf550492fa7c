"""Seeded generator checks (CPU): determinism, frame-addressability, value ranges."""
import numpy as np

import workloads as WL


def test_c1_recipe():
    wl = WL.generate("c1")
    assert wl.ch.shape == (1, 1, 8, 32, 32) and wl.ch.dtype == np.float32
    raw = np.random.default_rng(0).random((8, 32, 32))
    # interior voxel: plain 3x3 mean; corner: mean of the 4 in-bounds values
    assert wl.ch[0, 0, 3, 10, 10] == np.float32(raw[3, 9:12, 9:12].mean())
    assert wl.ch[0, 0, 0, 0, 0] == np.float32(raw[0, 0:2, 0:2].mean())
    assert (wl.ch > 0).all()


def test_c2_small_crop_deterministic_and_addressable():
    cfg = WL.get_config("c2", T=12, H=96, W=150)
    a = WL.generate("c2", cfg=cfg)
    b = WL.generate("c2", cfg=cfg)
    np.testing.assert_array_equal(a.ch, b.ch)
    c = WL.generate("c2", cfg=cfg, t_range=(5, 9))
    np.testing.assert_array_equal(a.ch[:, :, 5:9], c.ch)
    assert a.ch.min() >= 0 and a.ch.max() <= 1
    assert a.mask.any()
    # blob interior is bright (0.9 +- noise) and background dim
    assert a.ch[0, 0][a.mask[0]].mean() > 0.8
    assert a.ch[0, 0][~a.mask[0]].mean() < 0.15
    # exact zeros exist in F (clipped background), reading A15
    assert (a.ch == 0).any()


def test_c3_weights_and_dropouts():
    cfg = WL.get_config("c3", T=30, H=64, W=80)
    wl = WL.generate("c3", cfg=cfg)
    assert wl.ch.shape == (1, 6, 30, 64, 80)
    assert abs(float(wl.w.sum()) - 1.0) < 1e-6 and (wl.w > 0).all()
    dropped = (wl.ch.reshape(6, 30, -1).max(axis=2) == 0)
    assert dropped.any()
    c2 = WL.generate("c2", cfg=WL.get_config("c2", T=30, H=64, W=80))
    np.testing.assert_array_equal(wl.mask, c2.mask)      # same blobs -> same clean mask


def test_c4_volumes_independent():
    cfg = WL.get_config("c4", B=3, T=5, H=64, W=64)
    wl = WL.generate("c4", cfg=cfg)
    assert wl.ch.shape == (3, 4, 5, 64, 64)
    one = WL.generate("c4", cfg=cfg, volumes=[2])
    np.testing.assert_array_equal(wl.ch[2:3], one.ch)
    assert not np.array_equal(wl.ch[0], wl.ch[1])


def test_c5_crop():
    cfg = WL.get_config("c5", T=4, H=120, W=200)
    wl = WL.generate("c5", cfg=cfg, t_range=(1, 3))
    assert wl.ch.shape == (1, 2, 2, 120, 200)
    assert np.isfinite(wl.ch).all()
