"""Pins of the online / sub-window oracle (oracle/online.py)."""
import numpy as np
import pytest

import oracle as O


def test_window_starts_cover_every_frame():
    """every frame is covered; windows are q long (or the whole video)."""
    for T, q, s in ((20, 7, 3), (20, 7, 7), (21, 5, 5), (10, 12, 4), (33, 13, 1)):
        st = O.window_starts(T, q, s)
        cov = np.zeros(T, int)
        for a in st:
            cov[a:min(T, a + q)] += 1
            assert min(T, a + q) - a == min(q, T)
        assert (cov >= 1).all() and st[0] == 0 and min(T, st[-1] + q) == T


def test_online_whole_video_equals_offline():
    """q >= T gives exactly the offline solve."""
    rng = np.random.default_rng(0)
    F = rng.random((2, 9, 10, 12))
    gt, gs = O.gaussian_taps(1.0, 3), O.gaussian_taps(1.5, 4)
    x_on = O.power_iterate_online(F, gt, gs, 6, 9, 3)
    x_off, _ = O.power_iterate(F, gt, gs, 6)
    assert np.abs(x_on - x_off).max() == 0.0


def test_online_disjoint_windows_are_independent_crops():
    """q = 2t+1 with stride = q: no overlap, each window is a cold-started crop solve."""
    rng = np.random.default_rng(1)
    F = rng.random((1, 21, 8, 9))
    gt, gs = O.gaussian_taps(1.0, 3), O.gaussian_taps(1.0, 2)
    q = 7
    x_on = O.power_iterate_online(F, gt, gs, 5, q, q)
    for a in range(0, 21, q):
        xc, _ = O.power_iterate(F[:, a:a + q], gt, gs, 5)
        assert np.abs(x_on[:, a:a + q] - xc).max() <= 1e-15


def test_online_static_video_close_to_offline():
    """S:237 / P:386 ("almost identical results"): a static video, q = 5, stride 1 --
    per-frame thresholded masks agree with the offline solve on >= 99 % of pixels."""
    rng = np.random.default_rng(2)
    frame = np.zeros((24, 30))
    frame[6:18, 8:22] = 0.9
    F = np.clip(frame[None, None] + rng.normal(0, 0.03, (1, 16, 24, 30)), 0, 1)
    gt, gs = O.gaussian_taps(1.0, 2), O.gaussian_taps(2.0, 6)
    x_on = O.power_iterate_online(F, gt, gs, 20, 5, 1)
    x_off, _ = O.power_iterate(F, gt, gs, 20)
    m_on, m_off = O.threshold(x_on, 0.5), O.threshold(x_off, 0.5)
    assert (m_on == m_off).mean() >= 0.99
