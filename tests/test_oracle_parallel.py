"""The multi-process oracle driver (oracle/parallel.py) is the serial oracle split
into independent pieces: bitwise-equal results (CPU, not gpu)."""
import numpy as np

import oracle as O
from oracle import parallel as OP


def test_parallel_filter_bitwise_equals_serial():
    rng = np.random.default_rng(1)
    v = rng.random((9, 23, 31))
    gt, gs = O.gaussian_taps(1.5, 5), O.gaussian_taps(2.0, 6)
    with OP.ParallelFilter(v.shape, procs=3) as f:
        a = f(v, gt, gs, gs)
        b = f(v * 2.0, gt, gs, gs)
    assert np.array_equal(a, O.gaussian_filter(v, gt, gs, gs))
    assert np.array_equal(b, O.gaussian_filter(v * 2.0, gt, gs, gs))


def test_parallel_power_iterate_and_backward_equal_serial():
    rng = np.random.default_rng(2)
    ch = rng.random((2, 2, 6, 14, 17)) * 0.8 + 0.1
    w, b = [0.7, 0.4], 0.1
    gt, gs = O.gaussian_taps(1.0, 3), O.gaussian_taps(2.0, 6)
    F, _ = O.combine(ch, w, b, O.ACT_SIGMOID)
    xs, ss = O.power_iterate(F, gt, gs, 4)
    xp, sp = OP.power_iterate(F, gt, gs, 4, procs=2)
    assert np.array_equal(xs, xp)
    for key in ("gain", "rho", "nu"):
        assert np.array_equal(ss[key], sp[key])
    g = rng.normal(size=F.shape)
    dws, dbs = O.power_iterate_backward(ch, w, b, O.ACT_SIGMOID, gt, gs, 4, g)
    dwp, dbp = OP.power_iterate_backward(ch, w, b, O.ACT_SIGMOID, gt, gs, 4, g, procs=2)
    assert np.array_equal(dws, dwp) and dbs == dbp
