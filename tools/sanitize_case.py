"""Small cases of every kernel family for compute-sanitizer (one tool per gpurun call):

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2212_08058_b200 as sf
import workloads as WL

dev = torch.device("cuda")
rng = np.random.default_rng(0)


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


# f3d (c1) + threshold
wl = WL.generate("c1")
c = wl.cfg
s = sf.Solver((1, 8, 32, 32), 1, sf.Gauss(c.sigma_t, c.sigma_s, c.radius_t, c.radius_s), c.K)
x = s.forward(T(wl.ch), wl.w, want_rayleigh=True)
s.threshold(x, 0.5)
# two-pass large radius on a ragged crop, with tape + backward
cfg = WL.get_config("c3", T=10, H=70, W=150)
wl = WL.generate("c3", cfg=cfg)
B, C, TT, H, W = wl.ch.shape
g = sf.Gauss(2.0, 8.0, 6, 24)
s = sf.Solver((B, TT, H, W), C, g, 4, want_tape=True)
x = s.forward(T(wl.ch), wl.w, want_rayleigh=True)
dw, db = s.backward(T(wl.ch), wl.w, T(rng.normal(size=x.shape).astype(np.float32)))
# two-pass forced on small radii
sf.Solver((2, 5, 33, 90), 1, sf.Gauss(1.0, 1.0, 3, 3), 3, algo=sf.ALGO_TWO_PASS).forward(
    T(rng.random((2, 1, 5, 33, 90)).astype(np.float32)), [1.0])
# full operator
fs = sf.FullSolver((1, 6, 40, 100), 1, 2, g, 3)
fs.forward(T(rng.random((1, 1, 6, 40, 100)).astype(np.float32)), [1.0],
           T(rng.random((1, 2, 6, 40, 100)).astype(np.float32)), [0.5, 0.5], 0.2, 1.0)
# time-slab emulation (3 slabs on one GPU)
sf.power_iterate_slabs(T(rng.random((1, 1, 21, 40, 90)).astype(np.float32)), [1.0], g, 3, 3)
torch.cuda.synchronize()
print("sanitize cases done", dw, db)
