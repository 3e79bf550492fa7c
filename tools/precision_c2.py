"""Full-size c2 precision of the forward paths against the multi-process oracle:
x_K relative L2 and the per-frame bound max|x - x_orc| / max|x_orc| for the
tensor-core spatial pass (default two-pass plan) and the FP32-FMA spatial pass.
Prints one JSON line.  (Measurement tool; run on a GPU box.)"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
from oracle import parallel as OP  # noqa: E402
import paper_2212_08058_b200 as sf  # noqa: E402
import workloads as WL  # noqa: E402


def frame_err(x, xo):
    d = np.abs(x.astype(np.float64) - xo).reshape(xo.shape[0], xo.shape[1], -1).max(-1)
    m = np.abs(xo).reshape(xo.shape[0], xo.shape[1], -1).max(-1)
    return float((d / m).max())


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    wl = WL.generate(name)
    c = wl.cfg
    g = sf.Gauss(c.sigma_t, c.sigma_s, c.radius_t, c.radius_s)
    ch = torch.from_numpy(wl.ch).cuda()
    out = {"config": name, "cores": OP.host_cores()}
    t0 = time.time()
    F, _ = O.combine(wl.ch, wl.w)
    xo, sto = OP.power_iterate(F, O.gaussian_taps(c.sigma_t, c.radius_t), O.gaussian_taps(c.sigma_s, c.radius_s), c.K)
    out["oracle_s"] = time.time() - t0
    for tag, algo in (("tc", sf.ALGO_TWO_PASS_MMA_SYNC), ("tcgen05", sf.ALGO_TWO_PASS_TCGEN05),
                      ("f16", sf.ALGO_TWO_PASS_MMA_F16), ("fp32", sf.ALGO_TWO_PASS_FP32)):
        s = sf.Solver((c.B, c.T, c.H, c.W), c.C, g, c.K, algo=algo)
        x = s.forward(ch, wl.w).cpu().numpy()
        st = s.stats.cpu().numpy()
        out[tag] = {"rel_l2": float(np.linalg.norm(x - xo) / np.linalg.norm(xo)), "frame_max": frame_err(x, xo),
                    "gain_rel": float(np.abs(st[..., 1] / sto["gain"] - 1).max())}
    out["tc_over_fp32_l2"] = out["tc"]["rel_l2"] / out["fp32"]["rel_l2"]
    out["tcgen05_over_fp32_l2"] = out["tcgen05"]["rel_l2"] / out["fp32"]["rel_l2"]
    out["f16_over_fp32_l2"] = out["f16"]["rel_l2"] / out["fp32"]["rel_l2"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
