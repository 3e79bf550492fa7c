"""Run one forward solve for a given shape/radii (debug helper; one process per case)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_08058_b200 as sf

B, T, H, W, rt, rs = (int(v) for v in sys.argv[1:7])
ch = torch.rand((B, 1, T, H, W), device="cuda") * 0.8 + 0.1
s = sf.Solver((B, T, H, W), 1, sf.Gauss(max(rt, 1) / 3, max(rs, 1) / 3, rt, rs), 3)
try:
    x = s.forward(ch, [1.0])
    print("OK", sys.argv[1:7], float(x.norm()))
except Exception as e:
    print("ERR", sys.argv[1:7], e)
