"""Run the tcgen05 spatial pass on small cases, one per process (a fault kills the context)."""
import subprocess, sys
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2212_08058_b200 as sf
B, T, H, W, r = map(int, sys.argv[1:6])
rng = np.random.default_rng(0)
ch = torch.from_numpy((rng.random((B, 1, T, H, W)) * 0.8 + 0.1).astype(np.float32)).cuda()
s = sf.Solver((B, T, H, W), 1, sf.Gauss(1.0, r / 3.0, 2, r), int(sys.argv[6]), algo=sf.ALGO_TWO_PASS_TCGEN05)
x = s.forward(ch, [1.0])
print("ok", float(x.sum()))
'''
for case in sys.argv[1:]:
    args = case.split(",")
    r = subprocess.run([sys.executable, "-c", code] + args, capture_output=True, text=True, timeout=120)
    print(case, "->", (r.stdout.strip() or r.stderr.strip().splitlines()[-1])[:200], flush=True)
