"""Debug harness for the tcgen05 spatial pass (spass_tc6.cuh): each case in its own process
(a trap kills the context), x_K of the tcgen05 path against the mma.sync fp16 path, with the
rows / columns where they disagree.   python tools/t6_debug.py B,T,H,W,r,K[,rayleigh] ..."""
import subprocess
import sys

code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2212_08058_b200 as sf
B, T, H, W, r, K = map(int, sys.argv[1:7])
ray = len(sys.argv) > 7 and sys.argv[7] == "1"
rng = np.random.default_rng(0)
ch = torch.from_numpy((rng.random((B, 1, T, H, W)) * 0.8 + 0.1).astype(np.float32)).cuda()
g = sf.Gauss(1.0, r / 3.0, 2, r)
xs = {}
for name, algo in (("t6", sf.ALGO_TWO_PASS_TCGEN05), ("mma", sf.ALGO_TWO_PASS_MMA_F16)):
    s = sf.Solver((B, T, H, W), 1, g, K, algo=algo)
    xs[name] = s.forward(ch, [1.0], want_rayleigh=ray).cpu().numpy().astype(np.float64)
    xs[name + "_st"] = s.stats.cpu().numpy()
a, b = xs["t6"], xs["mma"]
rel = np.linalg.norm(a - b) / np.linalg.norm(b)
d = np.abs(a - b) / np.abs(b).max()
bad = np.argwhere(d > 1e-5)
msg = f"rel {rel:.3e} maxd {d.max():.3e} nbad {len(bad)} nu {xs['t6_st'][0, :, 0]} vs {xs['mma_st'][0, :, 0]}"
if len(bad):
    msg += f" rows {bad[:, 2].min()}..{bad[:, 2].max()} cols {bad[:, 3].min()}..{bad[:, 3].max()} frames {np.unique(bad[:, 1])[:8]}"
    i = np.unravel_index(np.argmax(d), d.shape)
    msg += f" worst {i} t6 {a[i]:.6e} mma {b[i]:.6e}"
print(msg)
'''
for case in sys.argv[1:]:
    args = case.split(",")
    r = subprocess.run([sys.executable, "-c", code] + args, capture_output=True, text=True, timeout=300)
    out = r.stdout.strip() or "\n".join(r.stderr.strip().splitlines()[-3:])
    print(case, "->", out[:1500], flush=True)
