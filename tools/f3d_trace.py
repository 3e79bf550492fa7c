"""Per-CTA timing of the fused 3D kernel on the probe workload (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2212_08058_b200 as sf
import workloads as WL

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/f3d_trace.csv"
cfg = WL.get_config("probe")
wl = WL.generate("probe", with_mask=False)
B, C, T, H, W = wl.ch.shape
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1
s = sf.Solver((B, T, H, W), C, sf.Gauss(cfg.sigma_t, cfg.sigma_s, cfg.radius_t, cfg.radius_s), K)
ch = torch.from_numpy(wl.ch).cuda()
for _ in range(3):
    s.forward(ch, wl.w)
os.environ["SFSEG_F3D_TRACE"] = out
s.forward(ch, wl.w)
os.environ["SFSEG_F3D_TRACE"] = ""
d = np.loadtxt(out, delimiter=",", skiprows=1)
t0 = d[:, 2].min()
dur = (d[:, 3] - d[:, 2]) / 1e3
ex = (d[:, 4] - d[:, 3]) / 1e3
st = (d[:, 2] - t0) / 1e3
print(f"span to last barrier {(d[:,3].max()-t0)/1e3:.1f} us, to last exit {(d[:,4].max()-t0)/1e3:.1f} us; "
      f"CTA body mean {dur.mean():.1f} max {dur.max():.1f}; bar->exit mean {ex.mean():.2f} max {ex.max():.2f}; "
      f"start max {st.max():.1f} us")
idx = np.argsort(-(d[:, 4]))[:5]
for i in idx:
    print(f"cta {int(d[i,0])} sm {int(d[i,1])} start {st[i]:.1f} body {dur[i]:.1f} exit {ex[i]:.2f}")
by_sm = {}
for r, du in zip(d, dur):
    by_sm.setdefault(int(r[1]), []).append(du)
print("CTAs per SM histogram:", np.bincount([len(v) for v in by_sm.values()]))
# event timing of the same solve (per launch, as bench.py measures it)
sf.profile_enable(True)
torch.cuda.synchronize()
s.forward(ch, wl.w)
torch.cuda.synchronize()
sf.profile_enable(False)
ms, n = sf.profile_read()["f3d"]
print(f"event timing: {n} f3d launches, {1e3 * ms / max(n, 1):.1f} us each")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
s.forward(ch, wl.w, check=False)
e1.record()
torch.cuda.synchronize()
print(f"whole solve (K={K}): {e0.elapsed_time(e1) * 1e3:.1f} us")
