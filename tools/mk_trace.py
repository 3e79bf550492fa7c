"""Run one c2 solve with SFSEG_MK_TRACE and summarise the megakernel schedule (debug)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2212_08058_b200 as sf
import workloads as WL

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/mk_trace.csv"
cfg = WL.get_config("c2")
wl = WL.generate("c2", with_mask=False)
dev = torch.device("cuda")
g = sf.Gauss(cfg.sigma_t, cfg.sigma_s, cfg.radius_t, cfg.radius_s)
B, C, T, H, W = wl.ch.shape
s = sf.Solver((B, T, H, W), C, g, cfg.K, device=dev)
ch = torch.from_numpy(wl.ch).to(dev)
for _ in range(2):
    s.forward(ch, wl.w)
torch.cuda.synchronize()
os.environ["SFSEG_MK_TRACE"] = out
s.forward(ch, wl.w)
torch.cuda.synchronize()
os.environ["SFSEG_MK_TRACE"] = ""
d = np.loadtxt(out, delimiter=",", skiprows=2, dtype=np.float64)
t0 = d[:, 3].min()
grab, ready, done = d[:, 3] - t0, d[:, 4] - t0, d[:, 5] - t0
kind = d[:, 2]
span = done.max()
print(f"span {span/1e3:.1f} us, items {len(d)}")
for kd, name in ((0, "T"), (1, "S")):
    m = kind == kd
    print(f"{name}: n={m.sum()} wait mean {np.mean(ready[m]-grab[m])/1e3:.2f} us  work mean {np.mean(done[m]-ready[m])/1e3:.2f} us "
          f"work p90 {np.percentile(done[m]-ready[m], 90)/1e3:.2f} us  total CTA-time {np.sum(done[m]-grab[m])/1e6:.2f} ms")
ncta = len(np.unique(d[:, 1])) 
print("busy fraction (work / (span * 444)):", np.sum(done - ready) / (span * 444))
print("wait fraction:", np.sum(ready - grab) / (span * 444))
