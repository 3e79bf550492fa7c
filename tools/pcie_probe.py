"""Host<->device copy bandwidth of the box (pinned memory), alone and both directions at once:
the bound of bench.py's `e2e` line (c2: 115 MB in, 143 MB out per volume).  Prints one JSON line.
    python tools/pcie_probe.py [MB]
"""
import json
import sys

import torch


def timed(fn, streams, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0 = [torch.cuda.Event(enable_timing=True) for _ in streams]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in streams]
    for s, e in zip(streams, e0):
        e.record(s)
    for _ in range(reps):
        fn()
    for s, e in zip(streams, e1):
        e.record(s)
    torch.cuda.synchronize()
    return max(a.elapsed_time(b) for a, b in zip(e0, e1)) / reps


def main():
    mb = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    n = mb * (1 << 20)
    dev = torch.device("cuda:0")
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device=dev)
    d_out = torch.empty(n, dtype=torch.uint8, device=dev)
    si, so = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def h2d():
        with torch.cuda.stream(si):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(so):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()

    t_in, t_out, t_both = timed(h2d, [si]), timed(d2h, [so]), timed(both, [si, so])
    gb = n / 1e9
    print(json.dumps({"mb": mb, "h2d_gbs": gb / (t_in * 1e-3), "d2h_gbs": gb / (t_out * 1e-3),
                      "both_each_gbs": gb / (t_both * 1e-3),
                      "c2_e2e_bound_voxel_iter_s": 28694400 * 15 / (143472000 / (gb / (t_both * 1e-3)) / 1e9)}))


if __name__ == "__main__":
    main()
