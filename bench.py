#!/usr/bin/env python
"""Benchmark of the SFSeg power-iteration hot path on B200 (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A "step" is one pass of the whole hot path over one synthetic volume (batch):
fused channel combine + K power iterations (temporal pass, fused spatial pass with
the F multiplies and the norm -- on the tensor pipe in fp32-class six-product split
bf16 for r_s >= 8 (A23), or the fused single-pass 3D kernel for small
radii) + final normalisation + per-frame threshold,
captured once and replayed as one CUDA graph per step (--graph 0: stream launches).

N=1: BASELINE.json configs[1] ("c2": 1x70x480x854, C=1, sigma_t=2, sigma_s=8,
15 iterations, tau=0.5).  N>1 (one process per GPU; `--gpus N` without torchrun
re-launches itself under torch.distributed.run): configs[4] ("c5": 1x512x1080x1920,
C=2, K=20) in time slabs of 512/N frames (NCCL halo exchange of r_t frames + fp64
norm allreduce every iteration, strong scaling); `--shard volume` runs configs[3]
("c4") with 64/N of its volumes per rank (no data-path collective, strong scaling).

metric: voxel-iterations/s = B*T*H*W*K per step, whole job.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "voxel-iterations/sec (T*H*W*iters/s)"
UNIT = "voxel-iterations/s"
ALU_PEAK_FMA_PER_CLK_PER_SM = 128     # FP32 lanes per SM (B200_PROFILING.md / blackwell guide)
SM_COUNT = 148
# legacy warp-level HMMA (mma.sync m16n8k16 bf16, fp32 accumulate) full-chip rate measured by
# tools/mma_microbench.cu on this pool's B200 (profiles/mma/mma.log): the ceiling of the
# tensor-core spatial pass's instruction choice
MMA_SYNC_BF16_TFLOPS = 555.6
TC_PRODUCTS = 6                       # bf16 products per tap (three planes per operand, A23)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.lower().startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self):
        def num(s):
            try:
                return float(s)
            except ValueError:
                return None
        sm = [num(r[1]) for r in self.rows if num(r[1]) is not None]
        mx = [num(r[2]) for r in self.rows if num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _default_config(args, world: int) -> str:
    if args.config:
        return args.config
    if world > 1 or getattr(args, "slab_at_1", False):
        return "c4" if args.shard == "volume" else "c5"
    return "c2"


def cpu_oracle_baseline(cfg_name: str, full_iters: bool = True, single_core: bool = True):
    """The oracle as it stands (oracle/: plain numpy f64), timed on this host's cores.

    multi-core: oracle.parallel (the serial oracle's filter split into independent frame /
      row pieces on every core -- bitwise the serial result) over ALL K iterations of the
      workload (c2: 15 iterations of 1x70x480x854), or over the first iteration(s) for the
      configs whose full solve exceeds ~30 s (c4: 1 of 10, c5: 1 iteration of a T=64 crop);
    single-core: one iteration of the serial oracle on the first 16 frames.
    Returns the cpu_baseline dict of the JSON line."""
    import numpy as np
    import oracle as O
    from oracle import parallel as OP
    import workloads as WL
    cfg = WL.get_config(cfg_name)
    gt, gs = O.gaussian_taps(cfg.sigma_t, cfg.radius_t), O.gaussian_taps(cfg.sigma_s, cfg.radius_s)
    cores = OP.host_cores()
    out = {"unit": UNIT, "cores": cores, "cpu_model": _cpu_model(), "kind": "oracle"}
    if cfg_name == "c5":
        wl = WL.generate(cfg_name, t_range=(0, 64), with_mask=False)
        iters, what = 1, "1 of 20 iterations of a 1x64x1080x1920 crop of c5"
    elif cfg_name == "c4":
        wl = WL.generate(cfg_name, volumes=range(16), with_mask=False)
        iters, what = 1, "1 of 10 iterations of 16 of the 64 c4 volumes"
    else:
        wl = WL.generate(cfg_name, with_mask=False)
        iters = cfg.K if full_iters else 1
        what = f"{iters} of {cfg.K} iterations of {cfg_name} {'x'.join(map(str, wl.ch.shape[:1] + wl.ch.shape[2:]))}"
    if cfg_name == "c2f":
        e = wl.extra
        S, U, F = O.combine_full(wl.ch, wl.w, wl.b, 0, e["f_ch"], e["wf"], 0.0, 0, e["p"])
        t0 = time.perf_counter()
        O.power_iterate_full(S, U, F, e["alpha"], gt, gs, 1)
        dt = time.perf_counter() - t0
        out.update(value=F.size / dt, cores=1, sample=f"1 of {cfg.K} iterations of the full operator (serial)",
                   seconds=dt)
        return out
    F, _ = O.combine(wl.ch, wl.w, wl.b, cfg.act)
    OP.power_iterate(F[:1, :min(F.shape[1], 8)], gt, gs, 1, procs=cores)   # pool start-up, imports
    t0 = time.perf_counter()
    OP.power_iterate(F, gt, gs, cfg.K, procs=cores, iters=iters)
    dt = time.perf_counter() - t0
    out.update(value=F.size * iters / dt, seconds=dt,
               sample=f"{what}, multi-process oracle (oracle/parallel.py) on {cores} cores; combine excluded")
    if single_core:
        crop = F[:1, :min(F.shape[1], 16)]
        t0 = time.perf_counter()
        O.power_iterate(crop, gt, gs, 1)
        d1 = time.perf_counter() - t0
        out["single_core"] = {"value": crop.size / d1, "seconds": d1,
                              "sample": f"1 iteration of the serial oracle on {'x'.join(map(str, crop.shape))}"}
    return out


def run_reference(args):
    """--impl reference: the oracle (the paper's method as plain f64 numpy) on the host cores,
    each step one power iteration of the workload (multi-process oracle), rank 0 only."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import numpy as np
    import oracle as O
    from oracle import parallel as OP
    import workloads as WL
    cfg_name = _default_config(args, ws)
    cfg = WL.get_config(cfg_name)
    if cfg_name == "c5":
        wl = WL.generate(cfg_name, t_range=(0, 64), with_mask=False)
        what = "one power iteration of a 1x64x1080x1920 crop of c5"
    elif cfg_name == "c4":
        wl = WL.generate(cfg_name, volumes=range(8), with_mask=False)
        what = "one power iteration of 8 of the 64 c4 volumes"
    else:
        wl = WL.generate(cfg_name if cfg_name != "c2f" else "c2", with_mask=False)
        what = f"one of the {cfg.K} power iterations of {cfg_name}"
    gt, gs = O.gaussian_taps(cfg.sigma_t, cfg.radius_t), O.gaussian_taps(cfg.sigma_s, cfg.radius_s)
    F, _ = O.combine(wl.ch, wl.w, wl.b, cfg.act)
    cores = OP.host_cores()
    total_t = 0.0
    with OP.ParallelFilter(F.shape[1:], cores) as filt:
        def one():   # y_1 = F * G(F * x_0), x_0 = F, and its norm (Eq.4/7/8)
            for b in range(F.shape[0]):
                y = F[b] * filt(F[b] * F[b], gt, gs, gs)
                float(np.sum(y * y))
        for _ in range(args.warmup):
            one()
        for _ in range(args.steps):
            t0 = time.perf_counter()
            one()
            total_t += time.perf_counter() - t0
    value = F.size * args.steps / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
        "higher_is_better": True, "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (workloads/ generator; DAVIS-2016-shaped blobs)",
        "config": {"workload": f"{cfg_name}: {cfg.note}", "shape": [cfg.B, cfg.T, cfg.H, cfg.W], "C": cfg.C,
                   "sigma_t": cfg.sigma_t, "sigma_s": cfg.sigma_s, "radius_t": cfg.radius_t,
                   "radius_s": cfg.radius_s, "iters": cfg.K},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "cpu_model": _cpu_model(), "kind": "oracle",
                         "sample": f"each step: {what} (multi-process oracle, oracle/parallel.py)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2212_08058_b200 as sf
    import workloads as WL

    world, rank, local = _dist()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sf.lib()

    cfg_name = _default_config(args, world)
    args.config = cfg_name
    algo = {"auto": sf.ALGO_AUTO, "tcgen05": sf.ALGO_TWO_PASS_TCGEN05, "mma": sf.ALGO_TWO_PASS_MMA_SYNC,
            "fp32": sf.ALGO_TWO_PASS_FP32,
            "f16": sf.ALGO_TWO_PASS_MMA_F16}[args.algo]
    cfg = WL.get_config(cfg_name)
    slab = (world > 1 or args.slab_at_1) and args.shard == "slab" and cfg_name != "c4"
    vshard = world > 1 and not slab      # independent volumes split across ranks (c4: 64/N each)
    K = cfg.K
    gauss = sf.Gauss(cfg.sigma_t, cfg.sigma_s, cfg.radius_t, cfg.radius_s)
    if slab:
        from paper_2212_08058_b200.dist import Comm, SlabSolver, broadcast_unique_id, slab_range
        t0, t1 = slab_range(cfg.T, world, rank)
        wl = WL.generate(args.config, t_range=(t0, t1), with_mask=False)
        uid = broadcast_unique_id(rank)
        comm = Comm(world, rank, local, uid)
    elif vshard:
        if cfg.B % world:
            raise SystemExit(f"{cfg_name}: {cfg.B} volumes do not split over {world} ranks")
        per = cfg.B // world
        wl = WL.generate(args.config, volumes=range(rank * per, (rank + 1) * per), with_mask=False)
    else:
        # c3 (SFSeg++ ensemble) times forward + backward (dL/dw for the MSE loss, reading A13)
        wl = WL.generate(args.config, with_mask=(args.config == "c3"))
    B, Cn, T, H, W = wl.ch.shape
    ch_host = torch.from_numpy(wl.ch).pin_memory()
    ch = ch_host.to(dev)
    if slab:
        solver = SlabSolver(comm, (B, T, H, W), cfg.T, t0, Cn, gauss, K, device=dev, algo=algo,
                            serial=args.slab_serial)
    else:
        solver = sf.Solver((B, T, H, W), Cn, gauss, K, device=dev, want_tape=(args.config == "c3"), algo=algo)
    full = args.config == "c2f" and not slab
    if full:   # the full SFSeg operator replaces the hot-path solve
        fsolver = sf.FullSolver((B, T, H, W), Cn, 2, gauss, K, device=dev)
        f_ch = torch.from_numpy(wl.extra["f_ch"]).to(dev)
    x = torch.empty((B, T, H, W), dtype=torch.float32, device=dev)
    mask = torch.empty((B, T, H, W), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    # the per-frame threshold (a9) is frame-local: each rank thresholds its own slab
    path_info = sf.forward_path((B, T, H, W), gauss, algo)
    path_tc = path_info[0] in (sf.PATH_TWO_PASS_TC, sf.PATH_TWO_PASS_TCGEN05, sf.PATH_TWO_PASS_TC_F16)
    path_f16 = path_info[0] == sf.PATH_TWO_PASS_TC_F16
    path_t6 = path_info[0] == sf.PATH_TWO_PASS_TCGEN05
    thr_solver = sf.Solver((B, T, H, W), Cn, gauss, K, device=dev) if slab else solver

    train = args.config == "c3" and not slab
    if train:
        # loss gradient of reading A13 (harness side, outside the ABI): L = mean (x_K - m_hat)^2
        m_hat = torch.from_numpy(wl.mask.astype(np.float32)).to(dev)
        m_hat /= torch.linalg.vector_norm(m_hat.double()).float()
        nvox = float(x.numel())
        grad = torch.empty_like(x)
        last_dw = {}

    def step():
        if full:
            e = wl.extra
            fsolver.forward(ch, wl.w, f_ch, e["wf"], e["p"], e["alpha"], x_out=x, check=False)
            thr_solver.threshold(x, cfg.tau, sf.THR_PER_FRAME_MAX, mask=mask)
            return
        solver.forward(ch, wl.w, wl.b, cfg.act, x_out=x, check=False)
        if train:
            torch.sub(x, m_hat, out=grad).mul_(2.0 / nvox)
            last_dw["dw"], last_dw["db"] = solver.backward(ch, wl.w, grad, wl.b, cfg.act)
        thr_solver.threshold(x, cfg.tau, sf.THR_PER_FRAME_MAX, mask=mask)

    for _ in range(max(args.warmup, 0)):
        step()
    (fsolver.forward(ch, wl.w, f_ch, wl.extra["wf"], wl.extra["p"], wl.extra["alpha"], x_out=x) if full
     else solver.sync())   # raises on a device-detected error
    timed_step = step
    graph = None
    if args.graph and not slab and not train:
        # the whole step (every kernel of combine, K iterations, final scale, threshold) captured
        # once into a CUDA graph and replayed: one launch per step from the host
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            with torch.cuda.graph(graph, stream=cap):
                step()
        stream.wait_stream(cap)
        torch.cuda.synchronize(dev)
        timed_step = graph.replay
        # the replayed graph must produce exactly what the stream launches produce (the
        # path is deterministic: fixed-order reductions), so check it bitwise once
        step()
        torch.cuda.synchronize(dev)
        ref_x, ref_m = x.clone(), mask.clone()
        for _ in range(2):
            timed_step()
        torch.cuda.synchronize(dev)
        if not (torch.equal(x, ref_x) and torch.equal(mask, ref_m)):
            raise RuntimeError("CUDA graph replay result differs from the stream-launched step")
        del ref_x, ref_m

    clocks = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[0])
                          if os.environ.get("CUDA_VISIBLE_DEVICES", "").isdigit() else local)
    clocks.start()
    time.sleep(0.2)
    # inputs (ch 115 MB + F/p/v 344 MB at c2) exceed the 126 MB L2: no flush needed
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]   # per-step ends (median / min)
    e0.record(stream)
    for i in range(args.steps):
        timed_step()
        ev[i].record(stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    step_ms = [e0.elapsed_time(ev[0])] + [ev[i - 1].elapsed_time(ev[i]) for i in range(1, args.steps)]
    (fsolver if full else solver).sync()   # device errors of the timed steps (sticky error word)
    if world > 1:
        dist.barrier()
    time.sleep(0.1)
    clocks.stop()
    ms = e0.elapsed_time(e1)
    # per-kernel durations for the roofline: a few extra steps with every pass launch bracketed
    # by CUDA events on its stream (kept out of the timed region: events between launches
    # defeat the programmatic dependent launch that overlaps a kernel's prologue with the
    # previous kernel's tail)
    prof_steps = max(1, min(3, args.steps))
    profiler = sf.Profiler()   # caller-owned event timing passed in the solvers' options
    for so in (solver, fsolver if full else None):
        if so is not None:
            so.profiler = profiler
    for _ in range(prof_steps):
        step()
    torch.cuda.synchronize(dev)
    for so in (solver, fsolver if full else None):
        if so is not None:
            so.profiler = None
    prof = profiler.read()
    profiler.close()
    prof = {k: (v[0] * args.steps / prof_steps, int(round(v[1] * args.steps / prof_steps))) for k, v in prof.items()}
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())

    vox = B * T * H * W
    units_per_step = vox * K
    if slab:   # strong scaling: the ranks together process one volume per step
        value = B * cfg.T * H * W * K * args.steps / (ms_max / 1e3)
    else:
        value = world * units_per_step * args.steps / (ms_max / 1e3)

    # ---------------------------------------------------------------- roofline of the dominant kernel
    peaks, peaks_src = _peaks()
    sp_ms, sp_n = prof["spass"]
    tp_ms, tp_n = prof["tpass"]
    sp_avg_s = sp_ms / max(sp_n, 1) / 1e3
    tp_avg_s = tp_ms / max(tp_n, 1) / 1e3
    r_s, r_t = cfg.radius_s, cfg.radius_t
    fma_per_vox = 2 * (2 * r_s + 1) + (0 if full else 3)   # x taps + y taps (+ F*u, F*y, y*y)
    flops_per_launch = 2.0 * fma_per_vox * vox
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak_tflops = SM_COUNT * ALU_PEAK_FMA_PER_CLK_PER_SM * 2 * sm_max * 1e6 / 1e12
    achieved = flops_per_launch / sp_avg_s / 1e12 if sp_n else None
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            # {config: {"spass": {"dram_bytes_per_launch": ..., "source": "profiles/<round>/..."}}}
            traffic = json.load(open(tfile)).get(args.config, {}).get("spass", {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    # temporal pass: read p, write v (8 B/voxel); the full operator's stacked pass reads a and F
    # and writes three outputs (20 B/voxel)
    tp_bytes = (20.0 if full else 8.0) * B * T * H * W
    f3_ms, f3_n = prof["f3d"]
    if f3_n:
        # small radii: the fused single-pass 3D kernel is the whole iteration (HBM-bound):
        # algorithmic bytes = read p_{k-1} + read F + write p_k = 12 B per voxel
        f3_avg_s = f3_ms / f3_n / 1e3
        f3_bytes = 12.0 * vox
        f3_traffic = None
        try:
            f3_traffic = json.load(open(tfile)).get(args.config, {}).get("f3d", {}).get("dram_bytes_per_launch")
        except Exception:
            pass
        roofline = {
            "kernel": f"f3d_kernel<RT={r_t}, R={r_s}> (fused t/x/y Gaussian + F multiplies + norm, one pass)",
            "bound": "hbm", "achieved": f3_bytes / f3_avg_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": f3_bytes / f3_avg_s / 1e9 / hbm_peak, "traffic": f3_traffic,
            "peak_source": f"{peaks_src} hbm_gbs (MEASURED_PEAKS.json)",
            "algorithmic_bytes_per_launch": f3_bytes, "launch_ms": f3_avg_s * 1e3, "launches": f3_n,
            "share_of_step": f3_ms / ms if ms > 0 else None,
            "path_hbm_frac_algorithmic_12B": 12.0 * value / world / 1e9 / hbm_peak,
        }
    elif path_tc:
        # tensor-core spatial pass: bound by HBM at speed of light (12 B/voxel: read v and F,
        # write p = 53 us at c2) rather than by the tensor pipe (its banded bf16x3 products
        # take 13.5 us at the measured dense bf16 peak); both reported
        RSc = path_info[2]
        NB_ = -(-H // 32)
        if path_t6:
            # per (frame, 128-column strip): NB6 64-row y-blocks (3 x NKY MMAs) and NB6 + 1 64-row
            # x-blocks (3 x NKX MMAs), M=128 N=64 K=16 (262144 flop); partial segments at CTA-range
            # boundaries add a few x-blocks (not counted)
            ra6 = 8 * ((RSc + 7) // 8)
            nkx6 = (128 + 2 * ra6) // 16
            nky6 = 4 + 2 * ((RSc + 15) // 16)
            nb6, s6 = -(-H // 64), -(-W // 128)
            tc_flops = float(B * T * s6) * 3 * (nb6 * nky6 + (nb6 + 1) * nkx6) * 262144
            kname = (f"spass_tc6_kernel<R={RSc}> (tcgen05.mma kind::f16 M=128 N=64, accumulators in TMEM: x-pass "
                     f"from SWIZZLE_128B TMA boxes of the fp16 planes of v, y-pass A operand in TMEM; two fp16 "
                     f"planes x three products per tap (fp32-class) + F multiplies + norm + max |p|)")
            tc_ceiling = float(peaks.get("bf16_tflops", 2250.0))
        else:
            ra = (RSc + 3) // 4 * 4
            nkx, nky = (16 + ra + RSc + 15) // 16, (16 + 2 * RSc + 15) // 16
            S_ = -(-W // 64)
            # mma.sync m16n8k16 (4096 flop): 16 x 6 HMMA per k step and warp, 4 warps per 32 x 64 block
            nprod = 3 if path_f16 else TC_PRODUCTS
            tc_flops = float(B * T * S_ * NB_) * 16 * nprod * (nkx + nky) * 4096
            kname = (f"spass_tc_kernel<R={RSc}> (mma.sync m16n8k16; x/y Gaussian as banded Toeplitz products, "
                     + ("two fp16 planes x three products per tap, per-volume power-of-two range scaling"
                        if path_f16 else "three bf16 planes x six products per tap (fp32-class)")
                     + " + F multiplies + norm)")
            tc_ceiling = MMA_SYNC_BF16_TFLOPS
        # read v (+ F unless the full operator's plain pass), write p (+ the tape u for training)
        sp_bytes = (8.0 + (0.0 if full else 4.0) + (4.0 if args.config == "c3" else 0.0)) * vox
        bf16_peak = float(peaks.get("bf16_tflops", 2250.0))
        try:
            tc_traffic = json.load(open(tfile)).get(args.config, {}).get("spass_tc", {}).get("dram_bytes_per_launch")
        except Exception:
            tc_traffic = None
        roofline = {
            "kernel": kname,
            "bound": "hbm", "achieved": sp_bytes / sp_avg_s / 1e9 if sp_n else None, "peak": hbm_peak,
            "unit": "GB/s", "frac": (sp_bytes / sp_avg_s / 1e9 / hbm_peak) if sp_n else None,
            "traffic": tc_traffic,
            "peak_source": f"{peaks_src} hbm_gbs (MEASURED_PEAKS.json)",
            "algorithmic_bytes_per_launch": sp_bytes,
            "launch_ms": sp_avg_s * 1e3, "launches": sp_n,
            "share_of_step": sp_ms / ms if ms > 0 else None,
            "tensor": {"hmma_flops_per_launch": tc_flops,
                       "achieved_TFLOPs": tc_flops / sp_avg_s / 1e12 if sp_n else None,
                       "peak_bf16_TFLOPs": bf16_peak, "peak_source": f"{peaks_src} bf16_tflops",
                       "frac": (tc_flops / sp_avg_s / 1e12 / bf16_peak) if sp_n else None,
                       "instruction_ceiling_TFLOPs": tc_ceiling,
                       "instruction_frac": (tc_flops / sp_avg_s / 1e12 / tc_ceiling) if sp_n else None,
                       "useful_fp32_TFLOPs": flops_per_launch / sp_avg_s / 1e12 if sp_n else None},
            "tpass": {"launch_ms": tp_avg_s * 1e3, "launches": tp_n,
                      "achieved_GBps": tp_bytes / tp_avg_s / 1e9 if tp_n else None, "peak_GBps": hbm_peak,
                      "bound": "hbm"},
            "path_hbm_frac_algorithmic_12B": 12.0 * value / world / 1e9 / hbm_peak,
        }
    else:
        roofline = {
            "kernel": f"spass_kernel<R={r_s}> (fused x/y Gaussian + F multiplies + norm)",
            "bound": "alu", "achieved": achieved, "peak": alu_peak_tflops, "unit": "TFLOP/s",
            "frac": (achieved / alu_peak_tflops) if achieved else None, "traffic": traffic,
            "peak_source": f"derived: {SM_COUNT} SM x {ALU_PEAK_FMA_PER_CLK_PER_SM} FP32 FMA/clk x 2 x "
                           f"{sm_max:.0f} MHz ({peaks_src} sm_max_mhz)",
            "algorithmic_flops_per_launch": flops_per_launch,
            "launch_ms": sp_avg_s * 1e3, "launches": sp_n,
            "share_of_step": sp_ms / ms if ms > 0 else None,
            "tpass": {"launch_ms": tp_avg_s * 1e3, "launches": tp_n,
                      "achieved_GBps": tp_bytes / tp_avg_s / 1e9 if tp_n else None, "peak_GBps": hbm_peak,
                      "bound": "hbm"},
            "path_hbm_frac_algorithmic_12B": 12.0 * value / world / 1e9 / hbm_peak,
        }
    if roofline.get("traffic"):   # ncu DRAM bytes per voxel of one launch (vs the algorithmic bytes)
        roofline["traffic_bytes_per_voxel"] = roofline["traffic"] / vox
    # our kernels launched in the timed region: the passes (counted by the library's
    # event instrumentation) + combine, final scale, frame max and threshold per step
    n_launch = int(sp_n + tp_n + f3_n + 4 * args.steps)
    if full:
        n_launch += K * args.steps   # the full operator's per-iteration epilogue kernel

    # ---------------------------------------------------------------- e2e through the C ABI with host buffers
    e2e = None
    if not args.no_e2e and not slab and not full:
        # end to end over pinned HOST buffers through ONE library call per batch of volumes
        # (sfseg_solve_host_batch): the library pipelines the H2D copy of volume i+1 and the D2H
        # copy of volume i-1 under the solve of volume i (one cudaMemcpyAsync per copy, caller's
        # copy streams); every volume copies its full input in and its x + mask out.
        e2e_steps = max(2, min(args.steps, 10))
        x_hosts = [torch.empty((B, T, H, W), dtype=torch.float32).pin_memory() for _ in range(e2e_steps)]
        m_hosts = [torch.empty((B, T, H, W), dtype=torch.uint8).pin_memory() for _ in range(e2e_steps)]
        hb = sf.HostBatch(solver)
        hb.run([ch_host] * 2, wl.w, cfg.tau, x_hosts[:2], m_hosts[:2], wl.b, cfg.act)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        hb.run([ch_host] * e2e_steps, wl.w, cfg.tau, x_hosts, m_hosts, wl.b, cfg.act)
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": world * units_per_step * e2e_steps / float(dt.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(ch_host.numel() * 4),
               "d2h_bytes_per_step": int(x_hosts[0].numel() * 4 + m_hosts[0].numel()),
               "steps": e2e_steps,
               "api": "sfseg_solve_host_batch (C ABI): H2D of pinned host channels, solve, threshold, D2H of "
                      "x_K and the mask per volume, copies pipelined inside the library on two copy streams"}
        del hb
        # the unpipelined single call (sfseg_solve_host: H2D, solve, threshold, D2H, sync) for reference
        d_ch = torch.empty_like(ch)
        sf.solve_host(ch_host, wl.w, gauss, K, cfg.tau, solver, d_ch, x, mask, x_hosts[0], m_hosts[0])
        t0 = time.perf_counter()
        for _ in range(2):
            sf.solve_host(ch_host, wl.w, gauss, K, cfg.tau, solver, d_ch, x, mask, x_hosts[0], m_hosts[0])
        e2e["unpipelined_value"] = units_per_step * 2 / (time.perf_counter() - t0)
        del x_hosts, m_hosts, d_ch

    # ---------------------------------------------------------------- the same step on FP32 FMA arithmetic only
    fp32_arm = None
    if path_tc and world == 1 and not slab and not full and not train and not args.no_fp32_arm:
        # north_star asks for fp32 arithmetic; the default spatial pass runs on the tensor pipe in split
        # fp16 operands (fp32-class, see "arithmetic").  Time the SAME step (combine, K iterations, final
        # scale, threshold) with every pass on FP32 FFMA (SFSEG_ALGO_TWO_PASS_FP32) in the same run, and
        # report how far the two x_K are apart.
        x_def = x.clone()
        s32 = sf.Solver((B, T, H, W), Cn, gauss, K, device=dev, algo=sf.ALGO_TWO_PASS_FP32)

        def step32():
            s32.forward(ch, wl.w, wl.b, cfg.act, x_out=x, check=False)
            thr_solver.threshold(x, cfg.tau, sf.THR_PER_FRAME_MAX, mask=mask)

        n32 = max(2, min(args.steps, 10))
        for _ in range(max(args.warmup, 3)):
            step32()
        s32.sync()
        torch.cuda.synchronize(dev)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(n32):
            step32()
        a1.record(stream)
        torch.cuda.synchronize(dev)
        s32.sync()
        ms32 = a0.elapsed_time(a1) / n32
        diff = float(torch.linalg.vector_norm((x.double() - x_def.double())) / torch.linalg.vector_norm(x.double()))
        fp32_arm = {"value": units_per_step / (ms32 * 1e-3), "unit": UNIT, "ms_per_step": ms32, "steps": n32,
                    "dtype": "f32", "algo": "SFSEG_ALGO_TWO_PASS_FP32 (temporal pass + FP32-FMA spatial pass, "
                                            "stream launches)",
                    "x_K_rel_l2_vs_default_path": diff}
        del s32, x_def

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_baseline(args.config)

    if path_t6 or path_f16:
        arith = ("fp32 FFMA everywhere except the forward spatial pass of r_s >= 8, which runs on the tensor "
                 "pipe with each operand and tap split into two fp16 planes (22 significant bits, per-volume "
                 "power-of-two range scaling) and three products per tap, fp32 accumulation (fp32-class: x_K "
                 "error vs the f64 oracle within 2x the FP32-FMA pass's at full c2, tests/test_gpu_fullsize.py; "
                 "DESIGN.md A25)")
    elif path_tc:
        arith = ("fp32 FFMA everywhere except the forward spatial pass of r_s >= 8, which runs on the tensor "
                 "pipe with each operand and tap split into three bf16 planes and six products per tap "
                 "(fp32-class; DESIGN.md A23)")
    else:
        arith = "fp32 FFMA throughout"
    # the arithmetic types that run: fp32 everywhere, except the tensor-core spatial pass's split operands
    dtype = ("f32+f16x2split" if (path_t6 or path_f16) else "f32+bf16x3split" if path_tc else "f32")
    if rank == 0:
        ck = clocks.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if (slab or vshard) else "weak", "vs_baseline": None, "dtype": dtype,
            "data": "synthetic (workloads/ generator; DAVIS-2016-shaped blobs, seed 0)",
            "config": {"workload": f"{args.config}: {cfg.note}", "shape": [B, T, H, W], "C": Cn,
                       "sigma_t": cfg.sigma_t, "sigma_s": cfg.sigma_s, "radius_t": r_t, "radius_s": r_s,
                       "iters": K, "tau": cfg.tau,
                       "parallelism": (f"time-slab x{world} (NCCL halo r_t frames + fp64 norm allreduce / iter; "
                                       f"NCCL communicator of {comm.nranks} ranks)" if slab else
                                       f"volume shards x{world} ({B} of {cfg.B} volumes per rank, no collective)"
                                       if vshard else "one GPU"),
                       "arithmetic": arith,
                       "l2": "inputs > L2 (ch 115 MB + F/p/v 344 MB vs 126 MB L2); no flush",
                       "launch": "one CUDA graph per step" if graph is not None else "stream launches"},
            "step_ms": {"median": float(statistics.median(step_ms)), "min": float(min(step_ms)),
                        "max": float(max(step_ms)), "rank": rank},
            "once_per_solve_ms_per_step": prof["once"][0] / args.steps,   # combine + final scale (events)
            "path_hbm_frac_12B_nameplate_8TBs": 12.0 * value / world / 1e9 / 8000.0,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "fp32_ffma_arm": fp32_arm,
            "gpu_launches": n_launch + (int(prof["backward"][1]) + 2 * args.steps if train else 0),
            "clocks": {k: ck[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")},
            "clock_samples": ck["samples"],
        }
        if train:
            bw_ms, bw_n = prof["backward"]
            line["step"] = ("forward (K iterations, tape) + MSE loss gradient (torch, harness) + backward "
                            "dL/dw (sfseg_power_iterate_backward) + threshold; value counts the forward's "
                            "K voxel-iterations only")
            line["backward"] = {"pass_ms_per_step": bw_ms / args.steps, "pass_launches": int(bw_n),
                                "dL_dw": last_dw.get("dw"), "dL_db": last_dw.get("db")}
            if e2e:
                e2e["api"] += " -- forward + threshold only"
        print(json.dumps(line), flush=True)
    if slab:
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None, choices=["c1", "c2", "c3", "c4", "c5", "probe", "c2f"],
                    help="default: c2 at N=1, c5 (time slabs) at N>1, c4 with --shard volume")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-fp32-arm", action="store_true",
                    help="skip the FP32-FMA-only arm of the same step (reported as fp32_ffma_arm)")
    ap.add_argument("--algo", default="auto", choices=["auto", "tcgen05", "mma", "fp32", "f16"],
                    help="forward path (sfseg_options.algo): auto, the tcgen05/TMEM spatial pass, the mma.sync "
                         "one, or the FP32-FMA one")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", type=int, default=1,
                    help="1 (default): replay the step as one captured CUDA graph (measured 2-3 %% faster than "
                         "stream launches at c2/probe/c2f, profiles/tc/ab_graph.txt); 0: stream launches. "
                         "Multi-rank time slabs and the training step (c3) always use stream launches")
    ap.add_argument("--slab-at-1", action="store_true",
                    help="run the time-slab path (NCCL communicator, overlapped schedule) with one rank: the N=1 "
                         "dry run of the multi-GPU launcher")
    ap.add_argument("--slab-serial", action="store_true",
                    help="time slabs: the serial schedule instead of the overlapped one (A/B)")
    ap.add_argument("--shard", default="slab", choices=["volume", "slab"],
                    help="N>1: time slabs of one volume with NCCL halos (default, c5) or the c4 batch split by "
                         "volume (64/N per rank, no collective)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run (rendezvous on 127.0.0.1)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus != ws and args.impl == "ours":
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; using {ws}", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
