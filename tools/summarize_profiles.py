"""Summarise one gpurun_out/<tag> directory into profiles/<tag>/ (tracked evidence).

    python tools/summarize_profiles.py gpurun_out/r01a profiles/r01a

Copies the bench JSON lines, microbenchmark logs and test logs; turns the ncu
launch list into a per-kernel table (count, mean us, share of the step); and
extracts the key raw metrics of every `--set full` capture (*.ncu-rep) into
<name>_ncu.txt, plus a JSON of DRAM bytes per launch (ncu_traffic.json) that
bench.py reads for the roofline `traffic` field.
"""
import collections
import csv
import glob
import io
import json
import os
import shutil
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.sum", "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "smsp__average_warp_latency_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "smsp__pcsamp_warps_issue_stalled_not_selected",
    "smsp__pcsamp_warps_issue_stalled_selected", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_dispatch_stall",
    "smsp__pcsamp_warps_issue_stalled_no_instructions", "smsp__pcsamp_warps_issue_stalled_membar",
    "smsp__pcsamp_warps_issue_stalled_sleeping", "smsp__pcsamp_warps_issue_stalled_drain",
]


def launches_table(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    if not rows:
        return ""
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = collections.OrderedDict()
    for r in rows[1:]:
        d.setdefault(r[ki], []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    out = io.StringIO()
    out.write(f"{'kernel':70s} {'n':>5s} {'mean_us':>10s} {'share':>7s}\n")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        out.write(f"{k[:70]:70s} {len(v):5d} {sum(v) / len(v) / 1e3:10.1f} {sum(v) / tot:7.3f}\n")
    out.write(f"total device time of listed launches: {tot / 1e3:.1f} us "
              "(ncu, serialised, cold caches: compare shares, not absolutes)\n")
    return out.getvalue()


def ncu_raw(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = []
    for row in rows[2:]:
        d = dict(zip(h, row))
        for k, u in zip(h, units):   # byte metrics normalised to bytes
            if u in scale and d.get(k):
                try:
                    d[k] = repr(float(d[k].replace(",", "")) * scale[u])
                except ValueError:
                    pass
        out.append(d)
    return out


def main(src, dst):
    os.makedirs(dst, exist_ok=True)
    for pat in ("*.json", "*.log", "nvidia-smi.txt"):
        for f in glob.glob(os.path.join(src, pat)):
            if os.path.basename(f).startswith("plain"):
                continue
            shutil.copy(f, dst)
    for lf in sorted(glob.glob(os.path.join(src, "launches*.csv"))):   # launches.csv, launches_<config>.csv
        tag = os.path.basename(lf)[len("launches"):-4]
        with open(os.path.join(dst, f"launches_summary{tag}.txt"), "w") as f:
            f.write(launches_table(lf))
    traffic = {}
    for rep in sorted(glob.glob(os.path.join(src, "*.ncu-rep"))):
        name = os.path.basename(rep)[:-8]
        launches = ncu_raw(rep)
        with open(os.path.join(dst, f"{name}_ncu.txt"), "w") as f:
            for i, d in enumerate(launches):
                f.write(f"# launch {i}: {d.get('Kernel Name', '')}\n")
                for k in KEYS:
                    if k in d:
                        f.write(f"{k} = {d[k]}\n")
                f.write("\n")
        if launches:
            rd = [float(d.get("dram__bytes_read.sum", "nan").replace(",", "")) for d in launches]
            wr = [float(d.get("dram__bytes_write.sum", "nan").replace(",", "")) for d in launches]
            traffic[name] = {"kernel": launches[0].get("Kernel Name", ""), "launches": len(launches),
                             "dram_read_bytes_per_launch": sum(rd) / len(rd),
                             "dram_write_bytes_per_launch": sum(wr) / len(wr),
                             "dram_bytes_per_launch": (sum(rd) + sum(wr)) / len(rd)}
    if traffic:
        with open(os.path.join(dst, "ncu_traffic.json"), "w") as f:
            json.dump(traffic, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
