"""Per-source-line instruction / stall attribution from an ncu report:
    python tools/ncu_lines.py <report.ncu-rep> [file-substring] [top]"""
import csv, subprocess, sys, collections

rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file, hdr = "", None
agg = collections.OrderedDict()
tot_i = tot_s = 0
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        isam = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    if r[0]:  # source line
        cur = (cur_file, int(r[0]), r[1].strip()[:70])
        continue
    try:
        n = int(r[ie] or 0)
        s = int(r[isam] or 0)
    except ValueError:
        continue
    a = agg.setdefault(cur, [0, 0])
    a[0] += n
    a[1] += s
    tot_i += n
    tot_s += s
print(f"total inst {tot_i}  samples {tot_s}")
for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    if sub and sub not in k[0]:
        continue
    print(f"{100*n/tot_i:5.1f}% inst {100*s/max(tot_s,1):5.1f}% stall  {k[0]}:{k[1]}  {k[2]}")
