#!/bin/bash
# A/B of compile-time variants of the kernels on the c2 bench (rebuilds per variant, then
# restores the product build).  gpurun -- 'bash tools/gpu_variants.sh <tag> "<defs1>" "<defs2>" ...'
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
i=0
for DEFS in "$@"; do
  export SFSEG_NVCC_DEFS="$DEFS"
  python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$i.log 2>&1
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 $BENCH_ARGS > $OUT/bench_$i.json 2> $OUT/bench_$i.err
  python - "$DEFS" $OUT/bench_$i.json <<'PY' >> $OUT/summary.txt
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
r = d["roofline"]
print(f"{sys.argv[1] or 'default':40s} ms/step {d['ms_per_step']:.3f}  spass {r['launch_ms']*1e3:.1f} us  "
      f"tpass {r.get('tpass', {}).get('launch_ms', 0)*1e3:.1f} us  value {d['value']:.3e}")
PY
  if [ -n "$NCU" ]; then   # DRAM bytes of one spatial-pass launch (after the plain run exited 0)
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:spass_tc -s 16 -c 1 python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 1 \
      > $OUT/ncu_$i.log 2>&1
    grep -E "dram__bytes|gpu__time" $OUT/ncu_$i.log | sed "s/^/  [$i] /" >> $OUT/summary.txt
  fi
  i=$((i+1))
done
unset SFSEG_NVCC_DEFS
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_restore.log 2>&1
cat $OUT/summary.txt
