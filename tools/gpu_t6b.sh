#!/bin/bash
TAG=${1:-t6c}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tcgen05.py -q -x > $OUT/pytest_t6.log 2>&1; tail -2 $OUT/pytest_t6.log
timeout 300 python bench.py --algo tcgen05 --no-cpu-baseline --no-e2e > $OUT/bench_t6.json 2> $OUT/bench_t6.err
python -c "
import json;d=json.loads(open('$OUT/bench_t6.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step']);r=d['roofline'];print({k:r[k] for k in ['achieved','frac','launch_ms','share_of_step']})"
BC="python bench.py --algo tcgen05 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BC > $OUT/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spass_tc6 -s 16 -c 1 -o $OUT/t6 $BC > $OUT/ncu.log 2>&1
ncu -i $OUT/t6.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); d=dict(zip(r[0],r[2]))
print({k:d.get(k) for k in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sector_hit_rate.pct']})"
SFSEG_NVCC_DEFS="-DT6_PROFILE" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python bench.py --algo tcgen05 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --graph 0 > $OUT/prof.log 2>&1
grep t6prof $OUT/prof.log | tail -4
python - <<PY
import numpy as np
v=[int(l.split()[2]) for l in open('$OUT/prof.log') if l.startswith('[t6cta]')]
v=np.array(v[-148:]) if len(v)>=148 else np.array(v)
print('per-CTA cycles: n', len(v), 'min', v.min(), 'mean', int(v.mean()), 'max', v.max())
PY
echo done > $OUT/DONE
