#!/bin/bash
# build, the whole GPU suite, smoke, and c2 / c3 / c2f / c5 bench lines
TAG=${1:-s}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
for c in c3 c2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  python -c "
import json;d=json.loads(open('$OUT/bench_$c.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$c',d['value'],d['ms_per_step'],r.get('launch_ms'),r.get('frac'),(r.get('tpass') or {}).get('launch_ms'))"
done
BC="python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BC > $OUT/plain_c3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3.csv $BC > $OUT/ncu_launches_c3.log 2>&1
echo done > $OUT/DONE
