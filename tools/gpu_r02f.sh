#!/bin/bash
# c2f / c3 with the tcgen05 plain + tape passes, full-operator tests, and the TP_FWD16 store-hint A/B.
TAG=${1:-r02f}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_full.py tests/test_gpu_tcgen05.py tests/test_gpu_binarize.py -q -x > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for c in c2f c3 c2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  python -c "
import json;d=json.loads(open('$OUT/bench_$c.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$c',d['value'],d['ms_per_step'],r.get('launch_ms'),r.get('frac'),(r.get('tpass') or {}).get('launch_ms'))"
done
SFSEG_NVCC_DEFS="-DTPASS16_HINT=0" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d['roofline'];print('hint0',d['ms_per_step'],r['launch_ms'],r['tpass']['launch_ms'])"
done
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d['roofline'];print('hint1',d['ms_per_step'],r['launch_ms'],r['tpass']['launch_ms'])"
done
BC="python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BC > $OUT/plain_c3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3.csv $BC > $OUT/ncu_launches_c3.log 2>&1
BC="python bench.py --config c2f --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BC > $OUT/plain_c2f.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2f.csv $BC > $OUT/ncu_launches_c2f.log 2>&1
echo done > $OUT/DONE
