#!/bin/bash
# quick A/B: build, a parity subset, c2 / c2f / c3 bench lines (tpass / spass launch times)
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_parity.py tests/test_gpu_full.py tests/test_gpu_slabs.py -q -x > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for c in c2 c2f c3 c5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  python -c "
import json;d=json.loads(open('$OUT/bench_$c.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$c',d['value'],d['ms_per_step'],r.get('launch_ms'),r.get('frac'),(r.get('tpass') or {}).get('launch_ms'))"
done
echo done > $OUT/DONE
