#!/bin/bash
# After the combine change: parity / fullsize / slab tests, default bench line, launch list.
TAG=${1:-r02m}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
BC="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-fp32-arm"
$BC > $OUT/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2.csv $BC > $OUT/ncu_launches_c2.log 2>&1
echo done > $OUT/DONE
