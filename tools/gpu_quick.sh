#!/bin/bash
# Quick GPU check: parity tests + c2/probe bench lines (+ optional ncu launch list).
#   gpurun --timeout 1200 -- 'bash tools/gpu_quick.sh <tag> [launches]'
TAG=${1:-quick}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --config probe --no-cpu-baseline --no-e2e > $OUT/bench_probe.json 2> $OUT/bench_probe.err
if [ "$2" == "launches" ]; then
  BC="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
  $BC > $OUT/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $BC > $OUT/ncu_launches.log 2>&1
fi
echo done > $OUT/DONE
