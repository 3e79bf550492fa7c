#!/bin/bash
# A/B timing: bench line + ncu launch list (no tests).  gpurun -- 'bash tools/gpu_ab.sh <tag> [config]'
TAG=${1:-ab}; CFG=${2:-c2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python bench.py --config $CFG --no-cpu-baseline --no-e2e > $OUT/bench.json 2> $OUT/bench.err
BC="python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BC > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $BC > $OUT/ncu_launches.log 2>&1
echo done > $OUT/DONE
