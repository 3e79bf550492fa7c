#!/bin/bash
# ncu --set full of one kernel in the c2 bench (or another config).
#   gpurun --timeout 1200 -- 'bash tools/gpu_ncu.sh <tag> <kernel-regex> [config] [skip]'
TAG=${1:-ncu}; K=${2:-spass}; CFG=${3:-c2}; SKIP=${4:-16}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
BC="python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BC > $OUT/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 -o $OUT/$K $BC > $OUT/ncu_$K.log 2>&1
echo done > $OUT/DONE
