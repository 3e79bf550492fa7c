#!/bin/bash
# tcgen05 spatial pass (spass_tc6) bring-up: debug cases, its tests, a bench line, launch list.
#   gpurun --timeout 1500 -- 'bash tools/gpu_t6.sh <tag>'
TAG=${1:-t6}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python tools/t6_debug.py 1,1,64,128,24,1 1,2,130,300,24,1 1,3,200,300,24,3 2,5,33,130,8,2 1,20,480,260,24,2 > $OUT/debug.log 2>&1
cat $OUT/debug.log
timeout 600 python -m pytest tests/test_gpu_tcgen05.py -q -x > $OUT/pytest_t6.log 2>&1; tail -3 $OUT/pytest_t6.log
timeout 300 python bench.py --algo tcgen05 --no-cpu-baseline --no-e2e > $OUT/bench_t6.json 2> $OUT/bench_t6.err
tail -c 600 $OUT/bench_t6.json
BC="python bench.py --algo tcgen05 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BC > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $BC > $OUT/ncu_launches.log 2>&1
echo done > $OUT/DONE
