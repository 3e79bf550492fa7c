#!/bin/bash
# A/B of an environment knob: gpurun -- 'bash tools/gpu_env_ab.sh <tag> <VAR> <val1> <val2> [config] [test-k]'
TAG=$1; VAR=$2; A=$3; B=$4; CFG=${5:-c2}; TK=${6:-tensor_core}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for v in $A $B; do
  env $VAR=$v timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "$TK" > $OUT/tests_$v.log 2>&1
  tail -1 $OUT/tests_$v.log
  env $VAR=$v timeout 300 python bench.py --config $CFG --no-cpu-baseline --no-e2e > $OUT/bench_$v.json 2> $OUT/bench_$v.err
done
for v in $A $B $A $B; do
  env $VAR=$v timeout 300 python bench.py --config $CFG --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$VAR=$v', d['ms_per_step'], d['roofline'].get('launch_ms'))" >> $OUT/ab.txt
done
cat $OUT/ab.txt
echo done > $OUT/DONE
