#!/bin/bash
# Mid-round check: build, GPU tests, smoke, the default c2 bench line, the mma (bf16) variant,
# and one ncu --set full capture of the default spatial pass.
#   gpurun --timeout 1800 -- 'bash tools/gpu_check.sh <tag>'
TAG=${1:-check}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --algo mma --no-cpu-baseline --no-e2e > $OUT/bench_c2_mma.json 2> $OUT/bench_c2_mma.err
BC="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BC > $OUT/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spass_tc -s 16 -c 1 -o $OUT/spass $BC > $OUT/ncu_spass.log 2>&1
echo done > $OUT/DONE
