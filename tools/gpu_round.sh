#!/bin/bash
# One gpurun call: GPU tests, microbenchmarks, bench line, ncu launch list + full capture of spass.
#   gpurun --timeout 2400 -- 'bash tools/gpu_round.sh <tag>'
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
[ -x tools/fp32_microbench ] && timeout 120 tools/fp32_microbench > $OUT/fp32_microbench.log 2>&1
[ -x tools/stencil_microbench ] && timeout 120 tools/stencil_microbench > $OUT/stencil_microbench.log 2>&1
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
for c in probe c4; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
BC="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BC > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $BC > $OUT/ncu_launches.log 2>&1
$BC > $OUT/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spass -s 16 -c 2 -o $OUT/spass $BC > $OUT/ncu_spass.log 2>&1
$BC > $OUT/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tpass -s 16 -c 2 -o $OUT/tpass $BC > $OUT/ncu_tpass.log 2>&1
echo done > $OUT/DONE
