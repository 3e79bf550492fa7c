#!/bin/bash
# r02 evidence pass A: variants of the tensor-core spatial pass, full GPU test suite, bench line,
# ncu launch list + one --set full capture of the spatial pass at c2.
TAG=${1:-r02a}
OUT=gpurun_out/$TAG
mkdir -p $OUT
bash tools/gpu_variants.sh $TAG/var "" "-DSPTC_MIN_CTAS=2" > $OUT/variants.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
BC="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BC > $OUT/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2.csv $BC > $OUT/ncu_launches_c2.log 2>&1
$BC > $OUT/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spass -s 16 -c 1 -o $OUT/spass $BC > $OUT/ncu_spass.log 2>&1
echo done > $OUT/DONE
