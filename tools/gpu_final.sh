#!/bin/bash
# Round-end evidence: tests, smoke, bench lines (c2 default, probe, c4, c3, c2f, reference arm),
# microbenchmarks, ncu launch lists (c2, probe) and full captures (spass, tpass at c2; f3d at probe).
TAG=${1:-final}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
[ -x tools/fp32_microbench ] && timeout 120 tools/fp32_microbench > $OUT/fp32_microbench.log 2>&1
[ -x tools/stencil_microbench ] && timeout 120 tools/stencil_microbench > $OUT/stencil_microbench.log 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for c in probe c4 c3 c2f c5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
for c in c2 probe; do
  BC="python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
  $BC > $OUT/plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$c.csv $BC > $OUT/ncu_launches_$c.log 2>&1
done
BC="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BC > $OUT/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spass -s 16 -c 1 -o $OUT/spass $BC > $OUT/ncu_spass.log 2>&1
[ -x tools/mma_microbench ] && timeout 120 tools/mma_microbench > $OUT/mma_microbench.log 2>&1
$BC > $OUT/plain_full2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tpass -s 16 -c 1 -o $OUT/tpass $BC > $OUT/ncu_tpass.log 2>&1
BP="python bench.py --config probe --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BP > $OUT/plain_full3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:f3d -s 16 -c 1 -o $OUT/f3d $BP > $OUT/ncu_f3d.log 2>&1
echo done > $OUT/DONE
