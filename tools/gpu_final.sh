#!/bin/bash
# Round-end evidence: tests, smoke, bench lines (c2 default, the other configs, the spatial-pass
# variants, the reference arm), ncu launch lists (c2, probe) and full captures (spass_tc at c2,
# tpass at c2, the tcgen05 pass at c2).  gpurun --timeout 3600 -- 'bash tools/gpu_final.sh <tag>'
TAG=${1:-final}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for c in probe c4 c3 c2f c5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 python bench.py --config c5 --slab-at-1 --steps 5 --no-cpu-baseline > $OUT/bench_c5_slab1.json 2> $OUT/bench_c5_slab1.err
for a in fp32 mma f16; do
  timeout 900 python bench.py --algo $a --no-cpu-baseline --no-e2e > $OUT/bench_c2_$a.json 2> $OUT/bench_c2_$a.err
done
timeout 300 python tools/precision_c2.py c2 > $OUT/precision_c2.json 2> $OUT/precision_c2.err
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc05_rate2 tools/tc05_rate2.cu && timeout 120 tools/tc05_rate2 > $OUT/tc05_rate2.log 2>&1
for c in c2 probe c3; do
  BC="python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
  $BC > $OUT/plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$c.csv $BC > $OUT/ncu_launches_$c.log 2>&1
done
BC="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BC > $OUT/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spass_tc6 -s 16 -c 1 -o $OUT/spass $BC > $OUT/ncu_spass.log 2>&1
$BC > $OUT/plain_full2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tpass -s 16 -c 1 -o $OUT/tpass $BC > $OUT/ncu_tpass.log 2>&1
BT="python bench.py --algo f16 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BT > $OUT/plain_full3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spass_tc_kernel -s 16 -c 1 -o $OUT/spass_mma_f16 $BT > $OUT/ncu_mma_f16.log 2>&1
echo done > $OUT/DONE
