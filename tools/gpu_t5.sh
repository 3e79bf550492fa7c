#!/bin/bash
# tcgen05 spatial pass: bench lines (c2, tcgen05 vs mma.sync), precision at full c2, ncu capture.
TAG=${1:-t5}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for a in tcgen05 mma; do
  timeout 300 python bench.py --algo $a --no-cpu-baseline --no-e2e > $OUT/bench_$a.json 2> $OUT/bench_$a.err
done
timeout 300 python tools/precision_c2.py c2 > $OUT/precision_c2.json 2> $OUT/precision_c2.err
BC="python bench.py --algo tcgen05 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BC > $OUT/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spass_tc5 -s 16 -c 1 -o $OUT/spass_tc5 $BC > $OUT/ncu.log 2>&1
echo done > $OUT/DONE
