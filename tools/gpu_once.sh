#!/bin/bash
# ncu --set full of the once-per-solve kernels at c2.  gpurun --timeout 900 -- 'bash tools/gpu_once.sh <tag>'
TAG=${1:-once}
OUT=gpurun_out/$TAG
mkdir -p $OUT
BC="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-fp32-arm --graph 0"
$BC > $OUT/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"combine_kernel|final_scale_kernel|frame_max_kernel|threshold_kernel" -s 4 -c 4 -o $OUT/once $BC > $OUT/ncu_once.log 2>&1
echo done > $OUT/DONE
