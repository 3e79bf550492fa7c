#!/bin/bash
# tcgen05 pass: ncu --set full of one launch, then a -DT6_PROFILE build's per-role wait profile.
TAG=${1:-t6p}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
BC="python bench.py --algo tcgen05 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BC > $OUT/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spass_tc6 -s 16 -c 1 -o $OUT/t6 $BC > $OUT/ncu.log 2>&1
SFSEG_NVCC_DEFS="-DT6_PROFILE" python -c "import __graft_entry__ as g; g.build()" > $OUT/build_prof.log 2>&1
timeout 300 python bench.py --algo tcgen05 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --graph 0 > $OUT/prof.log 2>&1
grep t6prof $OUT/prof.log | tail -8
echo done > $OUT/DONE
