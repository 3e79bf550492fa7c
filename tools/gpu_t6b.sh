#!/bin/bash
TAG=${1:-t6c}
OUT=gpurun_out/$TAG
mkdir -p $OUT

python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tcgen05.py -q -x > $OUT/pytest_t6.log 2>&1; tail -2 $OUT/pytest_t6.log
timeout 300 python bench.py --algo tcgen05 --no-cpu-baseline --no-e2e > $OUT/bench_t6.json 2> $OUT/bench_t6.err
python -c "
import json;d=json.loads(open('$OUT/bench_t6.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step']);r=d['roofline'];print({k:r[k] for k in ['achieved','frac','launch_ms','share_of_step']})"
BC="python bench.py --algo tcgen05 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$BC > $OUT/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spass_tc6 -s 16 -c 1 -o $OUT/t6 $BC > $OUT/ncu.log 2>&1
SFSEG_NVCC_DEFS="-DT6_PROFILE" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python bench.py --algo tcgen05 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --graph 0 2>&1 | grep t6prof | tail -4
echo done > $OUT/DONE
