#!/bin/bash
# tcgen05 spatial pass inside the time-slab path: slab tests, c5 through the NCCL slab path at one rank,
# host<->device copy bandwidth (the e2e bound).  gpurun --timeout 1500 -- 'bash tools/gpu_slab6.sh <tag>'
TAG=${1:-slab6}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_tcgen05.py -q -m gpu > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
timeout 600 python bench.py --config c5 --slab-at-1 --steps 5 --no-cpu-baseline > $OUT/bench_c5_slab1.json 2> $OUT/bench_c5_slab1.err
timeout 600 python bench.py --config c5 --slab-at-1 --slab-serial --steps 5 --no-cpu-baseline > $OUT/bench_c5_slab1_serial.json 2> $OUT/bench_c5_slab1_serial.err
timeout 120 python tools/pcie_probe.py 128 > $OUT/pcie_probe.json 2> $OUT/pcie_probe.err
echo done > $OUT/DONE
