#!/bin/bash
# Slab tests with the larger tcgen05 frame-range case, the default bench line with the FP32-FMA arm,
# full GPU suite.  gpurun --timeout 1800 -- 'bash tools/gpu_r02l.sh <tag>'
TAG=${1:-r02l}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_slabs.py -q -m gpu > $OUT/pytest_slabs.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_slabs.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
echo done > $OUT/DONE
