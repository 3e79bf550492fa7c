#!/bin/bash
# Last check of the in-tree build: smoke, the slab / tcgen05 / parity test files, the default bench line.
TAG=${1:-sanity}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_tcgen05.py tests/test_gpu_parity.py -q -m gpu > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo done > $OUT/DONE
