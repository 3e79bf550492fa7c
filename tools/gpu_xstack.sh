#!/bin/bash
# A/B of the tcgen05 pass's stacked x-pass (T6_XSTACK): parity tests of the default build,
# precision at full c2, bench c2 (alternating builds), c3 / c2f / c4 / c5 once each, and the
# per-role wait profile (-DT6_PROFILE) of both.
#   gpurun --timeout 1800 -- 'bash tools/gpu_xstack.sh <tag>'
TAG=${1:-xstack}
OUT=gpurun_out/$TAG
mkdir -p $OUT
LIB=paper_2212_08058_b200/libsfseg.so
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
cp $LIB /tmp/lib_default.so
for v in 1 0; do
  python tools/build_t6_variant.py /tmp/lib_x$v.so -DT6_XSTACK=$v >> $OUT/build.log 2>&1
  python tools/build_t6_variant.py /tmp/libprof_x$v.so -DT6_XSTACK=$v -DT6_PROFILE >> $OUT/build.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_full.py tests/test_gpu_parity.py -q -x > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
timeout 300 python tools/precision_c2.py c2 > $OUT/precision_c2.json 2> $OUT/precision_c2.err; cat $OUT/precision_c2.json
line() {
  python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d['roofline'];print('$1',d['value'],d['ms_per_step'],r.get('launch_ms'),r.get('frac'),(r.get('tpass') or {}).get('launch_ms'))"
}
for rep in 1 2 3; do
  for v in 1 0; do
    cp /tmp/lib_x$v.so $LIB
    timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e 2>/dev/null | line "x$v c2"
  done
done
for v in 1 0; do
  cp /tmp/lib_x$v.so $LIB
  for c in c3 c2f c4 c5; do
    timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | line "x$v $c"
  done
done
for v in 1 0; do
  cp /tmp/libprof_x$v.so $LIB
  timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --graph 0 > $OUT/prof$v.log 2>&1
  grep t6prof $OUT/prof$v.log | tail -4
  python - <<PY
import numpy as np
L=[l.split() for l in open('$OUT/prof$v.log') if l.startswith('[t6cta]')]
L=L[-147:]
cyc=np.array([int(x[2]) for x in L]); g0=np.array([int(x[3]) for x in L]); g1=np.array([int(x[4]) for x in L])
print('x$v n',len(L),'cycles min/mean/max',cyc.min(),int(cyc.mean()),cyc.max(), 'start spread us', (g0.max()-g0.min())/1e3, 'end spread us', (g1.max()-g1.min())/1e3, 'span us', (g1.max()-g0.min())/1e3)
PY
done
cp /tmp/lib_default.so $LIB
echo done > $OUT/DONE
