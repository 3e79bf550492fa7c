#!/bin/bash
# A/B of the tcgen05 pass's read-out and prefetch knobs (T6_LDALL, T6_L2PF): parity tests of the
# default build, bench c2 for each variant (two alternating rounds), c3 / c2f for the default vs
# the round-2 baseline, and the per-role wait profile (-DT6_PROFILE) of both.
#   gpurun --timeout 1800 -- 'bash tools/gpu_ldall.sh <tag>'
TAG=${1:-ldall}
OUT=gpurun_out/$TAG
mkdir -p $OUT
LIB=paper_2212_08058_b200/libsfseg.so
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
cp $LIB /tmp/lib_default.so
VARS="1,3 0,0 1,0 0,3 1,6"
for v in $VARS; do
  a=${v%,*}; p=${v#*,}
  python tools/build_t6_variant.py /tmp/lib_$a$p.so -DT6_LDALL=$a -DT6_L2PF=$p >> $OUT/build.log 2>&1
  python tools/build_t6_variant.py /tmp/libprof_$a$p.so -DT6_LDALL=$a -DT6_L2PF=$p -DT6_PROFILE >> $OUT/build.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_full.py -q -x > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
line() {
  python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d['roofline'];print('$1',d['value'],d['ms_per_step'],r.get('launch_ms'),r.get('frac'),(r.get('tpass') or {}).get('launch_ms'))"
}
for rep in 1 2; do
  for v in $VARS; do
    a=${v%,*}; p=${v#*,}
    cp /tmp/lib_$a$p.so $LIB
    timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e 2>/dev/null | line "v$a$p c2"
  done
done
for v in 1,3 0,0; do
  a=${v%,*}; p=${v#*,}
  cp /tmp/lib_$a$p.so $LIB
  for c in c3 c2f c4; do
    timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | line "v$a$p $c"
  done
done
for v in 1,3 0,0; do
  a=${v%,*}; p=${v#*,}
  cp /tmp/libprof_$a$p.so $LIB
  timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --graph 0 > $OUT/prof$a$p.log 2>&1
  grep t6prof $OUT/prof$a$p.log | tail -4
  python - <<PY
import numpy as np
L=[l.split() for l in open('$OUT/prof$a$p.log') if l.startswith('[t6cta]')]
L=L[-147:]
cyc=np.array([int(x[2]) for x in L]); g0=np.array([int(x[3]) for x in L]); g1=np.array([int(x[4]) for x in L])
print('v$a$p n',len(L),'cycles min/mean/max',cyc.min(),int(cyc.mean()),cyc.max(), 'start spread us', (g0.max()-g0.min())/1e3, 'end spread us', (g1.max()-g1.min())/1e3, 'span us', (g1.max()-g0.min())/1e3)
PY
done
cp /tmp/lib_default.so $LIB
echo done > $OUT/DONE
