#!/bin/bash
TAG=${1:-r02g}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for v in 0 1 0 1; do
SFSEG_NVCC_DEFS="-DTPASS16_HINT=$v" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);r=d['roofline'];print('hint$v',d['ms_per_step'],r['launch_ms'],r['tpass']['launch_ms'])"
done
SFSEG_NVCC_DEFS="-DT6_PROFILE" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --graph 0 > $OUT/prof.log 2>&1
python - <<PY
import numpy as np
L=[l.split() for l in open('$OUT/prof.log') if l.startswith('[t6cta]')]
L=L[-148:] if len(L)>=148 else L
cyc=np.array([int(x[2]) for x in L]); g0=np.array([int(x[3]) for x in L]); g1=np.array([int(x[4]) for x in L])
print('n',len(L),'cycles min/mean/max',cyc.min(),int(cyc.mean()),cyc.max())
print('start spread us', (g0.max()-g0.min())/1e3, 'end spread us', (g1.max()-g1.min())/1e3, 'span us', (g1.max()-g0.min())/1e3)
print('clock GHz est (cycles / wall per CTA) min/mean', (cyc/(g1-g0)).min(), (cyc/(g1-g0)).mean())
PY
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo done > $OUT/DONE
