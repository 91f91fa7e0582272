#!/bin/bash
# A/B of the GEMV across builds / settings on the same box (_ab_*/ trees, not tracked)
mkdir -p gpurun_out
CASES=${CASES:-49152:12288:3:128,12288:12288:3:128,12288:12288:1:128,22016:8192:4:128:1:1}
summ() { python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(f\"  {d['case']:28s} {d['us']:8.3f} us  iso {d.get('iso_us', 0):8.3f}\")
    elif 'rror' in l: print(l.rstrip())"; }
for i in 1 2; do
  for v in ${VARIANTS:-"X=0"}; do
    echo "== new $v $i"; env $v timeout 600 python tools/sweep.py --cases $CASES --steps 400 2>&1 | summ
  done
  for d in ${DIRS:-}; do
    echo "== $d $i"; (cd $d && timeout 600 python tools/sweep.py --cases $CASES --steps 400 2>&1 | summ)
  done
done
