#!/bin/bash
# A/B of the GEMV against an older build on the same box (_ab_old/, not tracked), then traces
mkdir -p gpurun_out
CASES=${CASES:-49152:12288:3:128,12288:12288:3:128,22016:8192:4:128:1:1}
for i in 1 2; do
  echo "== new $i"; timeout 600 python tools/sweep.py --cases $CASES --steps 400 2>&1 | grep '^{' | cut -c1-150
  echo "== old $i"; (cd _ab_old && LUTGEMM_SMEM_PF=0 timeout 600 python tools/sweep.py --cases $CASES --steps 400 2>&1 | grep '^{' | cut -c1-150)
done
timeout 600 python tools/trace_spread.py 2>&1 | tail -4
