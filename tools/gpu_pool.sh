#!/bin/bash
# HISTORICAL: the LUTGEMM_POOL knob was removed after this experiment (profiles/r02_tail_pool_dropped.md)
# A/B of the GEMV tail pool (LUTGEMM_POOL = quads per group moved to the per-slice pool)
mkdir -p gpurun_out
CASES=49152:12288:3:128,12288:49152:3:128,12288:12288:3:128,12288:12288:1:128,8192:8192:4:128:1:1,22016:8192:4:128:1:1,8192:22016:4:128:1:1
for T in ${POOLS:-0 8 16 32 64 0}; do
  echo "== POOL=$T"
  LUTGEMM_POOL=$T timeout 600 python tools/sweep.py --cases $CASES --steps 400 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(f\"{d['case']:28s} chain {d['us']:8.3f} us ({100*d['frac_hbm']:5.1f}%)\")"
done
LUTGEMM_POOL=${PT:-16} timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_general_shapes.py tests/test_gpu_p2p.py -q -x 2>&1 | tail -3
LUTGEMM_POOL=${PT:-16} timeout 300 python tools/trace_spread.py 2>&1 | tail -4 | cut -c1-400
