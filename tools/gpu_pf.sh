#!/bin/bash
# GEMV start-up experiments: shared-memory / L2 weight prefetch before the PDL wait, reducer count
mkdir -p gpurun_out
python paper_2206_09557_b200/_build.py > gpurun_out/pf_build.log 2>&1 || { tail gpurun_out/pf_build.log; exit 1; }
CASES=${CASES:-49152:12288:3:128,12288:49152:3:128,12288:12288:3:128,12288:12288:1:128,12288:12288:1:12288,12288:12288:2:128,8192:8192:4:128:1:1,8192:8192:4:128:1:2,22016:8192:4:128:1:1}
for cfg in "0 0" "1048576 0" "1048576 131072" "1048576 524288" "0 524288"; do
  set -- $cfg
  echo "== SMEM_PF=$1 L2_PF=$2"
  LUTGEMM_SMEM_PF=$1 LUTGEMM_L2_PF=$2 timeout 600 python tools/sweep.py --cases $CASES --steps 400 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(f\"{d['case']:28s} chain {d['us']:8.2f} us ({100*d['frac_hbm']:5.1f}%)  iso {d['iso_us']:8.2f} us ({100*d['frac_hbm_iso']:5.1f}%)\")
    else: print(l.rstrip())"
done
for r in 1 3 6; do
  echo "== reducers $r"
  LUTGEMM_GEMV_REDUCERS=$r timeout 600 python tools/sweep.py --cases 49152:12288:3:128,12288:49152:3:128,12288:12288:3:128 --steps 400 2>&1 | grep '^{' | cut -c1-200
done
