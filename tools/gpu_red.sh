#!/bin/bash
# reducers per row group (LUTGEMM_GEMV_REDUCERS) on small shapes: default (~8 KB of partials each) vs others
CASES=12288:12288:3:128,12288:12288:1:128,8192:8192:4:128:1:1,6144:12288:3:128,12288:6144:3:128,4608:12288:3:128,49152:12288:3:128
for R in 0 2 4 8 12 0; do
  echo "== R=$R"
  LUTGEMM_GEMV_REDUCERS=$R timeout 600 python tools/sweep.py --cases $CASES --steps 400 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(f\"{d['case']:28s} {d['us']:8.3f} us ({100*d['frac_hbm']:5.1f}%)\")"
done
