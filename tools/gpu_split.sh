#!/bin/bash
# b > 4 as chunks of <= 4 rows (default) vs the vector-slot kernel (LUTGEMM_BATCH_SPLIT=0)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_general_shapes.py tests/test_gpu_tp.py tests/test_gpu_perf.py tests/test_gpu_pack.py -q -x 2>&1 | tail -3
C=49152:12288:3:128
CASES=$C:1,$C:2,$C:3,$C:4,$C:5,$C:6,$C:7,$C:8,$C:12,$C:16,$C:32,12288:49152:3:128:8,12288:12288:3:128:8,8192:22016:4:128:8:1,22016:8192:4:128:8:2
for SPLIT in 1 0; do
  echo "== LUTGEMM_BATCH_SPLIT=$SPLIT"
  LUTGEMM_BATCH_SPLIT=$SPLIT timeout 900 python tools/sweep.py --cases $CASES --steps 200 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(f\"{d['case']:30s} {d['us']:9.3f} us  LDS roof {d['lds_roof_us']:8.2f} ({100*d['frac_of_binding_roof']:5.1f}% of binding roof)\")"
done
