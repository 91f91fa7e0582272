#!/bin/bash
mkdir -p gpurun_out
for GS in 0 1 2; do
  for mode in rows cols; do
    echo "== GPU_SCOPE=$GS $mode"
    LUTGEMM_P2P_GPU_SCOPE=$GS timeout 300 python tools/p2p_check.py --rounds 1 --timing --no-oracle --mode $mode --rows 49152 --cols 12288 2>&1 | grep -v Warn | tail -2
    LUTGEMM_P2P_GPU_SCOPE=$GS timeout 300 python tools/p2p_check.py --rounds 1 --timing --no-oracle --mode $mode --rows 12288 --cols 49152 2>&1 | grep -v Warn | tail -2
  done
done
for L in 8 96; do
  timeout 300 python tools/stack.py --layers $L --arena 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stack arena', d['layers'], d['ms_per_token'], round(d['ms_per_token']/d['layers']*1e3,1))"
done
