#!/bin/bash
# HISTORICAL: the LUTGEMM_TOUCH knob was removed after this experiment (DESIGN "Measured and dropped")
# A/B of LUTGEMM_TOUCH (translation warm-up before the PDL wait): chain over k distinct copies, 96-layer stack
set -u
mkdir -p gpurun_out
for T in 0 1 2 3; do
  echo "== TOUCH=$T"
  LUTGEMM_TOUCH=$T timeout 300 python tools/tlb_probe.py --copies 2,32 2>&1 | tail -4
  LUTGEMM_TOUCH=$T timeout 300 python tools/stack.py --layers 96 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stack96', d['ms_per_token'], d['per_linear_us_eager'])"
done
