#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_stack.py -q -x 2>&1 | tail -3
for mode in rows cols; do
  timeout 300 python tools/p2p_check.py --rounds 1 --timing --no-oracle --mode $mode --rows 49152 --cols 12288 2>&1 | grep -v Warn | tail -2
  timeout 300 python tools/p2p_check.py --rounds 1 --timing --no-oracle --mode $mode --rows 12288 --cols 12288 2>&1 | grep -v Warn | tail -2
done
nvidia-smi --query-gpu=name,memory.used --format=csv
