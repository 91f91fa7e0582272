#!/bin/bash
# P2P tests (rows all-gather and column all-reduce) on one GPU, plus world-1 timing
mkdir -p gpurun_out
python paper_2206_09557_b200/_build.py > gpurun_out/p2p_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_p2p.py -q -x > gpurun_out/p2p_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/p2p_tests.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29561 \
  tools/p2p_check.py --same-device --rounds 3 --mode cols --rows 49152 --cols 12288 > gpurun_out/p2p_cols_big.log 2>&1
echo "exit $?" >> gpurun_out/p2p_cols_big.log
tail -3 gpurun_out/p2p_tests.log; tail -8 gpurun_out/p2p_cols_big.log
timeout 300 python tools/p2p_check.py --rounds 1 --timing --mode cols --rows 12288 --cols 49152 > gpurun_out/p2p_cols_timing.log 2>&1
timeout 300 python tools/p2p_check.py --rounds 1 --timing --rows 49152 --cols 12288 > gpurun_out/p2p_rows_timing.log 2>&1
cat gpurun_out/p2p_cols_timing.log gpurun_out/p2p_rows_timing.log | grep -v Warn
