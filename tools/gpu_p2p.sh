#!/bin/bash
# P2P tests (rows all-gather, column reduce-scatter + all-gather; world 1 and 2/4 processes on one GPU,
# back-to-back and graph-captured rounds) plus world-1 timing of the fused calls
mkdir -p gpurun_out
python paper_2206_09557_b200/_build.py > gpurun_out/p2p_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_tp.py tests/test_gpu_quantize.py -q -x ${PYT:-} > gpurun_out/p2p_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/p2p_tests.log
tail -15 gpurun_out/p2p_tests.log
for mode in rows cols; do
  timeout 300 python tools/p2p_check.py --rounds 1 --timing --no-oracle --mode $mode --rows 49152 --cols 12288 2>&1 | grep -v Warn | tail -3
  timeout 300 python tools/p2p_check.py --rounds 1 --timing --no-oracle --mode $mode --rows 12288 --cols 49152 2>&1 | grep -v Warn | tail -3
done
