#!/bin/bash
# LL-protocol P2P epilogue: tests, world-1 timing, multi-process same-GPU rounds
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_tp.py tests/test_gpu_general_shapes.py tests/test_gpu_stack.py -q -x > gpurun_out/e5_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/e5_tests.log
tail -5 gpurun_out/e5_tests.log
for mode in rows cols; do
  timeout 300 python tools/p2p_check.py --rounds 1 --timing --no-oracle --mode $mode --rows 49152 --cols 12288 2>&1 | grep -v Warn | tail -2
  timeout 300 python tools/p2p_check.py --rounds 1 --timing --no-oracle --mode $mode --rows 12288 --cols 49152 2>&1 | grep -v Warn | tail -2
  timeout 300 python tools/p2p_check.py --rounds 1 --timing --no-oracle --mode $mode --rows 12288 --cols 12288 2>&1 | grep -v Warn | tail -2
done
for P in 2 4; do for mode in rows cols; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29611 tools/p2p_check.py --same-device --rounds 8 --mode $mode 2>&1 | grep -v Warn | tail -2
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29612 tools/p2p_check.py --same-device --rounds 4 --graph --mode $mode 2>&1 | grep -v Warn | tail -2
done; done
