#!/bin/bash
# TP paths after the LL exchange: the strong-scaling bench arm with 2 ranks on one GPU (validation only:
# the ranks share the GPU), the 96-layer stack through the fused exchange at world 1, oracle-checked stacks
mkdir -p gpurun_out
for mode in rows cols; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 \
    bench.py --gpus 2 --steps 50 --warmup 5 --tp-impl p2p --tp-mode $mode --same-device --no-cpu > gpurun_out/tp2_$mode.json 2> gpurun_out/tp2_$mode.err
  echo "bench 2 ranks same-device p2p $mode rc=$?"; tail -1 gpurun_out/tp2_$mode.json | cut -c1-600
done
timeout 600 python tools/stack.py --check > gpurun_out/stack_check.json 2> gpurun_out/stack_check.err; tail -1 gpurun_out/stack_check.json
timeout 600 python tools/stack.py --tp-impl p2p --check > gpurun_out/stack_p2p.json 2> gpurun_out/stack_p2p.err; tail -1 gpurun_out/stack_p2p.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 \
  tools/stack.py --tp-impl p2p --same-device --layers 2 --tokens 3 --check > gpurun_out/stack_p2p_2r.json 2> gpurun_out/stack_p2p_2r.err; tail -1 gpurun_out/stack_p2p_2r.json
