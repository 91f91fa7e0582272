#!/bin/bash
# per-GPU compute of TP-N per-token latency (rank 0's shards, no exchange), N = 1, 2, 4, 8
mkdir -p gpurun_out
for N in 1 2 4 8; do
  timeout 600 python tools/stack.py --shard-tp $N --check > gpurun_out/stack_shard$N.json 2> gpurun_out/stack_shard$N.err
  tail -1 gpurun_out/stack_shard$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('shard_tp', d['shard_tp'], d['ms_per_token'], 'ms/token', d['GBps_per_gpu'], 'GB/s', d['per_linear_us_eager'], 'max parity', max(d['parity_rel_l2_sampled'].values()))"
done
