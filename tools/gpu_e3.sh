#!/bin/bash
# P2P per-group protocol: tests + world-1 timing; stack layer-count / graph-size scan
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_tp.py tests/test_gpu_general_shapes.py tests/test_gpu_stack.py -q -x > gpurun_out/e3_tests.log 2>&1
echo "pytest exit $?" >> gpurun_out/e3_tests.log
tail -5 gpurun_out/e3_tests.log
for mode in rows cols; do
  timeout 300 python tools/p2p_check.py --rounds 1 --timing --no-oracle --mode $mode --rows 49152 --cols 12288 2>&1 | grep -v Warn | tail -2
  timeout 300 python tools/p2p_check.py --rounds 1 --timing --no-oracle --mode $mode --rows 12288 --cols 49152 2>&1 | grep -v Warn | tail -2
done
for L in 8 32 64 96; do
  timeout 300 python tools/stack.py --layers $L 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stack', d['layers'], d['graph_layers'], d['ms_per_token'], round(d['ms_per_token']/d['layers']*1e3,1))"
done
for GL in 8 24; do
  timeout 300 python tools/stack.py --layers 96 --graph-layers $GL 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stack', d['layers'], d['graph_layers'], d['ms_per_token'], round(d['ms_per_token']/d['layers']*1e3,1))"
done
