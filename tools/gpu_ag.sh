#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_stack.py -q -x 2>&1 | tail -3
timeout 600 python tools/stack.py --tp-impl p2p --tp-scheme allgather --check 2>/dev/null | tail -1 > gpurun_out/stack_ag_p2p.json; cut -c1-400 gpurun_out/stack_ag_p2p.json
