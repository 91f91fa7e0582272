#!/bin/bash
# stack working-set vs run-length: 8 layers for as long as the 96-layer run, clocks sampled
mkdir -p gpurun_out
(nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv -lms 200 > gpurun_out/e7_smi.csv 2>&1 &)
for args in "--layers 8 --tokens 20" "--layers 8 --tokens 260" "--layers 96 --tokens 20" "--layers 96 --tokens 3" "--layers 8 --tokens 20"; do
  timeout 300 python tools/stack.py $args 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stack', '$args', d['ms_per_token'], round(d['ms_per_token']/d['layers']*1e3,1))"
done
