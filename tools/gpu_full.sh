#!/bin/bash
# Full measurement round: build, smoke, GPU tests, default bench (+cpu baseline), reference arm,
# sweeps (GEMV shapes, batched), stack, ncu launch list of the bench command, ncu --set full of
# one GEMV kernel (fc1) and one batched kernel (fc1 b=8).
set -u
TAG=${1:-r}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,temperature.gpu,power.draw --format=csv > gpurun_out/gpu_$TAG.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_$TAG.txt; cat gpurun_out/pytest_$TAG.txt
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; cat gpurun_out/bench_ref_$TAG.json
timeout 900 python tools/sweep.py --steps 300 > gpurun_out/sweep_$TAG.jsonl 2> gpurun_out/sweep_$TAG.err
timeout 600 python tools/stack.py > gpurun_out/stack_$TAG.json 2> gpurun_out/stack_$TAG.err; tail -1 gpurun_out/stack_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-check > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lut_gemv -s 10 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 20 --warmup 5 --no-cpu --no-check > gpurun_out/ncu_$TAG.log 2>&1; tail -1 gpurun_out/ncu_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lut_gemvv -s 1 -c 1 -o gpurun_out/prof_b8_$TAG python tools/run_once.py 49152 12288 3 128 8 > gpurun_out/ncu_b8_$TAG.log 2>&1; tail -1 gpurun_out/ncu_b8_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lut_gemvv -s 1 -c 1 -o gpurun_out/prof_b2_$TAG python tools/run_once.py 49152 12288 3 128 2 > gpurun_out/ncu_b2_$TAG.log 2>&1; tail -1 gpurun_out/ncu_b2_$TAG.log
timeout 600 python tools/trace_spread.py > gpurun_out/trace_$TAG.jsonl 2>&1; tail -4 gpurun_out/trace_$TAG.jsonl | cut -c1-300
