#!/bin/bash
# Quick GPU round: smoke, all GPU tests (no -x, full failure list), default bench line
set -u
TAG=${1:-q}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; tail -2 gpurun_out/smoke_$TAG.txt
timeout 1500 python -m pytest tests -m gpu -q ${PYT:-} > gpurun_out/pytest_$TAG.txt 2>&1; tail -30 gpurun_out/pytest_$TAG.txt
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
