#!/bin/bash
# Full measurement round: build, GPU tests, default bench (+cpu baseline), reference arm,
# trace, ncu launch list of the bench command, ncu --set full of one LUT kernel.
set -u
TAG=${1:-r}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_$TAG.txt; cat gpurun_out/pytest_$TAG.txt
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_$TAG.csv &
SMI=$!
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
kill $SMI
cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; cat gpurun_out/bench_ref_$TAG.json
timeout 120 python tools/trace_gemv.py fc1 > gpurun_out/trace_$TAG.txt 2>&1; head -12 gpurun_out/trace_$TAG.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-check --no-graph > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lut_gemv -s 10 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 20 --warmup 5 --no-cpu --no-check --no-graph > gpurun_out/ncu_$TAG.log 2>&1; tail -1 gpurun_out/ncu_$TAG.log
