#!/bin/bash
# helper for gpurun calls: build, GPU tests, bench, trace, ncu (args: tag "pf list")
set -u
TAG=${1:-x}
python -c "import __graft_entry__ as g; g.build()" || exit 1
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > gpurun_out/pytest_$TAG.txt; tail -3 gpurun_out/pytest_$TAG.txt
fi
for PF in ${2:-8}; do
  LUTGEMM_PF_STEPS=$PF timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu > gpurun_out/bench_${TAG}_pf$PF.json 2> gpurun_out/bench_${TAG}_pf$PF.err
  echo "pf=$PF $(python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_pf$PF.json'));print(d['us_per_gemv'], d['value'], d['roofline']['kernel_us'], d['roofline']['frac'], d['clocks'])")"
done
timeout 120 python tools/trace_gemv.py fc1 > gpurun_out/trace_$TAG.txt 2>&1; cat gpurun_out/trace_$TAG.txt | head -40
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lut_gemv -s 10 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 20 --warmup 5 --no-cpu --no-check > gpurun_out/ncu_$TAG.log 2>&1; tail -1 gpurun_out/ncu_$TAG.log
fi
