#!/bin/bash
# NOTE: the GPU pool this repo is measured on has disabled compute-sanitizer (its wrapper exits 86);
# tests/test_gpu_sanitize.py skips there.  Round-1 results: profiles/r01_sanitizers.md.
# compute-sanitizer over every kernel path (tier T4); summaries to gpurun_out/sanitize_*.txt
set -u
mkdir -p gpurun_out
python paper_2206_09557_b200/_build.py || exit 1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_case.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|sanitize cases done' gpurun_out/sanitize_$tool.txt | tr '\n' ' ')"
done
