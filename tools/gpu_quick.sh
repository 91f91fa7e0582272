set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_s2.txt; cat gpurun_out/pytest_s2.txt
timeout 600 python bench.py > gpurun_out/bench_s2.json 2> gpurun_out/bench_s2.err; cat gpurun_out/bench_s2.json
timeout 600 python tools/sweep.py --only ffn,attn,llama --steps 300 > gpurun_out/sw_s2.jsonl 2>&1
