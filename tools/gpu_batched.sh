set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "batched or metamorphic" 2>&1 | tail -15
timeout 600 python tools/sweep.py --only batched --steps 200 2>&1 | tee gpurun_out/sw_batched.jsonl
