python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
python tools/sweep.py --only ffn,attn,llama --steps 300 > gpurun_out/sw0.jsonl 2>&1
LUTGEMM_XMODE=1 python tools/sweep.py --only ffn --steps 300 > gpurun_out/sw1.jsonl 2>&1
LUTGEMM_PF_STEPS=2 python tools/sweep.py --only ffn,attn,llama --steps 300 > gpurun_out/sw2.jsonl 2>&1
