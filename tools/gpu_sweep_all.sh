python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python tools/sweep.py --only ffn,attn,llama --steps 400 > gpurun_out/sw_lr.jsonl 2>&1; python -c "
import json
for l in open('gpurun_out/sw_lr.jsonl'):
  d=json.loads(l); print(d['case'], d['us'], d['frac_hbm'])"
timeout 300 python tools/stack.py 2>&1 | tail -3
