set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "batched or metamorphic" 2>&1 | tail -3
for cfg in ${CFGS:-256:0 128:0}; do
Q=${cfg%%:*}; X=${cfg##*:}
echo "rbq=$Q xmode=$X"; LUTGEMM_XMODE=$X LUTGEMM_BRBQ=$Q timeout 600 python tools/sweep.py --only batched --steps 200 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print(d['case'], d['us'], d['frac_of_binding_roof'])"
done
