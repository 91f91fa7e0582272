# batched parity tests + batched sweep (rbq = row quads per work item: LUTGEMM_BRBQ forces 256 or 128)
set -u
mkdir -p gpurun_out
python paper_2206_09557_b200/_build.py || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "batched or metamorphic" 2>&1 | tail -3
for Q in ${RBQS:-0}; do
echo "rbq=$Q"; LUTGEMM_BRBQ=$Q timeout 600 python tools/sweep.py --only batched --steps 200 2>&1 | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); print(d['case'], d['us'], d['frac_of_binding_roof'])"
done
