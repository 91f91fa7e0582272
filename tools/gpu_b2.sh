set -e
python paper_2206_09557_b200/_build.py
set +e
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "batched or random or compact or metamorphic" 2>&1 | tail -4
for X in 0 1; do
echo "LUTGEMM_B2_BATCHED=$X"; LUTGEMM_B2_BATCHED=$X python tools/sweep.py --cases 49152:12288:3:128:2,12288:49152:3:128:2,12288:12288:3:128:2,8192:22016:4:128:2:2,22016:8192:4:128:2:2 --steps 300 | python -c "
import sys,json
print('   ', [ (json.loads(l)['case'][:18], json.loads(l)['us']) for l in sys.stdin])"
done
