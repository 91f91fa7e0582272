set -e
python -c "import __graft_entry__ as g; g.build()"
set +e
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "batched or compact" 2>&1 | tail -1
for X in ${XMS:-0 24 25 0}; do
echo "xmode=$X"; LUTGEMM_XMODE=$X python tools/sweep.py --cases 49152:12288:3:128:2,12288:49152:3:128:2,12288:12288:3:128:2,8192:22016:4:128:2:2 --steps 300 | python -c "
import sys,json
print('   ', [ (json.loads(l)['case'][:16], json.loads(l)['us']) for l in sys.stdin])"
done
