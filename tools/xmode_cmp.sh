set -e
python -c "import __graft_entry__ as g; g.build()"
set +e
LUTGEMM_XMODE=${TESTX:-20} timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gemv or probe or metamorphic or full_size or tiny or attention" 2>&1 | tail -1
for X in ${XMS:-0 20 21 0 20}; do
echo "xmode=$X"; LUTGEMM_XMODE=$X python tools/sweep.py --cases ${CASES:-49152:12288:3:128,12288:49152:3:128,12288:12288:3:128,36864:12288:3:128} --steps 400 | python -c "
import sys,json
print('   ', [ (json.loads(l)['case'][:14], json.loads(l)['us']) for l in sys.stdin])"
done
