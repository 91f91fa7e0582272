set -e
python -c "import __graft_entry__ as g; g.build()"
set +e
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gemv or probe or metamorphic or full_size or tiny or attention or reduction" 2>&1 | tail -1
for cfg in "0 0" "23 0" "0 3" "0 6" "0 0"; do set -- $cfg
echo "xmode=$1 pf_init=$2"; LUTGEMM_XMODE=$1 LUTGEMM_PF_INIT=$2 python tools/sweep.py --cases 49152:12288:3:128,12288:49152:3:128,12288:12288:3:128,36864:12288:3:128,8192:8192:4:128:1:2 --steps 400 | python -c "
import sys,json
print('   ', [ (json.loads(l)['case'][:14], json.loads(l)['us']) for l in sys.stdin])"
done
