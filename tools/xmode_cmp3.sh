set -e
python -c "import __graft_entry__ as g; g.build()"
set +e
for cfg in "0 0" "44 0" "44 8" "44 16" "45 8" "43 8" "0 8"; do set -- $cfg
echo "xmode=$1 pf_init=$2"; LUTGEMM_XMODE=$1 LUTGEMM_PF_INIT=$2 python tools/sweep.py --cases 49152:12288:3:128,12288:49152:3:128,12288:12288:3:128,36864:12288:3:128 --steps 400 | python -c "
import sys,json
print('   ', [ (json.loads(l)['case'][:14], json.loads(l)['us']) for l in sys.stdin])"
done
