python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for cfg in "0 0" "3 0" "6 0" "64 0" "0 4" "6 4" "64 4"; do set -- $cfg
echo "pf_init=$1 pf_steps=$2"; LUTGEMM_PF_INIT=$1 LUTGEMM_PF_STEPS=$2 python tools/sweep.py --cases 49152:12288:3:128,12288:12288:3:128,8192:8192:4:128:1:2,12288:12288:1:128 --steps 300 | python -c "
import sys,json
print('   ', [ (json.loads(l)['case'][:14], json.loads(l)['us']) for l in sys.stdin])"
done
