python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.mem,temperature.gpu,power.draw,serial --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gemv or probe or metamorphic or full_size or tiny or attention or llama or compact or reduction" 2>&1 | tail -2
for X in ${XMS:-42 0 40 41 44 45}; do
echo "xmode=$X"; LUTGEMM_XMODE=$X python tools/sweep.py --cases 49152:12288:3:128,12288:49152:3:128,12288:12288:3:128,8192:8192:4:128:1:2,12288:12288:1:128,36864:12288:3:128 --steps 400 | python -c "
import sys,json
print('   ', [ (json.loads(l)['case'][:14], json.loads(l)['us']) for l in sys.stdin])"
done
