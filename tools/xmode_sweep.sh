# usage: bash tools/xmode_sweep.sh "xmodes" "pfs"  -> graph us/GEMV, eager us/GEMV, frac
for XM in ${1:-0}; do for PF in ${2:-4}; do
LUTGEMM_XMODE=$XM LUTGEMM_PF_STEPS=$PF timeout 300 python bench.py --steps 1000 --warmup 50 --no-cpu --no-check > gpurun_out/b.json 2>gpurun_out/b.err
echo "xmode=$XM pf=$PF $(python -c "import json;d=json.load(open('gpurun_out/b.json'));r=d['roofline'];print('graph', r['kernel_us'], 'eager', r['eager_us_per_gemv'], 'frac', r['frac'])" 2>&1 | tail -1)"
done; done
