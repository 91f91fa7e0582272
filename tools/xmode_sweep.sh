for XM in 0 10 11 12 14; do for PF in 0 4; do
LUTGEMM_XMODE=$XM LUTGEMM_PF_STEPS=$PF timeout 300 python bench.py --steps 1000 --warmup 20 --no-cpu --no-check > gpurun_out/b.json 2>/dev/null
echo "xmode=$XM pf=$PF $(python -c "import json;d=json.load(open('gpurun_out/b.json'));print(d['roofline']['kernel_us'], d['roofline']['frac'])")"
done; done
