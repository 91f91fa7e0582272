set -u
mkdir -p gpurun_out
python paper_2206_09557_b200/_build.py 2>&1 | tail -1
for B in ${BS:-2 32}; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lut_gemm_batched -s 1 -c 1 -o gpurun_out/prof_b$B python tools/run_once.py 49152 12288 3 128 $B > gpurun_out/ncu_b$B.log 2>&1; tail -1 gpurun_out/ncu_b$B.log
done
