set -u
mkdir -p gpurun_out
python paper_2206_09557_b200/_build.py || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lut_gemv2 -s 1 -c 1 -o gpurun_out/prof_g2 python tools/run_once.py 49152 12288 3 128 2 > gpurun_out/ncu_g2.log 2>&1; tail -1 gpurun_out/ncu_g2.log
python tools/trace_pair.py 49152,12288,3,128 2>&1 | tail -3
