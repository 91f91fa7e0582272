for per in 0.005 0.02 0.1 0.005 0.02 0.1; do
  LUTGEMM_CLOCK_PERIOD_S=$per timeout 300 python bench.py --no-cpu --no-check 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('period $per', d['us_per_gemv'], d['us_per_gemv_dist'], d['clocks']['samples'])"
done
for mode in rows cols; do
  timeout 300 python tools/p2p_check.py --rounds 1 --timing --no-oracle --mode $mode --rows 49152 --cols 12288 2>&1 | grep -v Warn | tail -2
  timeout 300 python tools/p2p_check.py --rounds 1 --timing --no-oracle --mode $mode --rows 12288 --cols 49152 2>&1 | grep -v Warn | tail -2
done
