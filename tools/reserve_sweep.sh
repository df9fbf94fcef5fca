# The bench round's time per reserved-SM count (side stream's share of the GPU
# during the horizon kernel): bash tools/reserve_sweep.sh 6 8 10 12 ...
for rep in 1 2; do
  for r in "$@"; do
    echo "reserve=$r $(python bench.py --no-e2e --no-cpu-baseline --no-configs --steps 40 --reserve-sms $r 2>/dev/null | tail -1 | python -c '
import json,sys
d=json.loads(sys.stdin.read())
print(round(1e3*d["ms_per_step"],1), round(1e3*d["roofline"]["launch_ms_mean"],1))')"
  done
done
