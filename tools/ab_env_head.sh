# A/B the headline round across environment settings (no other configs):
# bash tools/ab_env_head.sh "" "KR_PLAN_FORCE_TR=32" ...
for rep in 1 2; do
  for envs in "$@"; do
    echo "[$envs] $(env $envs python bench.py --no-e2e --no-cpu-baseline --no-configs --steps 40 2>/dev/null | tail -1 | python -c '
import json,sys
d=json.loads(sys.stdin.read())
print(round(1e3*d["ms_per_step"],1), round(1e3*d["roofline"]["launch_ms_mean"],1))')"
  done
done
