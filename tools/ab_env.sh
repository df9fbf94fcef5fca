# A/B the headline round and the other configs' rounds across environment
# settings of one build: bash tools/ab_env.sh "" "KR_ADMIT_SPLIT=1" ...
for rep in 1 2; do
  for envs in "$@"; do
    echo "[$envs] $(env $envs python bench.py --no-e2e --no-cpu-baseline --steps 30 2>/dev/null | tail -1 | python -c '
import json,sys
d=json.loads(sys.stdin.read())
print(round(1e3*d["ms_per_step"],1), [round(v["us_per_round"],1) for v in d["other_configs"].values()])')"
  done
done
