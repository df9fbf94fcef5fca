# confidence-kernel planner sweep (debug knobs KR_PLAN_MAX_THREADS / KR_PLAN_MIN_ROUNDS), run under gpurun
for cfg in "0 1" "0 2" "0 3" "0 4" "256 2" "192 4"; do
  set -- $cfg
  echo "max_threads=$1 min_rounds=$2"
  KR_PLAN_MAX_THREADS=$1 KR_PLAN_MIN_ROUNDS=$2 KR_TRACE_PLAN=1 python profiles/prof_kernels.py conf 2>&1 | sort -u | head -3
  KR_PLAN_MAX_THREADS=$1 KR_PLAN_MIN_ROUNDS=$2 python profiles/kernel_sweep.py 2>&1 | grep -i "conf.*float32"
done
