for cfg in "0 0" "0 1" "0 2" "256 4" "384 2" "192 1"; do
  set -- $cfg
  echo "max_threads=$1 min_rounds=$2"
  KR_PLAN_MAX_THREADS=$1 KR_PLAN_MIN_ROUNDS=$2 KR_TRACE_PLAN=1 python profiles/prof_kernels.py sweep16 2>&1 | grep sweep | sort -u | head -2
  KR_PLAN_MAX_THREADS=$1 KR_PLAN_MIN_ROUNDS=$2 python profiles/kernel_sweep.py 2>&1 | grep "sweep C=16 K"
done
