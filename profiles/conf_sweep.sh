# confidence-kernel planner sweep (debug knob KR_PLAN_MAX_THREADS), run under gpurun
for mt in 0 128 192 256 320 480; do
  echo "max_threads=$mt"
  KR_PLAN_MAX_THREADS=$mt KR_TRACE_PLAN=1 python profiles/prof_kernels.py conf 2>&1 | sort -u | head -3
  KR_PLAN_MAX_THREADS=$mt python profiles/kernel_sweep.py 2>&1 | grep -i conf
done
