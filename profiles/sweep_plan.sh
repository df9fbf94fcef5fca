# sweep-kernel tile sweep (debug knobs KR_SWEEP_G / KR_SWEEP_TR), run under gpurun
for cfg in "4 88" "4 48" "4 40" "4 24" "8 44" "8 24" "8 12"; do
  set -- $cfg
  echo "G=$1 TR=$2"
  KR_SWEEP_G=$1 KR_SWEEP_TR=$2 KR_TRACE_PLAN=1 python profiles/prof_kernels.py sweep16 2>&1 | grep sweep | sort -u | head -2
  KR_SWEEP_G=$1 KR_SWEEP_TR=$2 python profiles/kernel_sweep.py 2>&1 | grep "sweep C=16 K"
done
