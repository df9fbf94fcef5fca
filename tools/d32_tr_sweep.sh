for tr in 0 1 2 3 4 6 8; do
  echo "TR=$tr"; KR_PLAN_FORCE_TR=$tr KR_TRACE_PLAN=1 python tools/d32_scaling.py 2>&1 | grep -E "^8192|^65536|^262144|R=8192 " | sort -u
done
