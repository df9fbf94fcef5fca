# round-layout sweep: divergence ring depth / tile (debug knobs) x reserved SMs
for cfg in "0 0 12" "3 24 -1" "3 24 2" "3 24 4" "3 24 6" "3 20 4" "3 22 4" "0 0 12" "3 24 4"; do
  set -- $cfg
  KR_PLAN_MAX_STAGES=$1 KR_PLAN_FORCE_TR=$2 KR_TRACE_PLAN=1 timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-configs --reserve-sms $3 --steps 200 2>/tmp/p.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('stages<=$1 TR=$2 reserve $3', round(d['ms_per_step'],4), 'div', round(d['roofline']['launch_ms_mean'],4), 'side', round(k.get('side_stream_ms_in_round',0),4))"
  grep "kr_horizon_divergence R=1048576" /tmp/p.txt | sort -u | head -1 | cut -c1-150
done
