# A/B the fp32 confidence round (split/16 and urgency_first/1, 4 interleaved
# repeats each) across library builds: bash tools/ab_conf.sh lib1.so lib2.so ...
cp paper_2605_11381_b200/libkairos_b200.so /tmp/kr_base.so
for lib in "$@"; do
  cp "$lib" paper_2605_11381_b200/libkairos_b200.so
  touch paper_2605_11381_b200/libkairos_b200.so
  echo "== $lib"; CONF_DT=32 python tools/conf_layout_reps.py 2>/dev/null | grep -v "'split', 2)\|'urgency_first', 4)"
done
cp /tmp/kr_base.so paper_2605_11381_b200/libkairos_b200.so
