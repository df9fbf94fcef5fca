# A/B the headline round and the other BASELINE configs' rounds across library
# builds: bash tools/ab_configs.sh lib1.so lib2.so ...
# (each build is copied over the in-tree library for its run, then restored)
cp paper_2605_11381_b200/libkairos_b200.so /tmp/kr_base.so
for rep in 1 2; do
  for lib in "$@"; do
    cp "$lib" paper_2605_11381_b200/libkairos_b200.so
    touch paper_2605_11381_b200/libkairos_b200.so
    echo "$lib $(python bench.py --no-e2e --no-cpu-baseline --steps 30 2>/dev/null | tail -1 | python -c '
import json,sys
d=json.loads(sys.stdin.read())
print(round(1e3*d["ms_per_step"],1), [round(v["us_per_round"],1) for v in d["other_configs"].values()])')"
  done
done
cp /tmp/kr_base.so paper_2605_11381_b200/libkairos_b200.so
