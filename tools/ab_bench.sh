# A/B the headline round across library builds: bash tools/ab_bench.sh lib1.so lib2.so ...
# (each build is copied over the in-tree library for its run, then restored)
cp paper_2605_11381_b200/libkairos_b200.so /tmp/kr_base.so
for rep in 1 2; do
  for lib in "$@"; do
    cp "$lib" paper_2605_11381_b200/libkairos_b200.so
    touch paper_2605_11381_b200/libkairos_b200.so
    echo "$lib $(python bench.py --no-e2e --no-cpu-baseline --no-configs 2>/dev/null | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["ms_per_step"])')"
  done
done
cp /tmp/kr_base.so paper_2605_11381_b200/libkairos_b200.so
