# A/B build variants on one box: bench value + phase profile per library.
#   bash tools/ab.sh build/lib_a.so build/lib_b.so ...   (repeats the list twice)
for round in 1 2; do
for v in "$@"; do
  LRB_LIB=$v timeout 300 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
  b=$(python -c "import json; d=json.load(open('gpurun_out/ab.json')); print(d['value'], d['roofline']['kernel_ms'])" 2>/dev/null || tail -1 gpurun_out/ab.err)
  p=$(LRB_LIB=$v timeout 300 python tools/phase_profile.py --repeat 2 2>/dev/null | head -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(*(f\"{k}={d[k]['us']}\" for k in ('A','A_sync','B','B_sync','C','X') if k in d))" 2>/dev/null)
  echo "$round $(basename $v) bench=$b $p"
done; done
