# A/B build variants on one box for one workload: bash tools/ab_w.sh c1 lib_a.so lib_b.so ...
w=$1; shift
for round in 1 2; do
for v in "$@"; do
  LRB_LIB=$v timeout 300 python bench.py --workload $w --steps 10 --no-cpu-baseline > gpurun_out/abw.json 2> gpurun_out/abw.err
  b=$(python -c "import json; d=json.load(open('gpurun_out/abw.json')); print(d['value'], d['roofline']['kernel_ms'])" 2>/dev/null || tail -n 1 gpurun_out/abw.err)
  echo "$round $w $(basename $v) $b"
done; done
