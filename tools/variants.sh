# Compare build variants of the solver kernel on the bench workload (GPU box).
#   bash tools/variants.sh lib1.so lib2.so ...   (LRB_LIB selects the library)
for v in "$@"; do
  echo "== ${v}"
  LRB_LIB=$v timeout 300 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/variant.json 2> gpurun_out/variant.err
  python -c "import json; d=json.load(open('gpurun_out/variant.json')); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['breakdown']['scatter_gbs'], d['e2e']['value'])" || tail -5 gpurun_out/variant.err
done
