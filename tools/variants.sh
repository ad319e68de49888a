# Compare build variants of the solver kernel on the bench workload (GPU box).
for v in "$@"; do
  echo "== ${v}"; LRB_LIB=$v timeout 300 python bench.py --steps 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['breakdown']['scatter_gbs'], d['e2e']['value'])"
done
