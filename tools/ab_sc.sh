# A/B scatter variants: bench value, scatter ms and GB/s (algorithmic) per library
for round in 1 2; do for v in "$@"; do
  LRB_LIB=$v timeout 300 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/absc.json 2> gpurun_out/absc.err
  python -c "import json; d=json.load(open('gpurun_out/absc.json')); b=d['breakdown']; print('$round', '$(basename $v)', d['value'], b['scatter_ms'], b['scatter_gbs'], d['e2e']['value'])" 2>/dev/null || tail -n 1 gpurun_out/absc.err
done; done
