for v in "" build/lib_mb3_ch8.so build/lib_mb4_ch8.so build/lib_mb3_ch4.so build/lib_mb4_ch4.so build/lib_mb2_ch4.so; do
  echo "== $v"; LRB_LIB=$v timeout 300 python bench.py --steps 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['breakdown']['scatter_gbs'], d['e2e'])"
done
