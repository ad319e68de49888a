# A/B: pipecg with the deferred reduction read (default) vs reducing barrier.
O=gpurun_out/${1:-pipeab}; mkdir -p $O
for round in 1 2; do for w in c1 c2; do
  for v in paper_2510_08536_b200/libldurepart_b200.so build/lib_nodefer.so; do
    LRB_LIB=$v timeout 300 python bench.py --workload $w --method pipecg --no-cpu-baseline --no-pageable > $O/ab.json 2> $O/ab.err
    echo "$round $w $(basename $v) $(python -c "import json; d=json.load(open('$O/ab.json')); print(d['value'], d['roofline']['kernel_ms'])" 2>&1 | tail -1)"
  done
  LRB_LIB=paper_2510_08536_b200/libldurepart_b200.so timeout 300 python bench.py --workload $w --method pcg1 --no-cpu-baseline --no-pageable > $O/ab.json 2> $O/ab.err
  echo "$round $w pcg1 $(python -c "import json; d=json.load(open('$O/ab.json')); print(d['value'], d['roofline']['kernel_ms'])" 2>&1 | tail -1)"
done; done 2>&1 | tee $O/ab.txt
