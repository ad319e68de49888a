# A/B: pipecg staging its five own-row vectors (default) vs loading them per row (deeper ring)
O=gpurun_out/${1:-tails}; mkdir -p $O
LRB_LIB=build/lib_notails.so timeout 900 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_stream.py -q -x -k "pipecg" > $O/tests.log 2>&1; echo tests_notails=$? > $O/ab.txt; tail -1 $O/tests.log >> $O/ab.txt
for round in 1 2; do for w in c1 c2 c3; do
  for v in paper_2510_08536_b200/libldurepart_b200.so build/lib_notails.so; do
    LRB_LIB=$v timeout 300 python bench.py --workload $w --method pipecg --no-cpu-baseline --no-pageable > $O/ab.json 2> $O/ab.err
    echo "$round $w $(basename $v) $(python -c "import json; d=json.load(open('$O/ab.json')); print(d['value'], d['roofline']['kernel_ms'], d['roofline']['kernel_geometry']['stages'], d['roofline']['kernel_geometry']['stage_bytes'])" 2>&1 | tail -1)" >> $O/ab.txt
  done
done; done
cat $O/ab.txt
for round in 1 2; do LRB_LIB=paper_2510_08536_b200/libldurepart_b200.so timeout 300 python bench.py --workload c3 --no-cpu-baseline --no-pageable > $O/ab.json 2> $O/ab.err
echo "$round c3 pcg $(python -c "import json; d=json.load(open('$O/ab.json')); print(d['value'], d['roofline']['kernel_ms'])" 2>&1 | tail -1)" >> $O/ab.txt; done
cat $O/ab.txt
