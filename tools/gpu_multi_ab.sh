# A/B: flat multi-part barrier (lane_multi) vs HEAD (last-CTA reduction).
O=gpurun_out/${1:-multi}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$? > $O/ab.txt; tail -1 $O/gputests.log >> $O/ab.txt
for round in 1 2; do for v in paper_2510_08536_b200/libldurepart_b200.so build/lib_head.so; do
  for n in 100 200; do
    LRB_LIB=$v timeout 300 python tools/split_overhead.py --n $n --ranks 8 --repeat 2 2>/dev/null | head -1 > $O/so.json
    echo "$round $(basename $v) split n=$n $(cut -c1-160 $O/so.json)" >> $O/ab.txt
  done
  LRB_LIB=$v timeout 300 python bench.py --workload c3 --no-cpu-baseline --no-pageable > $O/ab.json 2> $O/ab.err
  echo "$round $(basename $v) c3 pcg $(python -c "import json; d=json.load(open('$O/ab.json')); print(d['value'], d['roofline']['kernel_ms'])" 2>&1 | tail -1)" >> $O/ab.txt
  LRB_LIB=$v timeout 300 python bench.py --workload c1 --method pcg --no-cpu-baseline --no-pageable > $O/ab.json 2> $O/ab.err
  echo "$round $(basename $v) c1 pcg $(python -c "import json; d=json.load(open('$O/ab.json')); print(d['value'], d['roofline']['kernel_ms'])" 2>&1 | tail -1)" >> $O/ab.txt
done; done
cat $O/ab.txt
