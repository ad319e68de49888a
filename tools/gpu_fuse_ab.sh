# A/B: pipelined PCG with the true-residual check fused into the next phase (default) vs a separate check phase.
O=gpurun_out/${1:-fuse}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_stream.py tests/test_gpu_large.py -q -x -k "pipecg or c3_bench" > $O/tests.log 2>&1; echo "tests=$? $(tail -1 $O/tests.log)" > $O/ab.txt
for round in 1 2; do for w in c3 c2 c1; do
  for v in paper_2510_08536_b200/libldurepart_b200.so build/lib_nofuse.so; do
    LRB_LIB=$v timeout 300 python bench.py --workload $w --no-cpu-baseline --no-pageable > $O/ab.json 2> $O/ab.err
    echo "$round $w $(basename $v) $(python -c "import json; d=json.load(open('$O/ab.json')); print(d['value'], d['roofline']['kernel_ms'], sum(d['breakdown']['iterations']))" 2>&1 | tail -1)" >> $O/ab.txt
  done
done; done
cat $O/ab.txt
