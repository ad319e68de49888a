set -x
O=gpurun_out/r2z; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_stream.py tests/test_gpu_halo.py tests/test_gpu_krylov.py tests/test_gpu_parity.py -x -q > $O/tests.log 2>&1; echo tests=$?; tail -2 $O/tests.log
timeout 600 python tools/split_overhead.py > $O/split200.jsonl 2>/dev/null; cat $O/split200.jsonl
timeout 1500 python bench.py --workload c4 --steps 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; python -c "import json; d=json.load(open('$O/bench_c4.json')); print(d['value'], d['roofline']['kernel_ms'], d['e2e']['value'])"
