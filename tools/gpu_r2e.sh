# f3 device producer, chunked pageable staging, one-pass multi-part barrier:
# tests, C2 phase profile + bench, C3 bench (all legs), C5 bench.
set -x
O=gpurun_out/r2e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_api.py tests/test_gpu_halo.py tests/test_gpu_stream.py -x -q > $O/tests_quick.log 2>&1; echo quick=$?; tail -3 $O/tests_quick.log
timeout 600 python tools/phase_profile.py --n 100 --ranks 64 --alpha 8 > $O/phase_c2.json 2> $O/phase_c2.err; echo phase=$?; cat $O/phase_c2.json
timeout 900 python bench.py --workload c2 --no-cpu-baseline --no-pageable > $O/bench_c2.json 2> $O/bench_c2.err; echo c2=$?
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
timeout 900 python bench.py --workload c5 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; echo c5=$?
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -3 $O/gputests.log
for f in $O/bench_c*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['value'], d['roofline']['frac'], d['e2e']['value'], d.get('e2e_pageable',{}).get('value'), d.get('e2e_device_producer',{}).get('value'))"; done
