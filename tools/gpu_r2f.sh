# update epochs (no owner-group barrier in direct mode): all GPU tests, C4 + C3 benches.
set -x
O=gpurun_out/r2f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_api.py -x -q > $O/api.log 2>&1; echo api=$?; tail -3 $O/api.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -3 $O/gputests.log
timeout 1200 python bench.py --workload c4 --steps 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo c4=$?
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
for f in $O/bench_c*.json; do python -c "import json; d=json.load(open('$f')); r=d['roofline']; print('$f', d['value'], r['frac'], r.get('dram_frac'), d['e2e']['value'], d.get('e2e_pageable',{}).get('value'), d.get('e2e_device_producer',{}).get('value'))"; done
