set -x
O=gpurun_out/r2p; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -3 $O/gputests.log
timeout 900 python bench.py --workload c5 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; echo c5=$?
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 900 python bench.py --workload c5 --no-cpu-baseline --no-pageable > $O/bench_c5_conn32.json 2> $O/bench_c5_conn32.err; echo c5b=$?
for f in $O/bench_c*.json; do python -c "import json; d=json.load(open('$f')); r=d['roofline']; print('$f', d['value'], r['frac'], d['e2e']['value'], d['e2e']['link_gbs'], (d.get('e2e_pageable') or {}).get('value'), (d.get('e2e_device_producer') or {}).get('value'))"; done
