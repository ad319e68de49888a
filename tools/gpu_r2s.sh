set -x
O=gpurun_out/r2s; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_api.py -x -q > $O/api.log 2>&1; echo api=$?; tail -3 $O/api.log
timeout 900 python bench.py --workload c5 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; echo c5=$?
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
for f in $O/bench_c*.json; do python -c "import json; d=json.load(open('$f')); r=d['roofline']; e=d['e2e']; print('$f', d['value'], r['frac'], e['value'], e.get('link_gbs'), e.get('update_wall_ms'), (d.get('e2e_pageable') or {}).get('value'), (d.get('e2e_device_producer') or {}).get('value'))"; done
