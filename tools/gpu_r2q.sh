set -x
O=gpurun_out/r2q; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -3 $O/gputests.log
timeout 900 python bench.py --workload c5 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; echo c5=$?
python -c "import json; d=json.load(open('$O/bench_c5.json')); r=d['roofline']; print(d['value'], r['frac'], d['e2e']['value'], d['e2e']['link_gbs'], (d.get('e2e_pageable') or {}).get('value'), (d.get('e2e_device_producer') or {}).get('value'))"
