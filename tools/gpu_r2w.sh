set -x
O=gpurun_out/r2w; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -q > $O/gputests.log 2>&1; echo tests=$?; tail -3 $O/gputests.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?
python -c "import json; d=json.load(open('$O/bench.json')); r=d['roofline']; print(d['value'], r['frac'], r.get('dram_frac'), d['breakdown']['scatter_gbs'], d['e2e']['value'], d['e2e_pageable']['value'], d['e2e_device_producer']['value'], d['cpu_baseline']['value'], d['gpu_launches'])"
