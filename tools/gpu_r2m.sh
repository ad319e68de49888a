set -x
O=gpurun_out/r2m; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -3 $O/gputests.log
timeout 900 python bench.py --workload c5 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; echo c5=$?
timeout 600 python bench.py --workload c1 > $O/bench_c1.json 2> $O/bench_c1.err; echo c1=$?
timeout 1800 python bench.py --workload c4 --steps 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo c4=$?
for f in $O/bench_c*.json; do python -c "import json; d=json.load(open('$f')); r=d['roofline']; print('$f', d['value'], r['frac'], r.get('dram_frac'), d['e2e']['value'], (d.get('e2e_device_producer') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'))"; done
