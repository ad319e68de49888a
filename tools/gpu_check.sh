# Quick evidence pass on one B200: smoke, all GPU tests, C3 and C1 bench lines.
set -x
O=gpurun_out/${1:-check}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -3 $O/gputests.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
timeout 600 python bench.py --workload c1 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err; echo c1=$?
for f in $O/bench_c*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['value'], d['roofline']['frac'], d['e2e']['value'], (d.get('cpu_baseline') or {}).get('value'))"; done
