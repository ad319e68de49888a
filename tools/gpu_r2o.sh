set -x
O=gpurun_out/r2o; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -3 $O/gputests.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
timeout 900 python bench.py --workload c5 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; echo c5=$?
timeout 900 python bench.py --rpg 16 --steps 10 --no-cpu-baseline --no-pageable > $O/bench_c3_rpg16.json 2> $O/bench_c3_rpg16.err; echo c3r16=$?
for f in $O/bench_c*.json; do python -c "import json; d=json.load(open('$f')); r=d['roofline']; print('$f', d['value'], r['frac'], r.get('dram_frac'), d['breakdown'].get('scatter_gbs'), d['e2e']['value'])"; done
