# Final evidence pass (pipelined PCG as the C1/C2/C3 bench solver): smoke, all
# GPU tests, every BASELINE config's bench line, the reference arm at C3, and
# the launch list of the headline bench command.
O=gpurun_out/${1:-r2f2}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/nvsmi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -1 $O/gputests.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
timeout 600 python bench.py --workload c1 > $O/bench_c1.json 2> $O/bench_c1.err; echo c1=$?
timeout 600 python bench.py --workload c2 --no-cpu-baseline --no-pageable > $O/bench_c2.json 2> $O/bench_c2.err; echo c2=$?
timeout 600 python bench.py --workload c5 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; echo c5=$?
timeout 900 python bench.py --workload c4 --steps 3 --no-cpu-baseline > $O/bench_c4_nocpu.json 2> $O/bench_c4.err; echo c4=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pageable > /dev/null 2> $O/c3_under_ncu.err; echo ncu_list=$?
timeout 1500 python bench.py --impl reference > $O/bench_ref_c3.json 2> $O/bench_ref_c3.err; echo ref=$?
for f in $O/bench_c*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['value'], d['roofline']['frac'], d['roofline'].get('dram_frac'), d['e2e']['value'], (d.get('cpu_baseline') or {}).get('value'))" 2>&1 | tail -1; done
python -c "import json; d=json.load(open('$O/bench_ref_c3.json')); print('ref', d['value'], d['e2e']['value'])" 2>&1 | tail -1
