# Evidence pass for the pipecg build: smoke, all GPU tests, C3 / C1 bench
# lines, the C1 launch list and a full ncu of the C1 pipecg solve launch.
O=gpurun_out/${1:-r2pf}; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -2 $O/gputests.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
timeout 600 python bench.py --workload c1 > $O/bench_c1.json 2> $O/bench_c1.err; echo c1=$?
timeout 600 python bench.py --workload c2 --no-cpu-baseline --no-pageable > $O/bench_c2.json 2> $O/bench_c2.err; echo c2=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c1_launches.csv python bench.py --workload c1 --steps 2 --warmup 3 --no-cpu-baseline --no-pageable > /dev/null 2> $O/c1_under_ncu.err; echo ncu_list=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:team_pipecg -c 1 -o $O/prof_c1_pipecg python tools/profile_step.py --n 32 --ranks 4 --step 5 --method pipecg > $O/profile_step_c1.json 2> $O/prof_c1.err; echo ncu_full=$?
for f in $O/bench_c*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['value'], d['roofline']['frac'], d['e2e']['value'], (d.get('cpu_baseline') or {}).get('value'))"; done
