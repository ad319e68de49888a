# Final round-2 evidence pass on one B200 (flat barrier + header cache build):
# smoke, all GPU tests, every BASELINE config's bench line, the launch list of
# the headline bench command and a full ncu capture of the C3 solve kernel.
set -x
O=gpurun_out/r2final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -3 $O/gputests.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
timeout 600 python bench.py --workload c1 > $O/bench_c1.json 2> $O/bench_c1.err; echo c1=$?
timeout 600 python bench.py --workload c2 --no-cpu-baseline --no-pageable > $O/bench_c2.json 2> $O/bench_c2.err; echo c2=$?
timeout 600 python bench.py --workload c5 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; echo c5=$?
timeout 900 python bench.py --workload c4 --steps 3 --no-cpu-baseline > $O/bench_c4_nocpu.json 2> $O/bench_c4_nocpu.err; echo c4=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pageable > /dev/null 2> $O/bench_under_ncu.err; echo ncu=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:team_cg -c 1 -o $O/prof_solve python tools/profile_step.py --step 6 > $O/profile_step.json 2> $O/prof_solve.err; echo ncu_solve=$?
timeout 2400 python bench.py --workload c4 --steps 3 > $O/bench_c4.json 2> $O/bench_c4.err; echo c4cpu=$?
for f in $O/bench_c*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['value'], d['roofline']['frac'], d['e2e']['value'], (d.get('cpu_baseline') or {}).get('value'))"; done
