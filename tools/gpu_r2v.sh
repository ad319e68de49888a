# Final-code evidence: ncu of the C3 solve kernel + launch list of the bench
# command, full GPU suite, bench line.
set -x
O=gpurun_out/r2v; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:team_cg -c 1 -o $O/prof_solve python tools/profile_step.py --step 6 > $O/profile_step.json 2> $O/prof_solve.err; echo ncu_solve=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pageable > /dev/null 2> $O/bench_under_ncu.err; echo ncu=$?
timeout 1800 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -3 $O/gputests.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?
python -c "import json; d=json.load(open('$O/bench.json')); r=d['roofline']; print(d['value'], r['frac'], r.get('dram_frac'), d['e2e']['value'], d['cpu_baseline']['value'])"
