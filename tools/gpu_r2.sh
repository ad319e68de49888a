# Round-2 evidence pass on one B200: smoke, GPU tests, bench (C3 headline +
# C4/C5), reference arm, launch list of the bench command, full ncu captures of
# the scatter and the solve kernel.  Outputs under gpurun_out/r2/.
set -x
O=gpurun_out/r2; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?
tail -3 $O/gputests.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?
cat $O/bench.json
timeout 900 python bench.py --workload c5 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; echo c5=$?
timeout 900 python bench.py --workload c4 --steps 3 --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err; echo c4=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pageable > /dev/null 2> $O/bench_under_ncu.err; echo ncu=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:team_cg -c 1 -o $O/prof_solve python tools/profile_step.py --step 6 > $O/profile_step.json 2> $O/prof_solve.err; echo ncu_solve=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scatter -c 2 -o $O/prof_scatter python tools/profile_step.py --step 6 > /dev/null 2> $O/prof_scatter.err; echo ncu_scatter=$?
