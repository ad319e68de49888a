# ncu evidence for profiles/: full capture of the solve kernel and of one
# scatter launch (one C3 timestep), plus the launch list of the same command.
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:team_cg -c 1 -o gpurun_out/prof_solve python tools/profile_step.py --step 6 > gpurun_out/profile_step.json 2> gpurun_out/prof_solve.err; echo ncu_solve=$?
timeout 900 ncu --set full --clock-control none -k regex:scatter_rows -c 2 -o gpurun_out/prof_scatter python tools/profile_step.py --step 6 > /dev/null 2> gpurun_out/prof_scatter.err; echo ncu_scatter=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --step 6 > /dev/null 2> gpurun_out/launches.err; echo ncu_launches=$?
cat gpurun_out/profile_step.json
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json
