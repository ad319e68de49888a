O=gpurun_out/${1:-pipe8}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_krylov.py -q -x -k "repeated" > $O/tests.log 2>&1; echo tests=$?; tail -1 $O/tests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:team_pipecg -c 1 -o $O/prof_c3_pipecg python tools/profile_step.py --step 6 --method pipecg > $O/profile_step_c3.json 2> $O/prof_c3.err; echo ncu=$?
