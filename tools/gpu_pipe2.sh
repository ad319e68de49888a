O=gpurun_out/${1:-pipe2}; mkdir -p $O
bash tools/pipe_repro.sh > $O/repro.txt 2>&1; cat $O/repro.txt
timeout 900 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_stream.py -q -x -k "pipecg" > $O/tests.log 2>&1; echo tests=$?; tail -2 $O/tests.log
bash tools/gpu_pipe_ab.sh $1 > /dev/null 2>&1; cat $O/ab.txt
