set -x
O=gpurun_out/r2g; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_api.py -x -q > $O/api.log 2>&1; echo api=$?; tail -3 $O/api.log
timeout 900 python tools/ref_suite.py -q > $O/ref_suite.log 2>&1; echo ref_suite=$?; tail -3 $O/ref_suite.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -3 $O/gputests.log
