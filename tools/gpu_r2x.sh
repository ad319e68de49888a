set -x
O=gpurun_out/r2x; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_stream.py tests/test_gpu_halo.py tests/test_gpu_api.py tests/test_gpu_parity.py -x -q > $O/tests.log 2>&1; echo tests=$?; tail -3 $O/tests.log
timeout 600 python tools/split_overhead.py > $O/split200.jsonl 2>/dev/null; cat $O/split200.jsonl
timeout 600 python tools/split_overhead.py --n 100 > $O/split100.jsonl 2>/dev/null; cat $O/split100.jsonl
timeout 600 python tools/phase_profile.py --n 100 --ranks 64 --alpha 8 > $O/phase_c2.json 2>/dev/null; head -c 600 $O/phase_c2.json
