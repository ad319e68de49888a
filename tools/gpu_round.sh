set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
ls MEASURED_PEAKS.json && cat MEASURED_PEAKS.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests=$?
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
