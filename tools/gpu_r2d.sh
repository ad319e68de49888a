# Halo mirrors + writable vals: tests, C3/C2 benches (mirrors vs LRB_HALO=direct),
# whole-part scatter ncu (skip the 8 create + 8 update per-segment launches).
set -x
O=gpurun_out/r2d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_halo.py tests/test_gpu_api.py tests/test_gpu_async.py -x -q > $O/halo_tests.log 2>&1; echo halo=$?; tail -3 $O/halo_tests.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -3 $O/gputests.log
timeout 900 python bench.py --no-cpu-baseline --no-pageable > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
timeout 900 python bench.py --workload c2 --no-cpu-baseline --no-pageable > $O/bench_c2.json 2> $O/bench_c2.err; echo c2=$?
LRB_HALO=direct timeout 900 python bench.py --workload c2 --no-cpu-baseline --no-pageable > $O/bench_c2_direct.json 2> $O/bench_c2_direct.err; echo c2d=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scatter --launch-skip 16 -c 1 -o $O/prof_scatter_part python tools/scatter_bench.py --reps 1 > /dev/null 2> $O/ncu_scatter.err; echo ncu_scatter=$?
for f in $O/bench_c*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['roofline']['frac'], d.get('e2e',{}).get('value'))"; done
