# pipecg bring-up: its GPU tests, then C1/C2/C3 bench lines for pcg, pcg1, pipecg.
set -x
O=gpurun_out/${1:-pipe}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_stream.py -q -x -k "pipecg" > $O/tests.log 2>&1; echo tests=$?; tail -15 $O/tests.log
for w in c1 c2 c3; do for m in pcg pcg1 pipecg; do
  timeout 600 python bench.py --workload $w --method $m --no-cpu-baseline --no-pageable > $O/bench_${w}_$m.json 2> $O/bench_${w}_$m.err; echo $w $m $?
done; done
for f in $O/bench_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['value'], d['roofline']['frac'], d['roofline'].get('kernel_ms'), sum(d['breakdown']['iterations']))" 2>&1 | tail -1; done
