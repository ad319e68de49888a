export LRB_BARRIER_TIMEOUT_S=10
timeout 900 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -3
for w in c1 c2 c3; do for m in pcg pcg1; do
timeout 600 python bench.py --workload $w --method $m --no-cpu-baseline > gpurun_out/b_${w}_$m.json 2>gpurun_out/b_${w}_$m.err
python -c "import json; d=json.load(open('gpurun_out/b_${w}_$m.json')); print('$w $m', d['value'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['e2e']['value'], d['breakdown']['iterations'][:4])" || tail -3 gpurun_out/b_${w}_$m.err
done; done
