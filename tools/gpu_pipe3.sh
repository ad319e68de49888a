O=gpurun_out/${1:-pipe6}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -2 $O/gputests.log
for w in c1 c2 c3; do for d in 0 1; do
  LRB_PIPE_DEFER=$d timeout 600 python bench.py --workload $w --method pipecg --no-cpu-baseline --no-pageable > $O/bench_${w}_pipecg_d$d.json 2> $O/bench_${w}_d$d.err
  python -c "import json; d=json.load(open('$O/bench_${w}_pipecg_d$d.json')); print('$w defer=$d', d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['e2e']['value'])" 2>&1 | tail -1
done; done
