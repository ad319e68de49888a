O=gpurun_out/${1:-pipe7}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -2 $O/gputests.log
for w in c1 c2 c3; do
  timeout 600 python bench.py --workload $w --method pipecg --no-cpu-baseline --no-pageable > $O/bench_${w}_pipecg.json 2> $O/bench_${w}_pipecg.err
  python -c "import json; d=json.load(open('$O/bench_${w}_pipecg.json')); g=d['roofline']['kernel_geometry']; print('$w pipecg', d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], g['stages'], g['stage_bytes'])" 2>&1 | tail -1
done
timeout 600 python bench.py --workload c3 --no-cpu-baseline --no-pageable > $O/bench_c3_pcg.json 2> $O/bench_c3_pcg.err
python -c "import json; d=json.load(open('$O/bench_c3_pcg.json')); print('c3 pcg', d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'])" 2>&1 | tail -1
