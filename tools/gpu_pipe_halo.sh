O=gpurun_out/${1:-halo}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_halo.py tests/test_gpu_krylov.py tests/test_gpu_stream.py -q -x > $O/tests.log 2>&1; echo tests=$?; tail -1 $O/tests.log
for m in pipecg pcg; do timeout 600 python tools/split_overhead.py --n 200 --ranks 8 --repeat 2 --method $m 2>/dev/null > $O/split_200_$m.jsonl; cat $O/split_200_$m.jsonl | cut -c1-200; done
for m in pipecg; do LRB_HALO=direct timeout 600 python tools/split_overhead.py --n 200 --ranks 8 --repeat 2 --method $m 2>/dev/null > $O/split_200_${m}_direct.jsonl; cat $O/split_200_${m}_direct.jsonl | cut -c1-200; done
timeout 600 python bench.py --no-cpu-baseline --no-pageable > $O/c3.json 2>/dev/null; python -c "import json; d=json.load(open('$O/c3.json')); print('c3', d['value'])"
