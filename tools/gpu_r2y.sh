set -x
O=gpurun_out/r2y; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo tests=$?; tail -3 $O/gputests.log
timeout 600 python tools/split_overhead.py > $O/split200.jsonl 2>/dev/null; cat $O/split200.jsonl
timeout 600 python tools/split_overhead.py --n 100 > $O/split100.jsonl 2>/dev/null; cat $O/split100.jsonl
