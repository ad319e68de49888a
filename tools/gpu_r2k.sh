# rpg sweep (C3 at 1 GPU) and the full reference arm as the driver runs it.
set -x
O=gpurun_out/r2k; mkdir -p $O
rm -f profiles/r2_curves_c3.csv.jsonl
timeout 2400 python tools/curves.py --steps 10 --out $O/r2_curves_c3.csv > $O/curves.log 2>&1; echo curves=$?; cat $O/curves.log
( time timeout 2400 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err ) 2> $O/bench_ref.time; echo ref=$?; cat $O/bench_ref.time; head -c 600 $O/bench_ref.json
