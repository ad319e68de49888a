# A/B: interpreter switch interval while rank threads run (e2e host overhead).
O=gpurun_out/${1:-sw}; mkdir -p $O; : > $O/ab.txt
for round in 1 2; do for w in c1 c2 c3; do for si in "" 0.0001 0.00001; do
  LRB_SWITCH_INTERVAL_S=$si timeout 300 python bench.py --workload $w --no-cpu-baseline --no-pageable > $O/ab.json 2> $O/ab.err
  echo "$round $w si=${si:-default} $(python -c "import json; d=json.load(open('$O/ab.json')); e=d['e2e']; print(d['value'], e['value'], e['update_wall_ms'], e['solve_wall_ms'], e['solve_kernel_ms'])" 2>&1 | tail -1)" >> $O/ab.txt
done; done; done
cat $O/ab.txt
