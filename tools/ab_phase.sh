# A/B of library variants: per-phase times (C3 step 2) and the bench value.
#   bash tools/ab_phase.sh OUTDIR lib1.so lib2.so ...
O=$1; shift; mkdir -p $O
for L in "$@"; do
  b=$(basename $L .so)
  LRB_LIB=$L timeout 600 python tools/phase_profile.py --step 2 --repeat 2 > $O/phase_$b.json 2> $O/phase_$b.err
  python -c "
import json
for l in open('$O/phase_$b.json'):
    d=json.loads(l)
    if d['family']=='stream': print('$b', 'solve_ms', d['device_ms'], {k: d[k]['us'] for k in d if k in ('A','A_sync','B','B_sync','C','C_sync')})"
  LRB_LIB=$L timeout 900 python bench.py --steps 10 --no-cpu-baseline --no-pageable > $O/bench_$b.json 2> $O/bench_$b.err
  python -c "import json; d=json.load(open('$O/bench_$b.json')); r=d['roofline']; print('$b', 'bench', d['value'], r['kernel_ms'], r['frac'])"
done
