export LRB_BARRIER_TIMEOUT_S=10
V=$PWD/paper_2510_08536_b200/var_t448.so
LRB_LIB=$V timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
LRB_LIB=$PWD/paper_2510_08536_b200/var_t448_prof.so timeout 300 python tools/phase_profile.py 2>/dev/null | head -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('t448', 'stages', d['info']['stages'], d['info']['stage_bytes'], {k:d[k]['us'] for k in ('A','B','C','A_sync','B_sync')}, 'A waits', d['waits_us']['A'])"
bash tools/variants.sh $PWD/paper_2510_08536_b200/libldurepart_b200.so $V 2>&1 | grep -v "^  \|Traceback\|^json\|^    "
