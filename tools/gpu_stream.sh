# streaming solver: parity tests, bench classic vs streaming, ncu of the streaming solve
set -x
export LRB_BARRIER_TIMEOUT_S=20
timeout 600 python -m pytest tests/test_gpu_stream.py -x -q > gpurun_out/stream_tests.log 2>&1; echo stream_tests=$?
tail -30 gpurun_out/stream_tests.log
if [ "${FULL:-0}" = 1 ]; then timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests=$?; tail -5 gpurun_out/gputests.log; fi
LRB_SOLVER=classic timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_classic.json 2> gpurun_out/bench_classic.err; echo bench_classic=$?
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_stream.json 2> gpurun_out/bench_stream.err; echo bench_stream=$?
python -c "
import json
for f in ('classic','stream'):
    try:
        d=json.load(open('gpurun_out/bench_%s.json'%f)); print(f, d['value'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['breakdown']['iterations'], d['e2e']['value'])
    except Exception as e: print(f, 'ERR', e)
"
if [ "${PROF:-0}" = 1 ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:team_cg_stream -c 1 -o gpurun_out/prof_stream python tools/profile_step.py --step 6 > gpurun_out/prof_stream.log 2>&1; echo ncu=$?
tail -3 gpurun_out/prof_stream.log
fi
if [ "${PHASE:-0}" = 1 ]; then
LRB_LIB=$PWD/paper_2510_08536_b200/libldurepart_b200_prof.so timeout 600 python tools/phase_profile.py > gpurun_out/phase.json 2> gpurun_out/phase.err; echo phase=$?
cat gpurun_out/phase.json; tail -3 gpurun_out/phase.err
fi
