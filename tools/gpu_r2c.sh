# ncu of the whole-part scatter and of the C4 solve kernels; compute-sanitizer
# (memcheck / racecheck / synccheck) over the hand-rolled synchronisation.
set -x
O=gpurun_out/r2c; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scatter --launch-skip 8 -c 1 -o $O/prof_scatter_part python tools/scatter_bench.py --reps 1 > $O/scatter_part.json 2> $O/ncu_scatter.err; echo ncu_scatter=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:team_bicgstab -c 1 -o $O/prof_c4_bicgstab python tools/profile_step.py --n 300 --ranks 16 --method bicgstab --step 3 > $O/profile_c4_bicgstab.json 2> $O/ncu_c4b.err; echo ncu_c4b=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:team_cg -c 1 -o $O/prof_c4_pcg python tools/profile_step.py --n 300 --ranks 16 --step 3 > $O/profile_c4_pcg.json 2> $O/ncu_c4p.err; echo ncu_c4p=$?
SAN="compute-sanitizer --target-processes all --print-limit 20"
K="cross_device_protocol or chain8_cg or bicgstab_matches_oracle"
timeout 900 $SAN --tool memcheck python -m pytest tests/test_gpu_api.py -x -q -k "$K" > $O/san_memcheck_api.log 2>&1; echo memcheck=$?
timeout 900 $SAN --tool memcheck python -m pytest tests/test_gpu_async.py -x -q > $O/san_memcheck_async.log 2>&1; echo memcheck_async=$?
timeout 900 $SAN --tool racecheck python -m pytest tests/test_gpu_api.py -x -q -k "cross_device_protocol or chain8_cg" > $O/san_racecheck.log 2>&1; echo racecheck=$?
timeout 900 $SAN --tool synccheck python -m pytest tests/test_gpu_api.py -x -q -k "cross_device_protocol or chain8_cg" > $O/san_synccheck.log 2>&1; echo synccheck=$?
timeout 900 $SAN --tool racecheck python -m pytest tests/test_gpu_stream.py -x -q -k "ring_depth" > $O/san_racecheck_ring.log 2>&1; echo racecheck_ring=$?
timeout 900 $SAN --tool synccheck python -m pytest tests/test_gpu_stream.py -x -q -k "ring_depth" > $O/san_synccheck_ring.log 2>&1; echo synccheck_ring=$?
timeout 600 $SAN --tool memcheck python tools/ipc_selftest.py > $O/san_memcheck_ipc.log 2>&1; echo memcheck_ipc=$?
for f in $O/san_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" $f | tail -3; done
