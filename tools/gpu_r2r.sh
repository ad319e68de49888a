# compute-sanitizer over the round-2 code paths: async ABI, halo mirrors,
# update epochs / device producer, multi-part barrier, multi-team geometry
set -x
O=gpurun_out/r2r; mkdir -p $O
SAN="compute-sanitizer --target-processes all --print-limit 20"
timeout 1200 $SAN --tool memcheck python -m pytest tests/test_gpu_async.py tests/test_gpu_halo.py -x -q > $O/san_memcheck_async_halo.log 2>&1; echo m1=$?
timeout 1200 $SAN --tool memcheck python -m pytest tests/test_gpu_api.py -x -q -k "update_on_device or two_systems or vals_write or pageable_update" > $O/san_memcheck_update.log 2>&1; echo m2=$?
timeout 1200 $SAN --tool memcheck python -m pytest tests/test_gpu_stream.py -x -q -k "coexist or split_devices" > $O/san_memcheck_stream.log 2>&1; echo m3=$?
timeout 1200 $SAN --tool synccheck python -m pytest tests/test_gpu_halo.py -x -q -k "bit_identical" > $O/san_synccheck_halo.log 2>&1; echo s1=$?
timeout 1200 $SAN --tool initcheck python -m pytest tests/test_gpu_halo.py -x -q -k "not_stale" > $O/san_initcheck_halo.log 2>&1; echo i1=$?
for f in $O/san_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|passed|failed" $f | tail -2; done
