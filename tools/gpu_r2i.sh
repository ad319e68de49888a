# fused true-residual check: correctness + A/B against -DLRB_FUSE_CHECK=0
set -x
O=gpurun_out/r2i; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py tests/test_gpu_halo.py tests/test_gpu_large.py -x -q > $O/tests.log 2>&1; echo tests=$?; tail -3 $O/tests.log
for L in libldurepart_b200 libldurepart_b200_nofuse; do
  LRB_LIB=paper_2510_08536_b200/$L.so timeout 600 python tools/phase_profile.py --step 2 --repeat 2 > $O/phase_$L.json 2> $O/phase_$L.err; echo phase_$L=$?
  LRB_LIB=paper_2510_08536_b200/$L.so timeout 900 python bench.py --steps 10 --no-cpu-baseline --no-pageable > $O/bench_$L.json 2> $O/bench_$L.err; echo bench_$L=$?
  python -c "import json; d=json.load(open('$O/bench_$L.json')); r=d['roofline']; print('$L', d['value'], r['kernel_ms'], r['frac'], r.get('dram_frac'), d['breakdown']['iterations'])"
done
head -c 1500 $O/phase_libldurepart_b200.json; echo; head -c 1500 $O/phase_libldurepart_b200_nofuse.json
