export LRB_BARRIER_TIMEOUT_S=3
timeout 120 python tools/pipe_repro.py pipecg 2,2,3,2,2,2 2>&1 | tail -1
N=200 timeout 120 python tools/pipe_repro.py pipecg 2,2,3 2>&1 | tail -1
