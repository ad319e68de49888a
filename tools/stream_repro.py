"""Streaming vs classic on growing single-part cavities (bit-identity + liveness)."""
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2510_08536_b200 as lrb
from helpers_b200 import cavity_case
from paper_2510_08536_b200.device import Team

for dims, n_cpu in [tuple(map(int, a.split(":")[0].split("x"))) + () and (tuple(map(int, a.split(":")[0].split("x"))), int(a.split(":")[1])) for a in (sys.argv[1:] or ["40x40x40:2", "64x64x64:2", "100x100x100:4"])]:
    _, asm, pm = cavity_case(dims, n_cpu, n_cpu)
    holder = {}

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        parts = s.comm.allgather(s.part) if s.is_owner else None
        if s.is_owner and s.comm.group_rank == 0:
            holder["parts"] = parts
            holder["keep"] = s
        return None

    lrb.run_world(n_cpu, program)
    parts = holder["parts"]
    os.environ["LRB_SOLVER"] = "classic"
    tc = Team(parts)
    os.environ.pop("LRB_SOLVER")
    ts = Team(parts)
    bs = [np.ones(p.n) for p in parts]
    for method in ("cg", "pcg"):
        xa, ra, ha = tc.solve(method, bs, 1e-9, 500, hist_cap=500)
        print(dims, method, "classic", ra.iterations, flush=True)
        xb, rb, hb = ts.solve(method, bs, 1e-9, 500, hist_cap=500)
        same = all(np.array_equal(a, b) for a, b in zip(xa, xb)) and np.array_equal(ha, hb)
        print(dims, method, "stream", rb.iterations, "identical" if same else "DIFFERENT", ts.kernel_info(method),
              flush=True)
