"""pipecg bring-up repro: C2-like system (100^3, 8 ranks -> 1 part), update +
cg_solve(method) per timestep; prints iterations per step."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_08536_b200 as lrb  # noqa: E402

N = int(os.environ.get("N", "100"))
NCPU, ALPHA = int(os.environ.get("NCPU", "8")), int(os.environ.get("ALPHA", "8"))
method = sys.argv[1] if len(sys.argv) > 1 else "pipecg"
steps = [int(s) for s in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["2", "3", "4"])]
hist = os.environ.get("HIST", "0") == "1"
parts = lrb.decompose_slab(lrb.StructuredGrid(N, N, N), NCPU)
asm = [lrb.assemble_poisson(p) for p in parts]
pm = lrb.make_partition_map([p.n_cells for p in parts], ALPHA)


def program(ctx):
    m, ifs = asm[ctx.rank]
    s = lrb.repartition(m, ifs, pm, ctx)
    out = []
    for st in steps:
        lrb.update(s, *lrb.perturb_coefficients(m, ifs, st), "direct")
        if s.is_owner:
            t0 = time.time()
            try:
                x, rep = lrb.cg_solve(s.matrix, s.halo, np.ones(s.matrix.n_owned), 1e-6, 2000, s.comm,
                                      method=method, history=hist)
                out.append((st, rep.iterations, rep.converged, rep.residual, round(time.time() - t0, 3)))
            except Exception as e:   # noqa: BLE001
                out.append((st, "ERR", repr(e)[:200]))
                print(out, flush=True)
                raise
    return out


res = lrb.run_world(NCPU, program)
print(method, N, NCPU, ALPHA, hist, res[0], flush=True)
