"""How far the pipelined PCG's recurrence residuals sit from the reference's
recorded CG logs at C3 (200^3, 8 ranks -> 1 part), timesteps 2..21: prints
one JSON line per method with the max relative deviation and iteration
differences.  Test infrastructure (reads tests/golden)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2510_08536_b200 as lrb  # noqa: E402
from golden_cases import large, ref_history  # noqa: E402
from helpers_b200 import cavity_case  # noqa: E402

TOL = 1e-6
g = large("c3")
_, asm, pm = cavity_case((200, 200, 200), 8, 8)
methods = sys.argv[1:] or ["pipecg", "pcg"]


def program(ctx):
    m, ifs = asm[ctx.rank]
    s = lrb.repartition(m, ifs, pm, ctx)
    out = {}
    for st in range(2, 22):
        lrb.update(s, *lrb.perturb_coefficients(m, ifs, st), "direct")
        if s.is_owner:
            for meth in methods:
                _, rep = lrb.cg_solve(s.matrix, s.halo, np.ones(s.matrix.n_owned), TOL, 2000, s.comm,
                                      method=meth, history=True)
                out[(meth, st)] = rep
    return out


res = lrb.run_world(8, program, timeout=3600)[0]
for meth in methods:
    devs, dits = [], []
    for st in range(2, 22):
        rep = res[(meth, st)]
        it_ref = int(g[f"k0__cg_{st}_rep"][0])
        ref = ref_history(g[f"k0__cg_{st}_log"], it_ref, TOL)
        n = min(len(ref), len(rep.history))
        devs.append(float(np.max(np.abs(np.asarray(rep.history[:n]) - ref[:n]) / ref[:n])))
        dits.append(rep.iterations - it_ref)
    print(json.dumps({"method": meth, "max_rel_dev": max(devs), "per_step_dev": devs, "iter_diff": dits}))
