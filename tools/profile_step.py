"""One C3 timestep under ncu: update (8 segment scatters) + one PCG solve.
(``--n 300 --ranks 16 --method bicgstab``: one C4 momentum BiCGStab solve on
the bench's momentum coefficients, right-hand side Ux.)

    ncu --set full -k regex:team_cg -c 1 -o gpurun_out/prof python tools/profile_step.py --step 5
    ncu --metrics gpu__time_duration.sum --csv --log-file ... python tools/profile_step.py

Prints one JSON line with the solve's iteration count and the algorithmic
bytes of that launch, so tools/summarize_ncu.py can relate ncu's DRAM bytes
to the algorithmic figure of the same launch.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import (MAX_ITER, TOL, Problem, bicgstab_bytes, momentum_eps, momentum_rhs,  # noqa: E402
                   momentum_values_into, n_checks, solve_bytes)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200)
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--step", type=int, default=5)
    ap.add_argument("--method", default="pcg")
    args = ap.parse_args()
    import paper_2510_08536_b200 as lrb
    prob = Problem(args.n, args.ranks, range(args.ranks))
    pm = lrb.make_partition_map(prob.cells, args.ranks)
    out = {}

    mom = args.method == "bicgstab"

    def inputs(r):
        if not mom:
            return prob.produce(r, args.step)
        m, ifs = prob.base[r]
        eu, el = momentum_eps(m, r)
        up, lo = np.zeros(m.n_faces), np.zeros(m.n_faces)
        momentum_values_into(eu, el, args.step, up, lo)
        return lrb.LduMatrix(m.n_cells, m.lower_addr, m.upper_addr, np.full(m.n_cells, 6.5), lo,
                             up), ifs

    def program(ctx):
        r = ctx.rank
        s = lrb.repartition(*prob.base[r], pm, ctx)
        lrb.update(s, *inputs(r), "direct")
        if s.is_owner:
            b = momentum_rhs(s.matrix.n_owned, 0) if mom else np.ones(s.matrix.n_owned)
            solve = lrb.bicgstab_solve if mom else lrb.cg_solve
            kw = {} if mom else {"method": args.method}
            x, rep = solve(s.matrix, s.halo, b, TOL, MAX_ITER, s.comm, history=True, **kw)
            p = s.part.plan
            nnz = p.nnz_local + p.nnz_nonlocal
            ck = n_checks(rep.history, rep.iterations, TOL)
            alg = (bicgstab_bytes(p.n, nnz, p.n_halo, rep.iterations, ck) if mom else
                   solve_bytes(p.n, nnz, p.n_halo, rep.iterations, ck, args.method))
            out.update(step=args.step, iterations=rep.iterations, checks=ck, n=p.n, nnz=nnz,
                       method=args.method,
                       sell_entries=p.sell_entries, uniform_entries=p.uniform_entries,
                       alg_bytes=alg,
                       scatter_alg_bytes=20 * p.n_buf, device_ms=rep.device_ms)

    lrb.run_world(args.ranks, program)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
