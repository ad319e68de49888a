"""Record the REFERENCE's CG iteration counts per timestep at the bench configs.

The bench's CPU-baseline leg times a bounded sample of the reference algorithm
(update + a few CG iterations, see bench.py) and scales it to a full timestep
with these counts, so it does not need 30 s of CPU per step on the GPU box.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_iters_c3.py [N n_cpu alpha steps]

Writes tests/golden/iters_<N>_r<n_cpu>_a<alpha>.json.
"""

import json
import os
import sys
import time

import numpy as np

import ldurepart as lr


def main():
    n, n_cpu, alpha, n_steps = (int(v) for v in (sys.argv[1:] or [200, 8, 8, 24]))
    grid = lr.StructuredGrid(n, n, n)
    parts = lr.decompose_slab(grid, n_cpu)
    pm = lr.make_partition_map([p.n_cells for p in parts], alpha)
    rows = []

    def program(ctx):
        m, ifs = lr.assemble_poisson(parts[ctx.rank])
        t0 = time.monotonic()
        system = lr.repartition(m, ifs, pm, ctx)
        t_create = time.monotonic() - t0
        for step in range(2, n_steps + 1):
            m_s, if_s = lr.perturb_coefficients(m, ifs, step)
            t0 = time.monotonic()
            lr.update(system, m_s, if_s, "direct")
            t_up = time.monotonic() - t0
            if system.is_owner:
                b = np.ones(system.matrix.n_owned)
                t0 = time.monotonic()
                _, rep = lr.cg_solve(system.matrix, system.halo, b, 1e-6, 2000, system.comm)
                t_solve = time.monotonic() - t0
                if ctx.rank == 0:
                    rows.append({"step": step, "iterations": rep.iterations,
                                 "residual": rep.residual, "t_update_s": t_up,
                                 "t_solve_s": t_solve})
                    print(rows[-1], file=sys.stderr, flush=True)
        return t_create

    t_create = lr.run_world(n_cpu, program, timeout=1e6)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                       f"iters_{n}_r{n_cpu}_a{alpha}.json")
    with open(out, "w") as fh:
        json.dump({"config": {"N": n, "n_cpu": n_cpu, "alpha": alpha, "tol": 1e-6},
                   "t_create_s": max(t_create), "steps": rows,
                   "note": "reference ldurepart run in the build container (1 core, "
                           "deterministic world); timings are context only"}, fh, indent=1)


if __name__ == "__main__":
    main()
