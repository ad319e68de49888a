"""Golden fixtures at the BASELINE sizes (C3, C4, C5), made by running the REFERENCE.

Build container only (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_large.py [case ...]

Cases (BASELINE.json configs; the decomposition is the one the bench runs):

* ``c3``      200^3, 8 ranks -> 1 owner (alpha 8): digests of every integer
              artifact, value digests at timesteps 2 and 3, and the recorded
              allreduce log (``cg_solve`` through a recording comm)
              of every timestep 2..21 — the bench's timed window.
* ``c3r16a2`` 200^3, 16 ranks -> 8 owners (alpha 2, SURVEY §6's measured
              case): value digests at step 2, CG log of step 2 (multi-part).
* ``c5``      200^3, 128 ranks -> 8 owners (alpha 16), update only: integer and
              value digests of every owner at timesteps 2 and 3.
* ``c4``      300^3, 16 ranks -> 1 owner (alpha 16, the bench's C4 pressure
              system): value digest at step 2, CG logs of steps 2 and 3.

Writes ``tests/golden/golden_large_<case>.npz``: digests, logs and reports only
(a few KB each).  Digests are sha256 over dtype string + bytes of the
reference's own arrays (int64 indices, bool masks, f64 values), the same
convention as make_golden.py.
"""

import hashlib
import os
import sys
import time

import numpy as np

import ldurepart as lr  # the reference (read-only mount)

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    # name: (N, n_cpu, alpha, value steps, solve steps, full integer digests)
    "c3": (200, 8, 8, (2, 3), tuple(range(2, 22)), True),
    "c3r16a2": (200, 16, 2, (2,), (2,), False),
    "c5": (200, 128, 16, (2, 3), (), True),
    "c4": (300, 16, 16, (2,), (2, 3), False),
}


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + a.tobytes()).hexdigest()


class RecordingComm:
    """Delegates to a reference CommGroup and records allreduce_sum results."""

    def __init__(self, comm):
        self._comm = comm
        self.log = []

    def allreduce_sum(self, value):
        out = self._comm.allreduce_sum(value)
        self.log.append(float(out))
        return out

    def __getattr__(self, name):
        return getattr(self._comm, name)


def run(name):
    N, n_cpu, alpha, vsteps, ssteps, ints = CASES[name]
    grid = lr.StructuredGrid(N, N, N)
    parts = lr.decompose_slab(grid, n_cpu)
    pm = lr.make_partition_map([p.n_cells for p in parts], alpha)
    store = {"meta": np.array([N, n_cpu, alpha, pm.n_gpu], np.int64),
             "offsets": pm.offsets.copy()}
    t0 = time.monotonic()

    def program(ctx):
        m, ifs = lr.assemble_poisson(parts[ctx.rank])
        parts[ctx.rank] = None
        system = lr.repartition(m, ifs, pm, ctx)
        out = {}
        if system.is_owner:
            mat = system.matrix
            out["recv_offsets"] = system.update_pattern.recv_offsets[system.gpu_rank].copy()
            out["halo_cols"] = mat.halo_cols.copy()
            out["nnz"] = np.array([mat.local.nnz, mat.non_local.nnz], np.int64)
            if ints:
                for key, arr in (("local_rows", mat.local.rows), ("local_cols", mat.local.cols),
                                 ("nl_rows", mat.non_local.rows), ("nl_cols", mat.non_local.cols),
                                 ("to_local", system.scatter.to_local),
                                 ("index", system.scatter.index)):
                    out[f"{key}__sha256"] = digest(arr)
        for s in sorted(set(vsteps) | set(ssteps)):
            m_s, if_s = lr.perturb_coefficients(m, ifs, s)
            lr.update(system, m_s, if_s, "direct")
            if not system.is_owner:
                continue
            if s in vsteps:
                out[f"vals_{s}_local__sha256"] = digest(system.matrix.local.vals)
                out[f"vals_{s}_nl__sha256"] = digest(system.matrix.non_local.vals)
            if s in ssteps:
                rc = RecordingComm(system.comm)
                b = np.ones(system.matrix.n_owned)
                ts = time.monotonic()
                x, rep = lr.cg_solve(system.matrix, system.halo, b, 1e-6, 2000, rc)
                out[f"cg_{s}_log"] = np.array(rc.log)
                out[f"cg_{s}_rep"] = np.array([rep.iterations, rep.residual, float(rep.converged),
                                               time.monotonic() - ts])
                out[f"cg_{s}_x__norm"] = np.float64(np.linalg.norm(x))
                out[f"cg_{s}_x__sample997"] = x[::997].copy()
                if ctx.rank == 0:
                    print(f"  {name} step {s}: {rep.iterations} its, "
                          f"{time.monotonic() - ts:.1f}s", file=sys.stderr, flush=True)
        return out

    results = lr.run_world(n_cpu, program, timeout=1e7)
    for k in range(pm.n_gpu):
        for key, val in results[alpha * k].items():
            store[f"k{k}__{key}"] = np.asarray(val)
    store["t_total_s"] = np.float64(time.monotonic() - t0)
    out = os.path.join(HERE, f"golden_large_{name}.npz")
    np.savez_compressed(out, **store)
    print(f"{name}: {len(store)} arrays -> {out} ({time.monotonic() - t0:.1f}s)",
          file=sys.stderr, flush=True)


def main():
    for name in sys.argv[1:] or list(CASES):
        run(name)


if __name__ == "__main__":
    main()
