"""Generate the golden parity fixtures by running the REFERENCE package.

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/golden.npz`` (small cases stored in full, larger cases as
sha256 digests plus solver histories).  Every array comes straight out of the
reference's public functions (``repartition``, ``fuse_patterns``,
``build_scatter_map``, ``build_halo_plan``, ``spmv``, ``cg_solve``), so the
fixtures pin the oracle and the CUDA path to the reference's own behaviour.

Residual histories are recovered without editing the reference: ``cg_solve``
is handed a delegating communicator that records every ``allreduce_sum``
result.  The log per solve is
``[b.b, (p.q, r.r, [|b-Ax|^2])...]``.
"""

import hashlib
import os
import sys
import time

import numpy as np

import ldurepart as lr  # the reference (read-only mount)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


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


def cavity(dims, n_cpu, alpha):
    grid = lr.StructuredGrid(*dims)
    parts = lr.decompose_slab(grid, n_cpu)
    assembled = [lr.assemble_poisson(p) for p in parts]
    pm = lr.make_partition_map([p.n_cells for p in parts], alpha)
    return grid, parts, assembled, pm


def run_case(store, name, pm, per_rank, full=True, steps=(), solve_steps=(),
             tol=1e-6, max_iter=2000, spmv_seed=None, perturb=True):
    """Repartition with the reference world; record integer and value outputs.

    ``per_rank`` holds the base (step-1) matrices.  ``steps`` lists
    perturbation steps whose scattered values are recorded; ``solve_steps``
    the steps (1 = base) whose CG solve history is recorded.
    """
    n_cpu = pm.n_cpu
    xs = None
    if spmv_seed is not None:
        rng = np.random.default_rng(spmv_seed)
        xs = rng.normal(size=(3, pm.total_cells))

    def program(ctx):
        m, ifs = per_rank[ctx.rank]
        system = lr.repartition(m, ifs, pm, ctx)
        out = {}
        if system.is_owner:
            mat = system.matrix
            out["local_rows"] = mat.local.rows.copy()
            out["local_cols"] = mat.local.cols.copy()
            out["nl_rows"] = mat.non_local.rows.copy()
            out["nl_cols"] = mat.non_local.cols.copy()
            out["halo_cols"] = mat.halo_cols.copy()
            out["to_local"] = system.scatter.to_local.copy()
            out["index"] = system.scatter.index.copy()
            out["vals_1_local"] = mat.local.vals.copy()
            out["vals_1_nl"] = mat.non_local.vals.copy()
            out["row_offset"] = np.int64(mat.row_offset)
            send = system.halo.send_indices
            recv = system.halo.recv_slots
            out["halo_send_nbrs"] = np.array(sorted(send), dtype=np.int64)
            out["halo_send_idx"] = (np.concatenate([send[j] for j in sorted(send)])
                                    if send else np.zeros(0, np.int64))
            out["halo_send_len"] = np.array([len(send[j]) for j in sorted(send)], np.int64)
            out["halo_recv_nbrs"] = np.array(sorted(recv), dtype=np.int64)
            out["halo_recv_idx"] = (np.concatenate([recv[j] for j in sorted(recv)])
                                    if recv else np.zeros(0, np.int64))
            out["halo_recv_len"] = np.array([len(recv[j]) for j in sorted(recv)], np.int64)
            if xs is not None:
                lo, hi = pm.gpu_range(mat.owner_gpu_rank)
                for i, x in enumerate(xs):
                    out[f"spmv_{i}"] = lr.spmv(mat, system.halo, x[lo:hi], system.comm)
        for s in sorted(set(steps) | set(solve_steps)):
            if s >= 2:
                m_s, if_s = lr.perturb_coefficients(m, ifs, s)
                lr.update(system, m_s, if_s, "direct")
                if system.is_owner and s in steps:
                    out[f"vals_{s}_local"] = system.matrix.local.vals.copy()
                    out[f"vals_{s}_nl"] = system.matrix.non_local.vals.copy()
            if s in solve_steps and system.is_owner:
                rc = RecordingComm(system.comm)
                b = np.ones(system.matrix.n_owned)
                x, rep = lr.cg_solve(system.matrix, system.halo, b, tol, max_iter, rc)
                out[f"cg_{s}_x"] = x
                out[f"cg_{s}_log"] = np.array(rc.log)
                out[f"cg_{s}_rep"] = np.array([rep.iterations, rep.residual,
                                               float(rep.converged)])
        if system.is_owner:
            out["recv_offsets"] = system.update_pattern.recv_offsets[system.gpu_rank].copy()
        return out

    t0 = time.monotonic()
    results = lr.run_world(n_cpu, program)
    store[f"{name}__meta"] = np.array([n_cpu, pm.alpha, pm.n_gpu, pm.total_cells], np.int64)
    store[f"{name}__offsets"] = pm.offsets.copy()
    for k in range(pm.n_gpu):
        res = results[pm.alpha * k]
        for key, val in res.items():
            val = np.asarray(val)
            big = val.size > 4096 and not key.startswith("cg_")
            if not full and key.startswith("cg_") and key.endswith("_x"):
                # solutions are tolerance-matched, not bit-exact: keep a strided sample
                store[f"{name}__k{k}__{key}__sample97"] = val[::97].copy()
                store[f"{name}__k{k}__{key}__norm"] = np.float64(np.linalg.norm(val))
            elif full or not big:
                store[f"{name}__k{k}__{key}"] = val
            else:
                store[f"{name}__k{k}__{key}__sha256"] = np.array(digest(val))
                store[f"{name}__k{k}__{key}__len"] = np.int64(val.size)
    print(f"  {name}: {time.monotonic() - t0:.1f}s", file=sys.stderr)


def store_inputs(store, name, pm, per_rank):
    """Random-system inputs, so the oracle and the CUDA path replay them."""
    store[f"{name}__in_cells"] = np.diff(pm.offsets)
    store[f"{name}__in_alpha"] = np.int64(pm.alpha)
    for r, (m, ifs) in enumerate(per_rank):
        p = f"{name}__in_r{r}"
        store[f"{p}__lower"] = m.lower_addr
        store[f"{p}__upper"] = m.upper_addr
        store[f"{p}__diag"] = m.diag
        store[f"{p}__lval"] = m.lower_val
        store[f"{p}__uval"] = m.upper_val
        store[f"{p}__nbr"] = np.array([b.neighbor_rank for b in ifs], np.int64)
        store[f"{p}__blen"] = np.array([len(b) for b in ifs], np.int64)
        cat = lambda f: (np.concatenate([f(b) for b in ifs]) if ifs else np.zeros(0))
        store[f"{p}__irow"] = cat(lambda b: b.rows).astype(np.int64)
        store[f"{p}__icol"] = cat(lambda b: b.cols_remote).astype(np.int64)
        store[f"{p}__ival"] = cat(lambda b: b.values).astype(np.float64)


def random_system(rng, max_cells=50, max_ranks=4):
    """Same construction as the reference's tests/helpers.py:19-69."""
    sys.path.insert(0, "/root/reference/pkg/tests")
    from helpers import random_partitioned_system
    return random_partitioned_system(rng, max_cells=max_cells, max_ranks=max_ranks)


def main():
    store = {}
    t0 = time.monotonic()
    # W1 chain (SPEC worked example) and the 1D CG known answer
    for n_cpu, alpha in ((4, 1), (4, 2), (4, 4), (8, 1), (8, 2), (8, 4), (8, 8)):
        _, _, assembled, pm = cavity((8, 1, 1), n_cpu, alpha)
        run_case(store, f"chain{n_cpu}_a{alpha}", pm, assembled, steps=(3,),
                 solve_steps=(1,), tol=1e-10, max_iter=100, spmv_seed=3)
    # small 3D cases, full arrays
    for dims, n_cpu, alphas in (((6, 6, 6), 4, (1, 2, 4)),
                                ((12, 12, 12), 8, (1, 2, 4, 8)),
                                ((10, 10, 10), 5, (1, 5)),
                                ((7, 9, 11), 6, (1, 2, 3, 6))):
        for alpha in alphas:
            _, _, assembled, pm = cavity(dims, n_cpu, alpha)
            tag = "x".join(map(str, dims))
            run_case(store, f"cav{tag}_r{n_cpu}_a{alpha}", pm, assembled,
                     steps=(2, 3, 20), solve_steps=(1, 2, 3), spmv_seed=5)
    # 20^3 CG to 1e-8 (acceptance 6)
    for alpha in (1, 2, 4):
        _, _, assembled, pm = cavity((20, 20, 20), 4, alpha)
        run_case(store, f"cav20_r4_a{alpha}", pm, assembled, full=False,
                 solve_steps=(1,), tol=1e-8, max_iter=1000)
    # C1: 32^3, 4 ranks -> 1 device (digests + histories)
    _, _, assembled, pm = cavity((32, 32, 32), 4, 4)
    run_case(store, "c1", pm, assembled, full=False, steps=(2,),
             solve_steps=(2, 3, 4))
    # C2: 100^3, 64 ranks -> 8 parts (digests + histories, steps 2..3)
    if os.environ.get("GOLDEN_C2", "1") == "1":
        _, _, assembled, pm = cavity((100, 100, 100), 64, 8)
        run_case(store, "c2", pm, assembled, full=False, steps=(2,),
                 solve_steps=(2, 3))
    # random systems with non-symmetric values (acceptance 3 construction)
    rng = np.random.default_rng(2024)
    n_rand = 0
    for i in range(60):
        pm, per_rank, _ = random_system(rng)
        name = f"rand{i}"
        store_inputs(store, name, pm, per_rank)
        run_case(store, name, pm, per_rank, steps=(), solve_steps=(),
                 spmv_seed=100 + i)
        n_rand += 1
    store["rand__count"] = np.int64(n_rand)
    np.savez_compressed(OUT, **store)
    print(f"wrote {len(store)} arrays to {OUT} in {time.monotonic() - t0:.1f}s",
          file=sys.stderr)


if __name__ == "__main__":
    main()
