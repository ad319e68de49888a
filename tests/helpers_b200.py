"""Shared builders for the product tests (mirrors the reference tests/helpers.py)."""

import numpy as np

import paper_2510_08536_b200 as lrb
from golden_cases import case_dims, case_meta, random_inputs


def cavity_case(dims, n_cpu, alpha):
    grid = lrb.StructuredGrid(*dims)
    parts = lrb.decompose_slab(grid, n_cpu)
    assembled = [lrb.assemble_poisson(p) for p in parts]
    pm = lrb.make_partition_map([p.n_cells for p in parts], alpha)
    return grid, assembled, pm


def chain_setup(n_ranks=4, n_cells=8, alpha=None):
    grid = lrb.StructuredGrid(n_cells, 1, 1)
    parts = lrb.decompose_slab(grid, n_ranks)
    assembled = [lrb.assemble_poisson(p) for p in parts]
    pm = None if alpha is None else lrb.make_partition_map([p.n_cells for p in parts], alpha)
    return grid, parts, assembled, pm


def golden_inputs(name):
    """(pm, per-rank (LduMatrix, [InterfaceBlock])) for a golden case."""
    dims = case_dims(name)
    n_cpu, alpha, _, _ = case_meta(name)
    if dims is not None:
        _, assembled, pm = cavity_case(dims, n_cpu, alpha)
        return pm, assembled
    cells, alpha, raw = random_inputs(name)
    pm = lrb.make_partition_map(cells, alpha)
    per_rank = []
    for r in raw:
        m = lrb.LduMatrix(r["n"], r["lower"], r["upper"], r["diag"], r["lval"], r["uval"])
        ifs = [lrb.InterfaceBlock(nb, rows, cols, vals) for nb, rows, cols, vals in r["blocks"]]
        per_rank.append((m, ifs))
    return pm, per_rank


def owner_plan(pm, per_rank, k):
    from paper_2510_08536_b200.repart import _Source, _owner_plan
    srcs = [_Source(*per_rank[r], pm, r) for r in range(pm.alpha * k, pm.alpha * (k + 1))]
    return _owner_plan(srcs, pm, k)


def owner_buffer(per_rank, pm, k):
    return np.concatenate([lrb.pack_coefficients(*per_rank[r], r).values
                           for r in range(pm.alpha * k, pm.alpha * (k + 1))])


def sell_spmv(plan, vals_sell, x_local, x_halo):
    """Numpy emulation of the device SpMV over the SELL layout (row-sequential, no FMA)."""
    sp, col, src, dpos = plan.sell()
    n = plan.n
    y = np.zeros(n)
    xe = np.concatenate((x_local, x_halo))
    for s in range(plan.n_slices):
        w = (sp[s + 1] - sp[s]) // 32
        rows = np.arange(32 * s, min(n, 32 * s + 32))
        lanes = rows - 32 * s
        acc = np.zeros(len(rows))
        for k in range(w):
            e = sp[s] + 32 * k + lanes
            c = col[e]
            live = c >= 0
            prod = np.where(live, vals_sell[e] * xe[np.where(live, c, 0)], 0.0)
            acc = np.where(live, acc + prod, acc)
        y[rows] = acc
    return y


_PINNED = []


def pinned_ldu(m, ifs):
    """(LduMatrix, [InterfaceBlock], diag) whose value arrays live in pinned host
    memory, as bench.py's producer builds them (the zero-copy update branch)."""
    import torch

    def pin(a):
        t = torch.empty(len(a), dtype=torch.float64, pin_memory=True)
        _PINNED.append(t)
        out = t.numpy()
        out[:] = a
        return out

    diag = pin(m.diag)
    mm = lrb.LduMatrix(m.n_cells, m.lower_addr, m.upper_addr, diag, pin(m.lower_val),
                       pin(m.upper_val))
    ifp = [lrb.InterfaceBlock(b.neighbor_rank, b.rows, b.cols_remote, pin(b.values)) for b in ifs]
    return mm, ifp, diag


def momentum_ldu(asm, seed=0):
    """Non-symmetric, diagonally dominant LDU on the cavity addressing:
    upper -1+eps, lower -1-eps, eps in [0, 0.05), diag 6.5."""
    rng = np.random.default_rng(seed)
    out = []
    for m, ifs in asm:
        eps_u = 0.05 * rng.random(m.n_faces)
        eps_l = 0.05 * rng.random(m.n_faces)
        mm = lrb.LduMatrix(m.n_cells, m.lower_addr, m.upper_addr, np.full(m.n_cells, 6.5),
                           -1.0 - eps_l, -1.0 + eps_u)
        out.append((mm, ifs))
    return out


def oracle_problems(per_rank):
    """The same per-rank LDU inputs as oracle RankProblems."""
    from oracle import cavity as ocav
    return [ocav.RankProblem(m.n_cells, m.lower_addr, m.upper_addr, m.diag, m.lower_val,
                             m.upper_val, tuple(ocav.Block(b.neighbor_rank, b.rows, b.cols_remote,
                                                           b.values) for b in ifs))
            for m, ifs in per_rank]
