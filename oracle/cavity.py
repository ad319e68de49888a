"""Oracle restatement of the model-problem generator (reference assembly.py).

A rank's problem is returned as a plain ``RankProblem`` tuple instead of the
reference's dataclasses.  Test infrastructure only (see oracle/__init__.py).
"""

from typing import NamedTuple

import numpy as np


class Block(NamedTuple):
    """Interface block: couplings of local rows to one neighbour rank."""
    nbr: int
    rows: np.ndarray      # local rows, int64
    cols: np.ndarray      # neighbour-local cells, int64
    vals: np.ndarray      # float64


class RankProblem(NamedTuple):
    """One CPU rank's LDU matrix plus interface blocks (core.py:50-112)."""
    n: int
    lower: np.ndarray
    upper: np.ndarray
    diag: np.ndarray
    lval: np.ndarray
    uval: np.ndarray
    blocks: tuple


def axis_order(dims):
    """Fastest→slowest axes; slab axis = longest, ties toward z (assembly.py:48-61)."""
    slow = 0
    for ax in (1, 2):
        if dims[ax] >= dims[slow]:
            slow = ax
    fast = [ax for ax in (0, 1, 2) if ax != slow]
    return fast[0], fast[1], slow


def slab_ranges(n_layers, n_parts):
    """Balanced contiguous layer ranges, extra layers first (assembly.py:108-117)."""
    q, rem = divmod(n_layers, n_parts)
    sizes = [q + (i < rem) for i in range(n_parts)]
    ends = np.cumsum([0] + sizes)
    return [(int(ends[i]), int(ends[i + 1])) for i in range(n_parts)]


def cavity_problems(dims, n_parts):
    """Slab decomposition + unit 7-point Laplacian per part.

    Follows decompose_slab (assembly.py:120-192) and assemble_poisson
    (assembly.py:195-222): faces strictly sorted by (lower, upper); diag =
    internal + interface + boundary face count; every coupling -1.
    """
    a0, a1, a2 = axis_order(dims)
    d0, d1, d2 = dims[a0], dims[a1], dims[a2]
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    if n_parts > d2:
        raise ValueError(f"too many parts: {n_parts} slabs along an axis of {d2} cells")
    plane = d0 * d1
    ranges = slab_ranges(d2, n_parts)
    out = []
    for r, (z0, z1) in enumerate(ranges):
        nz = z1 - z0
        n = plane * nz
        cell = np.arange(n, dtype=np.int64)
        ix, iy, iz = cell % d0, (cell // d0) % d1, cell // plane
        pairs = []
        if d0 > 1:
            c = cell[ix < d0 - 1]
            pairs.append(np.column_stack((c, c + 1)))
        if d1 > 1:
            c = cell[iy < d1 - 1]
            pairs.append(np.column_stack((c, c + d0)))
        if nz > 1:
            c = cell[iz < nz - 1]
            pairs.append(np.column_stack((c, c + plane)))
        faces = np.concatenate(pairs) if pairs else np.zeros((0, 2), np.int64)
        faces = faces[np.lexsort((faces[:, 1], faces[:, 0]))]
        count = np.zeros(n, dtype=np.int64)
        if d0 > 1:
            count += (ix == 0).astype(np.int64) + (ix == d0 - 1)
        if d1 > 1:
            count += (iy == 0).astype(np.int64) + (iy == d1 - 1)
        if d2 > 1:
            count += ((iz + z0) == 0).astype(np.int64) + ((iz + z0) == d2 - 1)
        np.add.at(count, faces[:, 0], 1)
        np.add.at(count, faces[:, 1], 1)
        blocks = []
        fp = np.arange(plane, dtype=np.int64)
        if z0 > 0:
            prev_nz = ranges[r - 1][1] - ranges[r - 1][0]
            blocks.append(Block(r - 1, fp.copy(), fp + plane * (prev_nz - 1),
                                -np.ones(plane)))
        if z1 < d2:
            blocks.append(Block(r + 1, fp + plane * (nz - 1), fp.copy(), -np.ones(plane)))
        for b in blocks:
            np.add.at(count, b.rows, 1)
        nf = len(faces)
        out.append(RankProblem(n, faces[:, 0].copy(), faces[:, 1].copy(),
                               count.astype(np.float64), -np.ones(nf), -np.ones(nf),
                               tuple(blocks)))
    return out


def perturb(p: RankProblem, step: int) -> RankProblem:
    """diag * (1 + step/100), everything else untouched (assembly.py:225-243)."""
    if step < 1:
        raise ValueError(f"step must be >= 1, got {step}")
    return p._replace(diag=p.diag * (1.0 + step / 100.0))
