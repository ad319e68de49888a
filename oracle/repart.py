"""Oracle restatement of the repartitioner and update path.

Reference: repart.py (extract/fuse/scatter), update.py (pack/scatter),
solver.py:48-77 (halo plan), core.py:163-244 (partition map, LDU->COO).
World-free: an owner's inputs are simply the list of its sources' problems.
Test infrastructure only (see oracle/__init__.py).
"""

from typing import NamedTuple

import numpy as np

from .cavity import RankProblem


def _lex(rows, cols):
    return np.lexsort((cols, rows))


def gpu_range(offsets, alpha, k):
    """I_GPU(k) = [off[alpha k], off[alpha k + alpha]) (core.py:198-202)."""
    return int(offsets[alpha * k]), int(offsets[alpha * (k + 1)])


def cpu_owner(offsets, cols):
    """CPU rank owning each global column (core.py:204-206)."""
    return np.searchsorted(offsets, cols, side="right") - 1


class Extract(NamedTuple):
    """SparsityPattern equivalent (repart.py:26-39)."""
    lrows: np.ndarray
    lcols: np.ndarray
    nrows: np.ndarray
    ncols: np.ndarray
    lo: int
    hi: int


def extract(p: RankProblem, offsets, rank) -> Extract:
    """Global-index local + interface pattern (repart.py:143-174, core.py:237-244)."""
    lo, hi = int(offsets[rank]), int(offsets[rank + 1])
    if hi - lo != p.n:
        raise ValueError(f"rank {rank} holds {p.n} cells but owns {hi - lo}")
    cell = np.arange(p.n, dtype=np.int64)
    r = np.concatenate((cell, p.lower, p.upper))
    c = np.concatenate((cell, p.upper, p.lower))
    o = _lex(r, c)
    nr, nc = [], []
    for b in sorted(p.blocks, key=lambda b: b.nbr):
        if b.nbr == rank:
            raise ValueError(f"inconsistent interface: rank {rank} lists itself as neighbor")
        nlo, nhi = int(offsets[b.nbr]), int(offsets[b.nbr + 1])
        if len(b.rows) and (int(b.cols.max()) >= nhi - nlo or int(b.rows.max()) >= p.n):
            raise ValueError(f"inconsistent interface: entry of rank {rank} toward "
                             f"rank {b.nbr} is out of range")
        nr.append(b.rows + lo)
        nc.append(b.cols + nlo)
    if nr:
        nr, nc = np.concatenate(nr), np.concatenate(nc)
        o2 = _lex(nr, nc)
        nr, nc = nr[o2], nc[o2]
        key = nr * np.int64(offsets[-1]) + nc
        if len(key) > 1 and (np.diff(key) == 0).any():
            raise ValueError("inconsistent interface: duplicate coupling entry")
    else:
        nr = nc = np.zeros(0, np.int64)
    return Extract(r[o] + lo, c[o] + lo, nr, nc, lo, hi)


def fuse(exts, offsets, alpha, k):
    """Localize couplings inside I_GPU(k); sort; reject duplicates (repart.py:197-236)."""
    lo, hi = gpu_range(offsets, alpha, k)
    nr = np.concatenate([e.nrows for e in exts])
    nc = np.concatenate([e.ncols for e in exts])
    inside = (nc >= lo) & (nc < hi)
    total = np.int64(offsets[-1])

    def uniq(rows, cols, what):
        o = _lex(rows, cols)
        rows, cols = rows[o], cols[o]
        key = rows * total + cols
        dup = np.flatnonzero(np.diff(key) == 0)
        if len(dup):
            i = dup[0]
            raise ValueError(f"overlapping ownership: duplicate {what} entry "
                             f"({rows[i]}, {cols[i]})")
        return rows, cols

    loc = uniq(np.concatenate([e.lrows for e in exts] + [nr[inside]]),
               np.concatenate([e.lcols for e in exts] + [nc[inside]]), "local")
    nl = uniq(nr[~inside], nc[~inside], "non-local")
    return loc, nl


def pack_order(e: Extract, offsets):
    """(row, col) provenance of the packed buffer of one source (repart.py:253-270)."""
    d = e.lrows[e.lrows == e.lcols]
    up = e.lrows < e.lcols
    ur, uc = e.lrows[up], e.lcols[up]
    o = np.lexsort((e.ncols, e.nrows, cpu_owner(offsets, e.ncols)))
    return (np.concatenate((d, ur, uc, e.nrows[o])),
            np.concatenate((d, uc, ur, e.ncols[o])))


def scatter_map(exts, loc, nl, offsets):
    """Buffer position -> (to_local, slot) via key search (repart.py:273-304)."""
    total = np.int64(offsets[-1])
    pr, pc = zip(*(pack_order(e, offsets) for e in exts))
    keys = np.concatenate(pr) * total + np.concatenate(pc)
    lk = loc[0] * total + loc[1]
    nk = nl[0] * total + nl[1]

    def find(sorted_keys, q):
        if len(sorted_keys) == 0:
            return np.zeros(len(q), np.int64), np.zeros(len(q), bool)
        pos = np.searchsorted(sorted_keys, q)
        hit = (pos < len(sorted_keys)) & (sorted_keys[np.minimum(pos, len(sorted_keys) - 1)] == q)
        return pos, hit

    pl, hl = find(lk, keys)
    pn, hn = find(nk, keys)
    if not (hl | hn).all():
        raise RuntimeError("scatter map: buffer entry matches no fused pattern slot")
    return hl, np.where(hl, pl, pn)


class OwnerPart(NamedTuple):
    """One fused owner part: DistributedCooMatrix + ScatterMap + recv offsets."""
    k: int
    lo: int
    hi: int
    loc_rows: np.ndarray   # part-local row
    loc_cols: np.ndarray   # part-local col
    nl_rows: np.ndarray    # part-local row
    nl_cols: np.ndarray    # index into halo_cols
    halo_cols: np.ndarray  # global, ascending
    g_loc: tuple           # global (rows, cols) local pattern
    g_nl: tuple            # global (rows, cols) non-local pattern
    to_local: np.ndarray
    index: np.ndarray
    recv_offsets: np.ndarray


def build_owner(problems, offsets, alpha, k) -> OwnerPart:
    """Create-once path of owner k (repart.py:321-354 without the world)."""
    srcs = range(alpha * k, alpha * (k + 1))
    exts = [extract(problems[r], offsets, r) for r in srcs]
    loc, nl = fuse(exts, offsets, alpha, k)
    to_local, index = scatter_map(exts, loc, nl, offsets)
    lo, hi = gpu_range(offsets, alpha, k)
    halo = np.unique(nl[1])
    counts = [len(e.lrows) + len(e.nrows) for e in exts]
    return OwnerPart(k, lo, hi, loc[0] - lo, loc[1] - lo, nl[0] - lo,
                     np.searchsorted(halo, nl[1]), halo, loc, nl, to_local, index,
                     np.concatenate(([0], np.cumsum(counts))).astype(np.int64))


def halo_plan(parts, offsets, alpha):
    """Per owner: send_indices / recv_slots dicts (solver.py:48-77)."""
    owners = [cpu_owner(offsets, p.halo_cols) // alpha for p in parts]
    plans = []
    for g, p in enumerate(parts):
        recv = {int(j): np.flatnonzero(owners[g] == j) for j in np.unique(owners[g])}
        send = {}
        for h, q in enumerate(parts):
            if h == g:
                continue
            want = q.halo_cols[owners[h] == g]
            if len(want):
                send[h] = want - p.lo
        plans.append((send, recv))
    return plans


def pack(p: RankProblem):
    """[diag | upper | lower | interface values by neighbour] (update.py:40-45)."""
    blocks = sorted(p.blocks, key=lambda b: b.nbr)
    return np.concatenate([p.diag, p.uval, p.lval] + [b.vals for b in blocks])


def scatter_values(part: OwnerPart, buf):
    """local.vals[index[m]] = buf[m]; non-local likewise (update.py:105-112)."""
    if len(buf) != len(part.index):
        raise ValueError(f"scatter length mismatch: buffer {len(buf)}, map {len(part.index)}")
    lv = np.zeros(len(part.loc_rows))
    nv = np.zeros(len(part.nl_rows))
    m = part.to_local
    lv[part.index[m]] = buf[m]
    nv[part.index[~m]] = buf[~m]
    return lv, nv


def owner_buffer(problems, alpha, k):
    """Owner k's receive buffer: sources' packs in ascending rank (update.py:48-102)."""
    return np.concatenate([pack(problems[r]) for r in range(alpha * k, alpha * (k + 1))])
