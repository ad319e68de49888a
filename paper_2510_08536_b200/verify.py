"""Verification helpers at scale: gather the owners' fused
parts into one global COO (reference oracle.py:23-43) and export measured
timings as the reference cost model's curves CSV (costmodel.py:227-255).

These sit beside the hot path: `gather_global` reads the parts' values back
from the device (one D2H copy per part) and is meant for checks and Matrix
Market export, not for the per-timestep loop.
"""
import csv

import numpy as np

from .core import CooMatrix, PartitionMap, coo_from_entries


def gather_global(matrix, pm: PartitionMap, comm):
    """Collect the owners' parts into one global COO on group rank 0.

    Collective over the active group (every owner passes its own part);
    non-root ranks return None.  Duplicate global entries mean two parts
    claimed the same (row, col): ValueError("overlap between gathered parts").
    """
    rows, cols, vals = matrix.global_entries()
    pieces = comm.gather((np.asarray(rows), np.asarray(cols), np.asarray(vals)), 0)
    if pieces is None:
        return None
    n = pm.total_cells
    try:
        return coo_from_entries(n, n, np.concatenate([p[0] for p in pieces]),
                                np.concatenate([p[1] for p in pieces]),
                                np.concatenate([p[2] for p in pieces]))
    except ValueError as exc:
        raise ValueError(f"overlap between gathered parts: {exc}") from exc


def write_curves_csv(path, rows) -> None:
    """Measured timings as the cost model's tabulated curves: columns n
    (ranks), t_as (assembly + coefficient update, s), t_ls (linear solve, s);
    sorted by n, one row per n, n = 1 required, timings positive — the
    contract of the reference's load_curves_csv."""
    rows = sorted((int(n), float(a), float(s)) for n, a, s in rows)
    ns = [r[0] for r in rows]
    if not rows or ns[0] != 1:
        raise ValueError("curves need a row for n = 1")
    if len(set(ns)) != len(ns):
        raise ValueError("curves need one row per n")
    if any(a <= 0 or s <= 0 for _, a, s in rows):
        raise ValueError("curve timings must be positive")
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(["n", "t_as", "t_ls"])
        for n, a, s in rows:
            w.writerow([n, repr(a), repr(s)])


def read_curves_csv(path):
    """(n, t_as, t_ls) arrays from a curves CSV (validated like the reference)."""
    ns, t_as, t_ls = [], [], []
    with open(path, newline="", encoding="utf-8") as fh:
        reader = csv.DictReader(fh)
        need = {"n", "t_as", "t_ls"}
        if reader.fieldnames is None or not need.issubset(reader.fieldnames):
            raise ValueError(f"curves CSV needs columns {sorted(need)}, got {reader.fieldnames}")
        for row in reader:
            ns.append(int(row["n"]))
            t_as.append(float(row["t_as"]))
            t_ls.append(float(row["t_ls"]))
    if not ns:
        raise ValueError("curves CSV has no data rows")
    o = np.argsort(ns)
    return np.asarray(ns)[o], np.asarray(t_as)[o], np.asarray(t_ls)[o]
