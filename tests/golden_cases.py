"""Access to tests/golden/golden.npz (made by tests/golden/make_golden.py from the
reference itself) and reconstruction of each case's inputs."""

import hashlib
import os
import re
from functools import lru_cache

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")


@lru_cache(maxsize=1)
def golden():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + a.tobytes()).hexdigest()


def case_names():
    return sorted({k.split("__")[0] for k in golden() if k.endswith("__meta")})


def case_meta(name):
    n_cpu, alpha, n_gpu, total = (int(v) for v in golden()[f"{name}__meta"])
    return n_cpu, alpha, n_gpu, total


def case_dims(name):
    """Grid dims of a cavity case, or None for random systems."""
    if name.startswith("chain"):
        return (8, 1, 1)
    if name == "c1":
        return (32, 32, 32)
    if name == "c2":
        return (100, 100, 100)
    m = re.match(r"cav(\d+)x(\d+)x(\d+)_r", name)
    if m:
        return tuple(int(v) for v in m.groups())
    m = re.match(r"cav(\d+)_r", name)
    if m:
        n = int(m.group(1))
        return (n, n, n)
    return None


def get(name, k, key):
    return golden().get(f"{name}__k{k}__{key}")


def matches(name, k, key, value) -> bool:
    """Exact comparison against the full array or its sha256 digest."""
    g = golden()
    value = np.asarray(value)
    full = g.get(f"{name}__k{k}__{key}")
    if full is not None:
        return (value.shape == full.shape and value.dtype.kind == full.dtype.kind
                and np.array_equal(value, full))
    dig = g.get(f"{name}__k{k}__{key}__sha256")
    if dig is None:
        raise KeyError(f"{name} k{k} {key} not in golden")
    # digests were taken on the reference's dtypes: int64 indices, bool masks, f64 values
    canon = {"i": np.int64, "u": np.int64, "b": np.bool_, "f": np.float64}[value.dtype.kind]
    return digest(value.astype(canon)) == str(dig)


def random_inputs(name):
    """(cells per rank, alpha, per-rank raw arrays) of a stored random system."""
    g = golden()
    cells = g[f"{name}__in_cells"]
    alpha = int(g[f"{name}__in_alpha"])
    ranks = []
    for r in range(len(cells)):
        p = f"{name}__in_r{r}"
        blen = g[f"{p}__blen"]
        cut = np.concatenate(([0], np.cumsum(blen))).astype(np.int64)
        blocks = [(int(nb), g[f"{p}__irow"][cut[i]:cut[i + 1]],
                   g[f"{p}__icol"][cut[i]:cut[i + 1]], g[f"{p}__ival"][cut[i]:cut[i + 1]])
                  for i, nb in enumerate(g[f"{p}__nbr"])]
        ranks.append(dict(n=int(cells[r]), lower=g[f"{p}__lower"], upper=g[f"{p}__upper"],
                          diag=g[f"{p}__diag"], lval=g[f"{p}__lval"], uval=g[f"{p}__uval"],
                          blocks=blocks))
    return cells, alpha, ranks


def case_config(name):
    """Mirror of the run_case arguments in tests/golden/make_golden.py."""
    if name.startswith("chain"):
        return dict(spmv_seed=3, steps=(3,), solve_steps=(1,), tol=1e-10, max_iter=100)
    if name.startswith("cav20_"):
        return dict(spmv_seed=None, steps=(), solve_steps=(1,), tol=1e-8, max_iter=1000)
    if name.startswith("cav"):
        return dict(spmv_seed=5, steps=(2, 3, 20), solve_steps=(1, 2, 3), tol=1e-6,
                    max_iter=2000)
    if name == "c1":
        return dict(spmv_seed=None, steps=(2,), solve_steps=(2, 3, 4), tol=1e-6,
                    max_iter=2000)
    if name == "c2":
        return dict(spmv_seed=None, steps=(2,), solve_steps=(2, 3), tol=1e-6, max_iter=2000)
    if name.startswith("rand"):
        return dict(spmv_seed=100 + int(name[4:]), steps=(), solve_steps=(), tol=1e-6,
                    max_iter=2000)
    raise KeyError(name)


def spmv_inputs(name, total):
    seed = case_config(name)["spmv_seed"]
    if seed is None:
        return None
    return np.random.default_rng(seed).normal(size=(3, total))


HIST_RTOL = 1e-10


def ref_history(log, iterations, tol):
    """sqrt(rr)/|b| per iteration from the reference's allreduce log
    ``[b.b, (p.q, r.r, [|b-Ax|^2 when rec<=tol or it%10==0])...]``."""
    bb = log[0]
    out, i = [], 1
    for it in range(1, iterations + 1):
        rec = np.sqrt(log[i + 1]) / np.sqrt(bb)
        out.append(rec)
        i += 2
        if rec <= tol or it % 10 == 0:
            i += 1
    return np.array(out)


def history_ok(ours, ref, rtol=HIST_RTOL, floor=1e-12):
    """Recurrence residuals within rtol relative; below the rounding floor
    (tiny systems reach exact convergence, e.g. the 8-cell chain) both must
    simply be negligible."""
    n = min(len(ours), len(ref))
    a, r = np.asarray(ours[:n]), np.asarray(ref[:n])
    ok = (np.abs(a - r) <= rtol * r) | ((r < floor) & (a < floor))
    return bool(ok.all()), n


LARGE_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@lru_cache(maxsize=None)
def large(name):
    """tests/golden/golden_large_<name>.npz (tests/golden/make_golden_large.py)."""
    with np.load(os.path.join(LARGE_DIR, f"golden_large_{name}.npz")) as z:
        return {k: z[k] for k in z.files}
