"""Distributed SpMV and Krylov solves on the repartitioned system.

Drop-in for the reference's solver.py (HaloPlan, build_halo_plan, spmv,
cg_solve, SolveReport).  A call is collective over the active group C_a;
group rank 0 drives one native team operation covering every owner part:
parts on the same GPU share one persistent kernel, the halo is read straight
from the neighbour part's vector (peer memory across GPUs) and the dot
products are reduced in ascending GPU rank like the reference's allreduce.
"""

import time
from dataclasses import dataclass, field

import numpy as np

from .transport import CommGroup

METHODS = ("cg", "pcg", "bicgstab", "pcg1", "pipecg")


@dataclass(frozen=True)
class HaloPlan:
    """send_indices[j]: my rows GPU j needs; recv_slots[j]: halo slots j fills (solver.py:19-37)."""

    send_indices: dict
    recv_slots: dict

    @property
    def send_neighbors(self):
        return tuple(sorted(self.send_indices))

    @property
    def recv_neighbors(self):
        return tuple(sorted(self.recv_slots))


@dataclass
class SolveReport:
    iterations: int
    residual: float
    converged: bool
    t_solve: float
    method: str = "cg"
    device_ms: float = 0.0
    history: np.ndarray = field(default=None, repr=False)   # recurrence residual per iteration
    breakdown: bool = False


def build_halo_plan(matrix, pm, comm: CommGroup) -> HaloPlan:
    """Exchange plan from every owner's halo columns; collective over C_a (solver.py:48-77)."""
    halo = matrix.halo_cols
    if len(halo) and (halo.min() < 0 or halo.max() >= pm.total_cells):
        raise ValueError("halo column owned by no rank")
    owners = pm.col_owner_gpu(halo)
    me = comm.group_rank
    if (owners == me).any():
        raise ValueError("halo plan: halo column inside own row range")
    wanted = [(int(j), halo[owners == j]) for j in np.unique(owners)]
    everyone = comm.allgather(wanted)
    recv = {j: np.flatnonzero(owners == j) for j, _ in wanted}
    send = {}
    for g, reqs in enumerate(everyone):
        if g == me:
            continue
        for j, cols in reqs:
            if j == me:
                send[g] = np.asarray(cols, dtype=np.int64) - matrix.row_offset
    return HaloPlan(send_indices=send, recv_slots=recv)


def _team_of(matrix):
    team = getattr(matrix, "_team", None)
    if team is None:
        raise TypeError("matrix is not device-backed: create it with repartition()")
    return team


def spmv(matrix, plan: HaloPlan, x, comm: CommGroup) -> np.ndarray:
    """y = A_local x + A_nonlocal x_halo on the GPUs (solver.py:80-97).

    Bit-identical to the reference: per row, local entries in stored order then
    non-local entries, each product rounded then accumulated (no FMA).
    """
    if len(x) != matrix.n_owned:
        raise ValueError(f"spmv dimension mismatch: x has {len(x)} entries, "
                         f"matrix owns {matrix.n_owned} rows")
    team = _team_of(matrix)
    return comm.leader_call(np.ascontiguousarray(x, dtype=np.float64),
                            lambda xs: team.spmv(xs))


def krylov_solve(matrix, plan: HaloPlan, b, tol: float, max_iter: int, comm: CommGroup,
                 method: str = "cg", history: bool = False):
    """Shared driver of cg_solve / pcg_solve / bicgstab_solve; returns (x, SolveReport)."""
    if method not in METHODS:
        raise ValueError(f"unknown method {method!r}")
    if tol <= 0:
        raise ValueError("tol must be positive")
    if len(b) != matrix.n_owned:
        raise ValueError("right-hand side length must match owned row count")
    team = _team_of(matrix)
    t0 = time.monotonic()
    cap = int(max_iter) if history else 0

    def run(bs):
        xs, rep, hist = team.solve(method, bs, tol, max_iter, want_x=True, hist_cap=cap)
        shared = (int(rep.iterations), float(rep.residual), bool(rep.converged),
                  float(rep.device_ms), bool(rep.breakdown), hist if history else None)
        return [(x, shared) for x in xs]

    x, (it, res, conv, dms, brk, hist) = comm.leader_call(
        np.ascontiguousarray(b, dtype=np.float64), run)
    return x, SolveReport(it, res, conv, time.monotonic() - t0, method, dms, hist, brk)


def cg_solve(matrix, plan: HaloPlan, b, tol: float, max_iter: int, comm: CommGroup,
             method: str = "cg", history: bool = False):
    """Distributed CG (solver.py:100-147): x0 = 0, true residual every 10
    iterations or when the recurrence residual meets tol, converged only on
    the true residual, max_iter reports instead of raising.  method="pcg"
    selects Jacobi-PCG (pressure), "bicgstab" BiCGStab (momentum), "pcg1" the
    single-reduction (Chronopoulos-Gear) Jacobi-PCG: one team barrier per
    iteration, CG's iterates up to rounding; "pipecg" the
    pipelined (Ghysels-Vanroose) Jacobi-PCG: one barrier per iteration that
    only waits for the arrivals, the reduction completes behind the next
    SpMV (§8 f1)."""
    return krylov_solve(matrix, plan, b, tol, max_iter, comm, method, history)


def pcg_solve(matrix, plan, b, tol, max_iter, comm, history=False):
    return krylov_solve(matrix, plan, b, tol, max_iter, comm, "pcg", history)


def bicgstab_solve(matrix, plan, b, tol, max_iter, comm, history=False):
    return krylov_solve(matrix, plan, b, tol, max_iter, comm, "bicgstab", history)
