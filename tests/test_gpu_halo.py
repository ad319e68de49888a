"""Halo mirrors (SURVEY §8 e, solver.py:86-90 "the halo is filled before the
multiply"): the owner of a boundary row pushes each new value of the mirrored
Krylov vectors into the readers' halo mirrors while it computes it, and the
streaming CG / PCG / BiCGStab kernels read halo operands from their own
mirror.  A mirror only changes where an operand is loaded from, never its
value, so every iterate must be bit-identical to the direct-load data path
(LRB_HALO=direct: peer loads from the owning part) — on multi-part devices and
on split device ranks (the cross-device peer protocol on one GPU)."""

import numpy as np
import pytest

import paper_2510_08536_b200 as lrb
from helpers_b200 import cavity_case, golden_inputs

pytestmark = pytest.mark.gpu


def _parts(asm, pm, step=3):
    holder = {}

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        lrb.update(s, *lrb.perturb_coefficients(*asm[ctx.rank], step), "direct")
        parts = s.comm.allgather(s.part) if s.is_owner else None
        if s.is_owner and s.comm.group_rank == 0:
            holder["parts"] = parts
        return s

    systems = lrb.run_world(len(asm), program)
    return holder["parts"], systems


def _team(parts, dev_ranks, monkeypatch, halo):
    from paper_2510_08536_b200.device import Team
    if halo == "direct":
        monkeypatch.setenv("LRB_HALO", "direct")
    else:
        monkeypatch.delenv("LRB_HALO", raising=False)
    t = Team(parts, dev_ranks=dev_ranks)
    monkeypatch.delenv("LRB_HALO", raising=False)
    return t


def _solve(team, method, bs, tol=1e-10, max_iter=500):
    xs, rep, hist = team.solve(method, bs, tol, max_iter, hist_cap=max_iter)
    return xs, rep, hist


def _same(a, b):
    xa, ra, ha = a
    xb, rb, hb = b
    assert (ra.iterations, ra.converged, ra.status) == (rb.iterations, rb.converged, rb.status)
    assert ra.residual == rb.residual
    assert np.array_equal(ha, hb)
    for u, v in zip(xa, xb):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("dims,n_cpu,alpha,dev_ranks", [
    ((24, 24, 24), 8, 2, None),              # 4 parts, one kernel
    ((20, 20, 20), 4, 1, [0, 0, 1, 1]),      # two device ranks on one GPU (peer protocol)
    ((20, 20, 20), 4, 1, [0, 1, 2, 3]),
    ((30, 28, 26), 6, 2, [0, 1, 2]),         # uneven layers
])
def test_mirror_bit_identical_to_direct(dims, n_cpu, alpha, dev_ranks, monkeypatch):
    _, asm, pm = cavity_case(dims, n_cpu, alpha)
    parts, _ = _parts(asm, pm)
    mir = _team(parts, dev_ranks, monkeypatch, "mirror")
    dirc = _team(parts, dev_ranks, monkeypatch, "direct")
    info = mir.kernel_info("pcg")
    assert info["halo_mirrors"] == 1 and info["streaming"] == 1
    assert dirc.kernel_info("pcg")["halo_mirrors"] == 0
    # slab parts: one run per neighbour (the first / last plane)
    first_dev = [p for p, d in enumerate(dev_ranks or [0] * len(parts)) if d == 0]
    want = sum((p > 0) + (p < len(parts) - 1) for p in first_dev)
    assert info["push_runs"] == want
    rng = np.random.default_rng(11)
    for method in ("cg", "pcg", "bicgstab"):
        for bs in ([np.ones(p.n) for p in parts], [rng.standard_normal(p.n) for p in parts]):
            _same(_solve(mir, method, bs), _solve(dirc, method, bs))


def test_mirror_not_stale_across_solves(monkeypatch):
    """A second solve on the same team must not read mirror values left by the
    first one (every mirrored read is preceded by a push in the same solve)."""
    _, asm, pm = cavity_case((20, 20, 20), 4, 1)
    parts, _ = _parts(asm, pm)
    mir = _team(parts, [0, 1, 2, 3], monkeypatch, "mirror")
    rng = np.random.default_rng(5)
    b1 = [rng.standard_normal(p.n) for p in parts]
    b2 = [np.ones(p.n) for p in parts]
    _solve(mir, "bicgstab", b1)
    _solve(mir, "pcg", b1, max_iter=7)   # stopped early: mirrors hold mid-solve values
    fresh = _team(parts, [0, 1, 2, 3], monkeypatch, "direct")
    for method in ("pcg", "cg", "bicgstab"):
        _same(_solve(mir, method, b2), _solve(fresh, method, b2))


def test_mirror_matches_reference_cg_history(monkeypatch):
    """Through the drop-in API (the team repartition() builds): the CG history
    equals the direct path's bit for bit, and the mirrors are on."""
    _, asm, pm = cavity_case((16, 16, 16), 8, 2)
    parts, systems = _parts(asm, pm)
    s0 = systems[0]
    assert s0.team.kernel_info("cg")["halo_mirrors"] == 1
    res = {}

    def program(ctx):
        s = systems[ctx.rank]
        if s.is_owner:
            x, rep = lrb.cg_solve(s.matrix, s.halo, np.ones(s.matrix.n_owned), 1e-8, 500, s.comm,
                                  history=True)
            res[ctx.rank] = (x, rep)
        return None

    lrb.run_world(8, program)
    dirc = _team(parts, None, monkeypatch, "direct")
    xs, rep, hist = _solve(dirc, "cg", [np.ones(p.n) for p in parts], tol=1e-8)
    assert res[0][1].iterations == rep.iterations
    assert np.array_equal(np.asarray(res[0][1].history), hist)
    for k in range(len(parts)):
        assert np.array_equal(res[2 * k][0], xs[k])


@pytest.mark.parametrize("name", ["rand0", "rand7"])
def test_irregular_systems_either_path(name, monkeypatch):
    """Random partitioned systems: many short runs may switch mirrors off
    (kMaxSndRuns); either way the first iterations equal the direct path."""
    pm, per_rank = golden_inputs(name)
    holder = {}

    def program(ctx):
        s = lrb.repartition(*per_rank[ctx.rank], pm, ctx)
        ps = s.comm.allgather(s.part) if s.is_owner else None
        if s.is_owner and s.comm.group_rank == 0:
            holder["parts"] = ps
        return None

    lrb.run_world(len(per_rank), program)
    parts = holder["parts"]
    mir = _team(parts, None, monkeypatch, "mirror")
    dirc = _team(parts, None, monkeypatch, "direct")
    bs = [np.ones(p.n) for p in parts]
    for method in ("cg", "bicgstab"):
        try:
            a = _solve(mir, method, bs, 1e-30, 5)
        except ValueError as e:
            a = str(e)
        try:
            b = _solve(dirc, method, bs, 1e-30, 5)
        except ValueError as e:
            b = str(e)
        if isinstance(a, str) or isinstance(b, str):
            assert a == b
        else:
            _same(a, b)
