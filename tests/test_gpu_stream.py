"""The streaming (bulk-copy / mbarrier ring) solvers against the classic
per-thread-gather solvers: same tiles, same rounding, same reduction tree, so
every iterate must be bit-identical — on stencil parts (every tile staged),
multi-part devices, split device ranks (peer-flag protocol) and irregular
random systems (tiles computed by the consumers' direct-load fallback)."""

import os

import numpy as np
import pytest

import paper_2510_08536_b200 as lrb
from helpers_b200 import cavity_case, golden_inputs

pytestmark = pytest.mark.gpu


def _teams(parts, dev_ranks=None):
    from paper_2510_08536_b200.device import Team
    old = os.environ.get("LRB_SOLVER")
    try:
        os.environ["LRB_SOLVER"] = "classic"
        classic = Team(parts, dev_ranks=dev_ranks)
        os.environ.pop("LRB_SOLVER")
        stream = Team(parts, dev_ranks=dev_ranks)
    finally:
        if old is None:
            os.environ.pop("LRB_SOLVER", None)
        else:
            os.environ["LRB_SOLVER"] = old
    return classic, stream


def _compare(parts, methods, tol, max_iter, dev_ranks=None, rhs_seed=None, expect_stream=True):
    classic, stream = _teams(parts, dev_ranks)
    out = {}
    for method in methods:
        info = stream.kernel_info(method)
        assert info["streaming"] == int(expect_stream), info
        if expect_stream:
            assert info["block"] > 512 and info["block"] % 32 == 0 and info["stages"] >= 2
        assert classic.kernel_info(method)["streaming"] == 0
        if rhs_seed is None:
            bs = [np.ones(p.n) for p in parts]
        else:
            rng = np.random.default_rng(rhs_seed)
            bs = [rng.standard_normal(p.n) for p in parts]
        xa, ra, ha = classic.solve(method, bs, tol, max_iter, hist_cap=max_iter)
        xb, rb, hb = stream.solve(method, bs, tol, max_iter, hist_cap=max_iter)
        assert (ra.iterations, ra.converged, ra.status) == (rb.iterations, rb.converged, rb.status)
        assert ra.residual == rb.residual and ra.bnorm == rb.bnorm
        assert np.array_equal(ha, hb)
        for a, b in zip(xa, xb):
            assert np.array_equal(a, b)
        out[method] = rb
    return out


def _owner_parts(asm, pm):
    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        parts = s.comm.allgather(s.part)
        return parts if s.comm.group_rank == 0 else None

    return lrb.run_world(len(asm), program)


@pytest.mark.parametrize("dims,n_cpu,alpha", [((16, 16, 16), 2, 2), ((32, 32, 32), 4, 4),
                                              ((48, 40, 36), 3, 3), ((24, 24, 24), 8, 2),
                                              # many ring revolutions per CTA (every slot reused by
                                              # both consumer teams): 1954 / 1458 tiles on 148 SMs
                                              ((100, 100, 100), 4, 4), ((90, 90, 90), 6, 3)])
def test_stream_bit_identical_cavity(dims, n_cpu, alpha):
    _, asm, pm = cavity_case(dims, n_cpu, alpha)
    holder = {}

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        lrb.update(s, *lrb.perturb_coefficients(*asm[ctx.rank], 3), "direct")
        parts = s.comm.allgather(s.part) if s.is_owner else None
        if s.is_owner and s.comm.group_rank == 0:
            holder["r"] = _compare(parts, ("cg", "pcg"), 1e-9, 400)
            holder["r2"] = _compare(parts, ("pcg",), 1e-30, 23, rhs_seed=7)   # max_iter exit
        return None

    lrb.run_world(n_cpu, program)
    assert holder["r"]["cg"].converged and holder["r"]["pcg"].converged
    assert not holder["r2"]["pcg"].converged and holder["r2"]["pcg"].iterations == 23


def test_stream_bit_identical_split_devices():
    _, asm, pm = cavity_case((20, 20, 20), 4, 1)
    holder = {}

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        parts = s.comm.allgather(s.part)
        if s.comm.group_rank == 0:
            holder["a"] = _compare(parts, ("cg", "pcg"), 1e-9, 400, dev_ranks=[0, 0, 1, 1])
            holder["b"] = _compare(parts, ("pcg",), 1e-9, 400, dev_ranks=[0, 1, 2, 3])
        return None

    lrb.run_world(4, program)
    assert holder["a"]["cg"].converged and holder["b"]["pcg"].converged


@pytest.mark.parametrize("name", ["rand0", "rand7", "rand23"])
def test_stream_bit_identical_irregular(name):
    """Random systems: irregular slices fall back to direct loads per tile."""
    pm, per_rank = golden_inputs(name)
    parts = _owner_parts(per_rank, pm)[0]
    # the random values are not SPD in general: compare the first iterations
    classic, stream = _teams(parts)
    bs = [np.ones(p.n) for p in parts]
    for method in ("cg", "pcg"):
        try:
            xa, ra, ha = classic.solve(method, bs, 1e-30, 6, hist_cap=6)
            ea = None
        except ValueError as e:
            ea = str(e)
        try:
            xb, rb, hb = stream.solve(method, bs, 1e-30, 6, hist_cap=6)
            eb = None
        except ValueError as e:
            eb = str(e)
        assert ea == eb
        if ea is None:
            assert ra.iterations == rb.iterations and np.array_equal(ha, hb)
            for a, b in zip(xa, xb):
                assert np.array_equal(a, b)


def test_stream_solver_is_default_and_reports_geometry():
    _, asm, pm = cavity_case((32, 32, 32), 4, 4)
    parts = _owner_parts(asm, pm)[0]
    from paper_2510_08536_b200.device import Team
    info = Team(parts).kernel_info("pcg")
    assert info["streaming"] == 1 and info["block"] > 512
    assert info["grid"] >= 1 and info["stage_bytes"] % 128 == 0
    assert info["smem"] >= info["stages"] * info["stage_bytes"]


def _momentum(asm, seed=0):
    """Non-symmetric, diagonally dominant LDU on the cavity addressing."""
    rng = np.random.default_rng(seed)
    out = []
    for m, ifs in asm:
        eps_u = 0.05 * rng.random(m.n_faces)
        eps_l = 0.05 * rng.random(m.n_faces)
        mm = lrb.LduMatrix(m.n_cells, m.lower_addr, m.upper_addr, np.full(m.n_cells, 6.5),
                           -1.0 - eps_l, -1.0 + eps_u)
        out.append((mm, [lrb.InterfaceBlock(b.neighbor_rank, b.rows, b.cols_remote,
                                            b.values * (1.0 + 0.01 * b.neighbor_rank)) for b in ifs]))
    return out


@pytest.mark.parametrize("dims,n_cpu,alpha,dev_ranks", [((24, 24, 24), 4, 2, None),
                                                        ((20, 20, 20), 4, 1, [0, 0, 1, 1]),
                                                        ((100, 100, 100), 4, 4, None)])
def test_stream_bicgstab_bit_identical(dims, n_cpu, alpha, dev_ranks):
    _, asm, pm = cavity_case(dims, n_cpu, alpha)
    mom = _momentum(asm)
    holder = {}

    def program(ctx):
        s = lrb.repartition(*mom[ctx.rank], pm, ctx)
        parts = s.comm.allgather(s.part) if s.is_owner else None
        if s.is_owner and s.comm.group_rank == 0:
            holder["r"] = _compare(parts, ("bicgstab",), 1e-10, 300, dev_ranks=dev_ranks, rhs_seed=3)
        return None

    lrb.run_world(n_cpu, program)
    assert holder["r"]["bicgstab"].converged


@pytest.mark.parametrize("dims,n_cpu,alpha,dev_ranks", [((24, 24, 24), 4, 2, None),
                                                        ((20, 20, 20), 4, 1, [0, 0, 1, 1]),
                                                        ((100, 100, 100), 4, 4, None)])
def test_pcg1_matches_pcg(dims, n_cpu, alpha, dev_ranks):
    """Single-reduction PCG: CG's iterates in exact arithmetic, so the same
    iteration count (+-1) and residual history / solution to rounding."""
    from paper_2510_08536_b200.device import Team
    _, asm, pm = cavity_case(dims, n_cpu, alpha)
    holder = {}

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        lrb.update(s, *lrb.perturb_coefficients(*asm[ctx.rank], 3), "direct")
        parts = s.comm.allgather(s.part) if s.is_owner else None
        if s.is_owner and s.comm.group_rank == 0:
            team = Team(parts, dev_ranks=dev_ranks)
            assert team.kernel_info("pcg1")["streaming"] == 1
            bs = [np.ones(p.n) for p in parts]
            holder["pcg"] = team.solve("pcg", bs, 1e-9, 500, hist_cap=500)
            holder["pcg1"] = team.solve("pcg1", bs, 1e-9, 500, hist_cap=500)
            holder["pcg1b"] = team.solve("pcg1", bs, 1e-9, 500, hist_cap=500)
        return None

    lrb.run_world(n_cpu, program)
    (xa, ra, ha), (xb, rb, hb), (xc, rc, hc) = holder["pcg"], holder["pcg1"], holder["pcg1b"]
    assert ra.converged and rb.converged and abs(ra.iterations - rb.iterations) <= 1
    n = min(len(ha), len(hb))
    np.testing.assert_allclose(hb[:n], ha[:n], rtol=1e-6, atol=1e-14)
    xa, xb = np.concatenate(xa), np.concatenate(xb)
    assert np.linalg.norm(xb - xa) <= 1e-7 * np.linalg.norm(xa)
    # deterministic run to run
    assert rc.iterations == rb.iterations and np.array_equal(hc, hb)
    assert all(np.array_equal(a, b) for a, b in zip(xc, holder["pcg1"][0]))


@pytest.mark.parametrize("dims,n_cpu,alpha,dev_ranks", [((24, 24, 24), 4, 4, None),
                                                        ((24, 24, 24), 4, 2, None),
                                                        ((20, 20, 20), 4, 1, [0, 0, 1, 1]),
                                                        ((64, 64, 64), 4, 1, [0, 0, 1, 1]),
                                                        ((100, 100, 100), 4, 4, None)])
@pytest.mark.parametrize("defer", ["0", "1"])
def test_pipecg_matches_pcg(dims, n_cpu, alpha, dev_ranks, defer, monkeypatch):
    """Pipelined PCG: CG's iterates in exact arithmetic (same iterations +-1,
    history and solution to rounding); deterministic run to run on flat teams
    (deferred reductions) and on multi-part / split-device teams (reducing
    barrier).  defer "1": LRB_PIPE_DEFER=1 (reductions read one phase late
    on flat teams)."""
    from paper_2510_08536_b200.device import Team
    monkeypatch.setenv("LRB_PIPE_DEFER", defer)
    _, asm, pm = cavity_case(dims, n_cpu, alpha)
    holder = {}

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        lrb.update(s, *lrb.perturb_coefficients(*asm[ctx.rank], 3), "direct")
        parts = s.comm.allgather(s.part) if s.is_owner else None
        if s.is_owner and s.comm.group_rank == 0:
            team = Team(parts, dev_ranks=dev_ranks)
            assert team.kernel_info("pipecg")["streaming"] == 1
            bs = [np.ones(p.n) for p in parts]
            holder["pcg"] = team.solve("pcg", bs, 1e-9, 500, hist_cap=500)
            holder["pipe"] = team.solve("pipecg", bs, 1e-9, 500, hist_cap=500)
            holder["pipeb"] = team.solve("pipecg", bs, 1e-9, 500, hist_cap=500)
        return None

    lrb.run_world(n_cpu, program)
    (xa, ra, ha), (xb, rb, hb), (xc, rc, hc) = holder["pcg"], holder["pipe"], holder["pipeb"]
    assert ra.converged and rb.converged and abs(ra.iterations - rb.iterations) <= 1
    n = min(len(ha), len(hb))
    np.testing.assert_allclose(hb[:n], ha[:n], rtol=1e-6, atol=1e-14)
    xa, xb = np.concatenate(xa), np.concatenate(xb)
    assert np.linalg.norm(xb - xa) <= 1e-7 * np.linalg.norm(xa)
    assert rc.iterations == rb.iterations and np.array_equal(hc, hb)
    assert all(np.array_equal(a, b) for a, b in zip(xc, holder["pipe"][0]))


@pytest.mark.parametrize("stages", ["2", "3"])
def test_stream_ring_depth_variants(stages, monkeypatch):
    """Two- and three-stage rings (L = lcm(stages, 2) = 2 / 6 ring periods
    against 8 group-sum slots): the reducer hand-off, the lane tree and the
    stage bookkeeping stay bit-identical to the classic kernels."""
    monkeypatch.setenv("LRB_STREAM_STAGES", stages)
    _, asm, pm = cavity_case((80, 80, 80), 4, 4)
    holder = {}

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        lrb.update(s, *lrb.perturb_coefficients(*asm[ctx.rank], 4), "direct")
        parts = s.comm.allgather(s.part) if s.is_owner else None
        if s.is_owner and s.comm.group_rank == 0:
            from paper_2510_08536_b200.device import Team
            assert Team(parts).kernel_info("pcg")["stages"] == int(stages)
            holder["r"] = _compare(parts, ("cg", "pcg"), 1e-9, 400)
        return None

    lrb.run_world(4, program)
    assert holder["r"]["pcg"].converged


def test_teams_of_different_geometry_coexist():
    """Kernel launch attributes are per function and shared by every team: a
    team created later with smaller stages must not break an earlier team's
    launches (interleaved solves, each equal to a fresh team's result)."""
    from paper_2510_08536_b200.device import Team
    teams = []
    for dims, n_cpu, alpha in (((48, 44, 40), 2, 2), ((12, 12, 12), 4, 2), ((30, 30, 30), 3, 1)):
        _, asm, pm = cavity_case(dims, n_cpu, alpha)
        parts = _owner_parts(asm, pm)[0]
        teams.append((parts, Team(parts), Team(parts, dev_ranks=list(range(len(parts))))))
    ref = [t.solve("pcg", [np.ones(p.n) for p in parts], 1e-9, 500) for parts, t, _ in teams]
    for k in (0, 2, 1, 0):
        parts, team, split = teams[k]
        bs = [np.ones(p.n) for p in parts]
        for tm in (team, split):
            xs, rep, _ = tm.solve("pcg", bs, 1e-9, 500)
            assert rep.iterations == ref[k][1].iterations
            for a, b in zip(xs, ref[k][0]):
                assert np.array_equal(a, b)
