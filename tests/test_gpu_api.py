"""The reference's own hot-path tests (tests/test_repart.py, test_update.py,
test_solver.py, test_acceptance.py 4-6) ported to the drop-in, plus BiCGStab
against the oracle and the cross-device team protocol on one GPU."""

import numpy as np
import pytest

import paper_2510_08536_b200 as lrb
from helpers_b200 import cavity_case, chain_setup
from oracle import cavity as ocav
from oracle.pipeline import OraclePipeline

pytestmark = pytest.mark.gpu


@pytest.fixture
def chain():
    grid, parts, assembled, _ = chain_setup(4)
    pm = lrb.make_partition_map([p.n_cells for p in parts], 2)
    return grid, parts, assembled, pm


def test_chain_alpha2_values(chain):
    _, _, asm, pm = chain

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        if s.is_owner:
            return s.matrix.local.vals.tolist(), s.matrix.non_local.vals.tolist()

    res = lrb.run_world(4, program)
    assert res[0] == ([2, -1, -1, 2, -1, -1, 2, -1, -1, 2], [-1])
    assert res[2] == ([2, -1, -1, 2, -1, -1, 2, -1, -1, 2], [-1])


def test_inactive_ranks_never_allocate(chain):
    _, _, asm, pm = chain
    world = lrb.World(4)
    world.run(lambda ctx: lrb.repartition(*asm[ctx.rank], pm, ctx) and None)
    assert world.device_allocations == [1, 0, 1, 0]


def test_device_buffer_and_apply_scatter(chain):
    _, _, asm, pm = chain

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        if s.is_owner:
            buf = s.device.values()
            s.device.fill(0, np.zeros(len(s.device)))
            lrb.apply_scatter(s.device, s.scatter, s.matrix)
            zero = (s.matrix.local.vals.tolist(), s.matrix.non_local.vals.tolist())
            s.device.fill(0, buf)
            lrb.apply_scatter(s.device, s.scatter, s.matrix)
            return buf.tolist(), zero, s.matrix.local.vals.tolist()

    res = lrb.run_world(4, program)
    assert res[0][0] == [2, 2, -1, -1, -1, 2, 2, -1, -1, -1, -1]
    assert res[0][1] == ([0.0] * 10, [0.0])
    assert res[0][2] == [2, -1, -1, 2, -1, -1, 2, -1, -1, 2]


def test_update_twenty_steps_match_fresh_repartition():
    _, asm, pm = cavity_case((6, 6, 6), 4, 2)

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        ok = True
        for step in range(1, 21):
            ms, ifs = lrb.perturb_coefficients(*asm[ctx.rank], step)
            lrb.update(s, ms, ifs, "direct" if step % 2 else "staged")
            fresh = lrb.repartition(ms, ifs, pm, ctx)
            if s.is_owner:
                ok &= np.array_equal(s.matrix.local.vals, fresh.matrix.local.vals)
                ok &= np.array_equal(s.matrix.non_local.vals, fresh.matrix.non_local.vals)
        return ok

    assert all(lrb.run_world(4, program))


@pytest.mark.parametrize("alpha", [2, 4])
def test_transfer_counts_direct_vs_staged(alpha):
    _, asm, pm = cavity_case((12, 12, 12), 8, alpha)

    def program(ctx):
        d = lrb.repartition(*asm[ctx.rank], pm, ctx)
        st = lrb.repartition(*asm[ctx.rank], pm, ctx)
        for step in (2, 3):
            ms, ifs = lrb.perturb_coefficients(*asm[ctx.rank], step)
            bd = d.device.transfer_count if d.is_owner else 0
            lrb.update(d, ms, ifs, "direct")
            bs = st.device.transfer_count if st.is_owner else 0
            lrb.update(st, ms, ifs, "staged")
            if d.is_owner:
                assert d.device.transfer_count - bd == pm.alpha
                assert st.device.transfer_count - bs == 1
                assert np.array_equal(d.matrix.local.vals, st.matrix.local.vals)
                assert np.array_equal(d.matrix.non_local.vals, st.matrix.non_local.vals)
        return True

    assert all(lrb.run_world(8, program))


def test_pattern_drift_detected(chain):
    _, _, asm, pm = chain

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        m, _ = asm[ctx.rank]
        lrb.update(s, lrb.LduMatrix(m.n_cells, [], [], m.diag, [], []), [], "direct")

    with pytest.raises(lrb.RankFailedError) as err:
        lrb.run_world(4, program)
    assert isinstance(err.value.cause, lrb.PatternDriftError)
    assert "pattern drift" in str(err.value.cause)


def test_pattern_arrays_never_rewritten(chain):
    _, _, asm, pm = chain

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        before = s.matrix.local.rows if s.is_owner else None
        ms, ifs = lrb.perturb_coefficients(*asm[ctx.rank], 2)
        lrb.update(s, ms, ifs, "direct")
        if s.is_owner:
            assert s.matrix.local.rows is before
            assert not s.matrix.local.rows.flags.writeable
        return True

    assert all(lrb.run_world(4, program))


def test_unknown_mode_and_length_violation(chain):
    _, _, asm, pm = chain

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        with pytest.raises(ValueError, match="mode"):
            lrb.update(s, *asm[ctx.rank], "bogus")
        return True

    assert all(lrb.run_world(4, program))


def test_spmv_row_sums_and_dimension_mismatch():
    _, _, asm, pm = chain_setup(4, alpha=2)

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        if s.is_owner:
            y = lrb.spmv(s.matrix, s.halo, np.ones(s.matrix.n_owned), s.comm)
            z = lrb.spmv(s.matrix, s.halo, np.zeros(s.matrix.n_owned), s.comm)
            return y.tolist(), z.tolist()

    res = lrb.run_world(4, program)
    assert res[0] == ([1, 0, 0, 0], [0, 0, 0, 0]) and res[2] == ([0, 0, 0, 1], [0, 0, 0, 0])

    def bad(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        if s.is_owner:
            lrb.spmv(s.matrix, s.halo, np.zeros(3), s.comm)

    with pytest.raises(lrb.RankFailedError, match="rank"):
        lrb.run_world(4, bad)


def solve_case(dims, n_cpu, alpha, tol=1e-10, b_value=1.0, max_iter=500, method="cg", step=None):
    _, asm, pm = cavity_case(dims, n_cpu, alpha)

    def program(ctx):
        m, ifs = asm[ctx.rank]
        s = lrb.repartition(m, ifs, pm, ctx)
        if step:
            lrb.update(s, *lrb.perturb_coefficients(m, ifs, step), "direct")
        if not s.is_owner:
            return None
        b = np.full(s.matrix.n_owned, b_value)
        x, rep = lrb.cg_solve(s.matrix, s.halo, b, tol, max_iter, s.comm, method=method,
                              history=True)
        pieces = s.comm.gather(x, 0)
        return (np.concatenate(pieces), rep) if pieces is not None else rep

    return lrb.run_world(n_cpu, program)[0]


@pytest.mark.parametrize("alpha", [1, 2, 4, 8])
def test_chain8_cg_solution(alpha):
    x, rep = solve_case((8, 1, 1), 8, alpha)
    np.testing.assert_allclose(x, [4, 7, 9, 10, 10, 9, 7, 4], atol=1e-10)
    assert rep.converged and rep.iterations <= 8


def test_zero_rhs_and_max_iter():
    x, rep = solve_case((8, 1, 1), 4, 2, b_value=0.0)
    assert rep.iterations == 0 and rep.converged and (x == 0).all()
    _, rep = solve_case((6, 6, 6), 4, 2, tol=1e-30, max_iter=40)
    assert not rep.converged and rep.iterations == 40


def test_converged_residual_is_true_residual():
    from oracle.repart import build_owner  # noqa: F401  (oracle used as checker only)
    grid, asm, pm = cavity_case((6, 6, 6), 4, 2)
    x, rep = solve_case((6, 6, 6), 4, 2, tol=1e-8)
    probs = ocav.cavity_problems((6, 6, 6), 4)
    pipe = OraclePipeline(probs, pm.offsets, 2)
    ys = pipe.system.spmv([x[p.lo:p.hi] for p in pipe.parts])
    r = 1.0 - np.concatenate(ys)
    true_res = np.linalg.norm(r) / np.sqrt(len(r))
    assert rep.converged and true_res <= 1e-8
    assert abs(true_res - rep.residual) <= 1e-12


def test_solve_deterministic_and_alpha_invariant():
    runs = [solve_case((12, 12, 12), 8, 2, tol=1e-9) for _ in range(3)]
    for x, rep in runs[1:]:
        assert np.array_equal(x, runs[0][0]) and rep.iterations == runs[0][1].iterations
        assert rep.residual == runs[0][1].residual
    # (2 ranks, alpha 1) and (4 ranks, alpha 2) give identical I_GPU at 12^3
    xa, ra = solve_case((12, 12, 12), 2, 1, tol=1e-9)
    xb, rb = solve_case((12, 12, 12), 4, 2, tol=1e-9)
    assert np.array_equal(xa, xb) and ra.iterations == rb.iterations


def test_not_positive_definite_raises():
    grid = lrb.StructuredGrid(6, 6, 6)
    parts = lrb.decompose_slab(grid, 2)
    asm = []
    for p in parts:
        m, ifs = lrb.assemble_poisson(p)
        asm.append((lrb.LduMatrix(m.n_cells, m.lower_addr, m.upper_addr, -m.diag, m.lower_val,
                                  m.upper_val), ifs))
    pm = lrb.make_partition_map([p.n_cells for p in parts], 1)

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        lrb.cg_solve(s.matrix, s.halo, np.ones(s.matrix.n_owned), 1e-8, 100, s.comm)

    with pytest.raises(lrb.RankFailedError) as err:
        lrb.run_world(2, program)
    assert "not positive definite" in str(err.value.cause)


def _momentum(asm, seed=0):
    """Non-symmetric, diagonally dominant LDU on the cavity addressing."""
    rng = np.random.default_rng(seed)
    out = []
    for m, ifs in asm:
        eps_u = 0.05 * rng.random(m.n_faces)
        eps_l = 0.05 * rng.random(m.n_faces)
        mm = lrb.LduMatrix(m.n_cells, m.lower_addr, m.upper_addr, np.full(m.n_cells, 6.5),
                           -1.0 - eps_l, -1.0 + eps_u)
        out.append((mm, ifs))
    return out


@pytest.mark.parametrize("alpha", [1, 2, 4])
def test_bicgstab_matches_oracle(alpha):
    _, asm, pm = cavity_case((12, 12, 12), 4, alpha)
    mom = _momentum(asm)

    def program(ctx):
        s = lrb.repartition(*mom[ctx.rank], pm, ctx)
        if not s.is_owner:
            return None
        x, rep = lrb.bicgstab_solve(s.matrix, s.halo, np.ones(s.matrix.n_owned), 1e-10, 500,
                                    s.comm, history=True)
        pieces = s.comm.gather(x, 0)
        return (np.concatenate(pieces), rep) if pieces is not None else rep

    x, rep = lrb.run_world(4, program)[0]
    probs = [ocav.RankProblem(m.n_cells, m.lower_addr, m.upper_addr, m.diag, m.lower_val,
                              m.upper_val, tuple(ocav.Block(b.neighbor_rank, b.rows, b.cols_remote,
                                                            b.values) for b in ifs))
             for m, ifs in mom]
    pipe = OraclePipeline(probs, pm.offsets, alpha)
    xo, ro = pipe.solve("bicgstab", 1e-10, 500)
    assert rep.converged and ro.converged
    assert abs(rep.iterations - ro.iterations) <= 1
    n = min(len(ro.history), len(rep.history))
    # history is |r|/|b|; the in-part dot order differs from the oracle's, so
    # the tail carries cancellation noise of a few ulps of |b| (atol 1e-13)
    np.testing.assert_allclose(rep.history[:n], ro.history[:n], rtol=1e-8, atol=1e-13)
    np.testing.assert_allclose(x, np.concatenate(xo), rtol=1e-8, atol=1e-12)


def test_cross_device_protocol_on_one_gpu():
    """Parts split into separate 'device ranks' (separate kernels talking through
    the peer-flag protocol) must give bit-identical results to one kernel."""
    from paper_2510_08536_b200.device import Team
    _, asm, pm = cavity_case((16, 16, 16), 4, 1)

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        parts = s.comm.allgather(s.part)
        if s.comm.group_rank == 0:
            bs = [np.ones(p.n) for p in parts]
            one = s.team.solve("cg", bs, 1e-9, 500)
            split = Team(parts, dev_ranks=[0, 0, 1, 1]).solve("cg", bs, 1e-9, 500)
            split4 = Team(parts, dev_ranks=[0, 1, 2, 3]).solve("pcg", bs, 1e-9, 500)
            pcg = s.team.solve("pcg", bs, 1e-9, 500)
            return one, split, split4, pcg
        return None

    one, split, split4, pcg = lrb.run_world(4, program)[0]
    assert one[1].iterations == split[1].iterations
    for a, b in zip(one[0], split[0]):
        assert np.array_equal(a, b)
    assert pcg[1].iterations == split4[1].iterations
    for a, b in zip(pcg[0], split4[0]):
        assert np.array_equal(a, b)


def test_vals_write_through():
    """matrix.local/non_local.vals stay writable (reference tests/test_core.py:121):
    scaling both blocks by 2 in place rewrites the device values and the Jacobi
    diagonal, so Jacobi-PCG on 2A returns exactly x/2 in the same iterations."""
    _, asm, pm = cavity_case((12, 12, 12), 4, 2)

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        lrb.update(s, *lrb.perturb_coefficients(*asm[ctx.rank], 3), "direct")
        out = None
        if s.is_owner:
            b = np.ones(s.matrix.n_owned)
            x1, r1 = lrb.cg_solve(s.matrix, s.halo, b, 1e-8, 500, s.comm, method="pcg")
            lv0, nv0 = s.matrix.local.vals.copy(), s.matrix.non_local.vals.copy()
            v = s.matrix.local.vals
            v *= 2.0
            w = s.matrix.non_local.vals
            w *= 2.0
            ok = np.array_equal(s.matrix.local.vals, 2 * lv0) and \
                np.array_equal(s.matrix.non_local.vals, 2 * nv0)
            x2, r2 = lrb.cg_solve(s.matrix, s.halo, b, 1e-8, 500, s.comm, method="pcg")
            one = s.matrix.local.vals
            one[0] = 123.0
            ok &= s.matrix.local.vals[0] == 123.0
            out = ok, np.array_equal(x2, x1 / 2), r1.iterations == r2.iterations
        return out

    for r in lrb.run_world(4, program):
        if r is not None:
            assert all(r), r


def test_update_on_device_equals_host_update():
    """GPU-side perturb_coefficients installs the host path's
    values bit for bit, step after step, in either order with host updates."""
    _, asm, pm = cavity_case((12, 12, 12), 8, 4)

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        lrb.capture_device_base(s)
        ok = True
        for step in (2, 3, 7, 20):
            lrb.update_on_device(s, step)
            dev = (s.matrix.local.vals.copy(), s.matrix.non_local.vals.copy()) if s.is_owner else None
            lrb.update(s, *lrb.perturb_coefficients(*asm[ctx.rank], step), "direct")
            if s.is_owner:
                ok &= np.array_equal(dev[0], s.matrix.local.vals)
                ok &= np.array_equal(dev[1], s.matrix.non_local.vals)
        if s.is_owner:   # the Jacobi diagonal follows: PCG equals the host-updated solve
            lrb.update_on_device(s, 5)
            xa, ra = lrb.cg_solve(s.matrix, s.halo, np.ones(s.matrix.n_owned), 1e-8, 500, s.comm,
                                  method="pcg")
        else:
            lrb.update_on_device(s, 5)
        lrb.update(s, *lrb.perturb_coefficients(*asm[ctx.rank], 5), "direct")
        if s.is_owner:
            xb, rb = lrb.cg_solve(s.matrix, s.halo, np.ones(s.matrix.n_owned), 1e-8, 500, s.comm,
                                  method="pcg")
            ok &= np.array_equal(xa, xb) and ra.iterations == rb.iterations
        return ok

    assert all(lrb.run_world(8, program))
    with pytest.raises(ValueError, match="step must be >= 1"):
        lrb.update_on_device(None, 0)


def test_pageable_update_chunked_pipeline_values():
    """Pageable inputs larger than the 4 MB host-copy chunk (the pipelined
    stage path) land bit-exactly."""
    _, asm, pm = cavity_case((64, 64, 64), 2, 2)

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        m, ifs = lrb.perturb_coefficients(*asm[ctx.rank], 9)    # fresh pageable arrays
        lrb.update(s, m, ifs, "direct")
        if s.is_owner:
            st = s.part.stats()
            return st["pageable_pieces"] > 0, s.matrix.local.vals, s.matrix.non_local.vals
        return None

    res = lrb.run_world(2, program)
    probs = [ocav.perturb(p, 9) for p in ocav.cavity_problems((64, 64, 64), 2)]
    pipe = OraclePipeline(probs, pm.offsets, 2)
    staged, lv, nv = res[0]
    assert staged
    assert np.array_equal(lv, pipe.values[0][0]) and np.array_equal(nv, pipe.values[0][1])


def test_two_systems_interleaved_updates_and_solves():
    """C4's flow (momentum + pressure systems on the same ranks): sources
    upload the second system's coefficients while the owner is still solving
    the first (update epochs, no owner-group barrier); every value and solve
    equals a fresh repartition of the same step."""
    _, asm, pm = cavity_case((16, 16, 16), 8, 4)

    def program(ctx):
        base = asm[ctx.rank]
        sa = lrb.repartition(*base, pm, ctx)
        sb = lrb.repartition(*base, pm, ctx)
        ok = True
        for step in range(2, 8):
            ma = lrb.perturb_coefficients(*base, step)
            mb = lrb.perturb_coefficients(*base, step + 30)
            lrb.update(sa, *ma, "direct" if step != 5 else "staged")
            if sa.is_owner:
                xa, _ = lrb.cg_solve(sa.matrix, sa.halo, np.ones(sa.matrix.n_owned), 1e-8, 500,
                                     sa.comm, method="pcg")
            lrb.update(sb, *mb, "direct")
            if sb.is_owner:
                xb, _ = lrb.cg_solve(sb.matrix, sb.halo, np.ones(sb.matrix.n_owned), 1e-8, 500,
                                     sb.comm)
            fa = lrb.repartition(*ma, pm, ctx)
            fb = lrb.repartition(*mb, pm, ctx)
            if sa.is_owner:
                ok &= np.array_equal(sa.matrix.local.vals, fa.matrix.local.vals)
                ok &= np.array_equal(sb.matrix.non_local.vals, fb.matrix.non_local.vals)
                ya, _ = lrb.cg_solve(fa.matrix, fa.halo, np.ones(fa.matrix.n_owned), 1e-8, 500,
                                     fa.comm, method="pcg")
                yb, _ = lrb.cg_solve(fb.matrix, fb.halo, np.ones(fb.matrix.n_owned), 1e-8, 500,
                                     fb.comm)
                ok &= np.array_equal(xa, ya) and np.array_equal(xb, yb)
        return ok

    assert all(lrb.run_world(8, program))


def test_update_segments_contiguous_runs():
    """lrb_update_segments: a part's sources produced in pack order into one
    pinned block move as merged host-contiguous runs (across pieces and
    segments); values equal the per-source update bit for bit, also with a
    gap that splits the runs."""
    import torch

    from paper_2510_08536_b200.repart import _pieces
    _, asm, pm = cavity_case((16, 16, 16), 8, 4)
    systems = lrb.run_world(8, lambda ctx: lrb.repartition(*asm[ctx.rank], pm, ctx))
    step = 6
    new = [lrb.perturb_coefficients(*asm[r], step) for r in range(8)]
    for gap in (0, 3):
        for k in range(pm.n_gpu):
            ranks = range(pm.alpha * k, pm.alpha * (k + 1))
            pcs = [_pieces(*new[r]) for r in ranks]
            total = sum(len(p) for ps in pcs for p in ps) + gap * len(ranks)
            block = torch.zeros(total, dtype=torch.float64).pin_memory().numpy()
            views, o = [], 0
            for ps in pcs:
                vs = []
                for p in ps:
                    v = block[o:o + len(p)]
                    v[:] = p
                    vs.append(v)
                    o += len(p)
                o += gap
                views.append(vs)
            part = systems[pm.alpha * k].part
            assert part.update_segments([r % pm.alpha for r in ranks], views)
            part.join()
        dev = [(systems[pm.alpha * k].matrix.local.vals.copy(),
                systems[pm.alpha * k].matrix.non_local.vals.copy()) for k in range(pm.n_gpu)]
        probs = [ocav.perturb(p, step) for p in ocav.cavity_problems((16, 16, 16), 8)]
        pipe = OraclePipeline(probs, pm.offsets, pm.alpha)
        for k in range(pm.n_gpu):
            assert np.array_equal(dev[k][0], pipe.values[k][0])
            assert np.array_equal(dev[k][1], pipe.values[k][1])
        # pageable pieces are refused before anything moves
        assert not systems[0].part.update_segments([0], [_pieces(*asm[0])])


@pytest.mark.parametrize("seed", [1, 2])
def test_random_interleaving_of_update_paths(seed):
    """A seeded random sequence of direct / staged / device-producer updates
    and solves on two systems sharing the ranks: after every operation the
    owners' values equal a fresh repartition of the same coefficients, and
    every solve equals the solve of that fresh system."""
    _, asm, pm = cavity_case((14, 14, 14), 8, 4)
    rng = np.random.default_rng(seed)
    ops = [(int(rng.integers(2)), ["direct", "staged", "device"][int(rng.integers(3))],
            int(rng.integers(2, 40)), bool(rng.integers(2))) for _ in range(10)]

    def program(ctx):
        base = asm[ctx.rank]
        sys_ = [lrb.repartition(*base, pm, ctx), lrb.repartition(*base, pm, ctx)]
        for s in sys_:
            lrb.capture_device_base(s)
        ok = True
        for which, how, step, solve in ops:
            s = sys_[which]
            if how == "device":
                lrb.update_on_device(s, step)
            else:
                lrb.update(s, *lrb.perturb_coefficients(*base, step), how)
            fresh = lrb.repartition(*lrb.perturb_coefficients(*base, step), pm, ctx)
            if s.is_owner:
                ok &= np.array_equal(s.matrix.local.vals, fresh.matrix.local.vals)
                ok &= np.array_equal(s.matrix.non_local.vals, fresh.matrix.non_local.vals)
                if solve:
                    b = np.ones(s.matrix.n_owned)
                    xa, ra = lrb.cg_solve(s.matrix, s.halo, b, 1e-8, 500, s.comm, method="pcg")
                    xb, rb = lrb.cg_solve(fresh.matrix, fresh.halo, b, 1e-8, 500, fresh.comm,
                                          method="pcg")
                    ok &= np.array_equal(xa, xb) and ra.iterations == rb.iterations
        return ok

    assert all(lrb.run_world(8, program))


def test_pageable_arrays_pinned_in_place_on_reuse():
    """The reference generator's arrays (fresh diagonal, the same off-diagonal
    arrays every step): from the second update on, the reused >= 4 MB arrays
    are page-locked in place and go straight to the device (pinned pieces
    counted), the fresh diagonal keeps going through the stage; values stay
    bit-exact and the registration dies with the arrays."""
    import gc

    from paper_2510_08536_b200.device import _host_pins
    _, asm, pm = cavity_case((96, 96, 96), 2, 2)

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        before = s.part.stats() if s.is_owner else None
        for step in (2, 3, 4):
            lrb.update(s, *lrb.perturb_coefficients(*asm[ctx.rank], step), "direct")
        if s.is_owner:
            after = s.part.stats()
            return after["pinned_pieces"] - before["pinned_pieces"], s.matrix.local.vals.copy()
        return None

    res = lrb.run_world(2, program)
    pinned_pieces, lv = res[0]
    assert pinned_pieces >= 2      # upper / lower of both sources at steps 3 and 4
    probs = [ocav.perturb(p, 4) for p in ocav.cavity_problems((96, 96, 96), 2)]
    pipe = OraclePipeline(probs, pm.offsets, 2)
    assert np.array_equal(lv, pipe.values[0][0])
    registered = [k for k, v in _host_pins._seen.items() if v == 2]
    assert registered
    asm.clear()
    gc.collect()
    assert not [k for k in registered if k in _host_pins._seen]
