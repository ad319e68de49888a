"""Krylov parity beyond the reference's CG, at the north_star bar (recurrence
residual history within 1e-10 relative, iterations +-1).

* BiCGStab (momentum; not in the reference): against the oracle's
  restatement (oracle/krylov.py bicgstab) at 12^3, 48^3 and
  100^3 on the non-symmetric momentum LDU, tol 1e-6 as the configs.
* Single-reduction Jacobi-PCG (method "pcg1"): against the
  oracle's Chronopoulos-Gear restatement (krylov.pcg1) and, on the
  uniform-diagonal cavity, against the reference's own CG logs.
* Pipelined Jacobi-PCG (method "pipecg"): against the oracle's
  Ghysels-Vanroose restatement (krylov.pipecg), the reference's CG logs, and
  the max_iter edge (the kernel decides iteration k one phase late).
"""

import numpy as np
import pytest

import paper_2510_08536_b200 as lrb
from golden_cases import get, history_ok, ref_history
from helpers_b200 import cavity_case, golden_inputs, momentum_ldu, oracle_problems
from oracle.pipeline import OraclePipeline

pytestmark = pytest.mark.gpu

TOL = 1e-6


def _solve_gpu(pm, per_rank, method, step=None, tol=TOL):
    def program(ctx):
        m, ifs = per_rank[ctx.rank]
        s = lrb.repartition(m, ifs, pm, ctx)
        if step is not None:
            lrb.update(s, *lrb.perturb_coefficients(m, ifs, step), "direct")
        if not s.is_owner:
            return None
        x, rep = lrb.cg_solve(s.matrix, s.halo, np.ones(s.matrix.n_owned), tol, 2000, s.comm,
                              method=method, history=True)
        pieces = s.comm.gather(x, 0)
        return (np.concatenate(pieces), rep) if pieces is not None else rep

    return lrb.run_world(pm.n_cpu, program, timeout=1800)[0]


def _compare(rep, ro, x, xo, rtol=1e-10):
    assert rep.converged and ro.converged
    assert abs(rep.iterations - ro.iterations) <= 1, (rep.iterations, ro.iterations)
    ok, n = history_ok(rep.history, ro.history, rtol=rtol)
    assert ok and n >= min(len(ro.history), rep.iterations) - 1, (rep.history, ro.history)
    np.testing.assert_allclose(x, np.concatenate(xo), rtol=1e-8, atol=1e-12)


# BiCGStab's recurrence amplifies dot-product rounding far more than CG's: the
# oracle against ITSELF with another equally valid dot order (owner partition
# alpha 2 vs 8, or exactly rounded math.fsum dots) moves the history by
# 7e-10 / 1.1e-9 at 48^3 and 1.9e-8 / 1.7e-8 at 100^3 (tests/test_oracle_golden.py
# test_oracle_bicgstab_dot_order_envelope).  No implementation whose in-part
# dot order differs from numpy's can meet 1e-10 there, so the bar is 1e-10
# where the envelope allows it (12^3) and ~5x the measured envelope above.
BICG_RTOL = {12: 1e-10, 48: 5e-9, 100: 1e-7}


@pytest.mark.parametrize("dims,n_cpu,alpha", [((12, 12, 12), 4, 1), ((12, 12, 12), 4, 2),
                                              ((12, 12, 12), 4, 4), ((48, 48, 48), 8, 2),
                                              ((100, 100, 100), 8, 8)])
def test_bicgstab_matches_oracle(dims, n_cpu, alpha):
    _, asm, pm = cavity_case(dims, n_cpu, alpha)
    mom = momentum_ldu(asm)
    x, rep = _solve_gpu(pm, mom, "bicgstab")
    pipe = OraclePipeline(oracle_problems(mom), pm.offsets, alpha)
    xo, ro = pipe.solve("bicgstab", TOL, 2000)
    rtol = BICG_RTOL[dims[0]]
    assert rep.converged and ro.converged
    assert abs(rep.iterations - ro.iterations) <= 1, (rep.iterations, ro.iterations)
    ok, n = history_ok(rep.history, ro.history, rtol=rtol)
    dev = np.max(np.abs(np.asarray(rep.history[:n]) - ro.history[:n]) / np.asarray(ro.history[:n]))
    assert ok and n >= min(len(ro.history), rep.iterations) - 1, (dev, rtol)
    np.testing.assert_allclose(x, np.concatenate(xo), rtol=max(1e-8, 10 * rtol), atol=1e-12)


@pytest.mark.parametrize("dims,n_cpu,alpha", [((12, 12, 12), 8, 4), ((48, 48, 48), 8, 2),
                                              ((100, 100, 100), 8, 8)])
def test_pcg1_matches_oracle_pcg1(dims, n_cpu, alpha):
    _, asm, pm = cavity_case(dims, n_cpu, alpha)
    x, rep = _solve_gpu(pm, asm, "pcg1", step=3)
    from oracle import cavity as ocav
    probs = [ocav.perturb(p, 3) for p in oracle_problems(asm)]
    pipe = OraclePipeline(probs, pm.offsets, alpha)
    xo, ro = pipe.solve("pcg1", TOL, 2000)
    _compare(rep, ro, x, xo)


# GV's recurrences carry one more level of accumulated rounding than CG's
# (tests/test_oracle_golden.py: 2.1e-10 against the reference's CG at c1)
PIPE_RTOL = 1e-9


@pytest.mark.parametrize("dims,n_cpu,alpha", [((12, 12, 12), 8, 4), ((12, 12, 12), 8, 8),
                                              ((48, 48, 48), 8, 2), ((100, 100, 100), 8, 8)])
@pytest.mark.parametrize("defer", ["0", "1"])
def test_pipecg_matches_oracle_pipecg(dims, n_cpu, alpha, defer, monkeypatch):
    monkeypatch.setenv("LRB_PIPE_DEFER", defer)
    _, asm, pm = cavity_case(dims, n_cpu, alpha)
    x, rep = _solve_gpu(pm, asm, "pipecg", step=3)
    from oracle import cavity as ocav
    probs = [ocav.perturb(p, 3) for p in oracle_problems(asm)]
    pipe = OraclePipeline(probs, pm.offsets, alpha)
    xo, ro = pipe.solve("pipecg", TOL, 2000)
    _compare(rep, ro, x, xo, rtol=PIPE_RTOL)


@pytest.mark.parametrize("name", ["c1", "cav12x12x12_r8_a2", "cav7x9x11_r6_a3"])
def test_pipecg_matches_reference_cg(name):
    """Uniform cavity diagonal: pipecg's iterates are CG's up to rounding, so
    its recurrence residuals follow the reference's recorded CG log."""
    pm, per_rank = golden_inputs(name)
    for s in (2, 3):
        _, rep = _solve_gpu(pm, per_rank, "pipecg", step=s)
        it_ref = int(get(name, 0, f"cg_{s}_rep")[0])
        ref = ref_history(get(name, 0, f"cg_{s}_log"), it_ref, TOL)
        assert rep.converged and abs(rep.iterations - it_ref) <= 1
        assert history_ok(rep.history, ref, rtol=PIPE_RTOL)[0], (rep.history, ref)


@pytest.mark.parametrize("defer", ["0", "1"])
@pytest.mark.parametrize("alpha", [8, 4])   # one part (flat team) / two parts
@pytest.mark.parametrize("max_iter", [1, 2, 9, 10, 11, 17])
def test_pipecg_max_iter_edge(alpha, max_iter, defer, monkeypatch):
    """With LRB_PIPE_DEFER=1 the kernel learns iteration k's residual during
    phase k+1: at max_iter it must still take the last decision (true
    residual at the 10th), report max_iter iterations and return x_max_iter,
    exactly as the oracle (and as the reducing variant)."""
    monkeypatch.setenv("LRB_PIPE_DEFER", defer)
    _, asm, pm = cavity_case((24, 24, 24), 8, alpha)

    def program(ctx):
        m, ifs = asm[ctx.rank]
        s = lrb.repartition(m, ifs, pm, ctx)
        lrb.update(s, *lrb.perturb_coefficients(m, ifs, 3), "direct")
        if not s.is_owner:
            return None
        x, rep = lrb.cg_solve(s.matrix, s.halo, np.ones(s.matrix.n_owned), TOL, max_iter, s.comm,
                              method="pipecg", history=True)
        pieces = s.comm.gather(x, 0)
        return (np.concatenate(pieces), rep) if pieces is not None else rep

    x, rep = lrb.run_world(pm.n_cpu, program, timeout=600)[0]
    from oracle import cavity as ocav
    probs = [ocav.perturb(p, 3) for p in oracle_problems(asm)]
    xo, ro = OraclePipeline(probs, pm.offsets, alpha).solve("pipecg", TOL, max_iter)
    assert rep.iterations == ro.iterations == max_iter and not rep.converged and not ro.converged
    assert len(rep.history) == max_iter
    assert history_ok(rep.history, ro.history, rtol=PIPE_RTOL)[0]
    np.testing.assert_allclose(rep.residual, ro.residual, rtol=1e-8)
    np.testing.assert_allclose(x, np.concatenate(xo), rtol=1e-9, atol=1e-13)


@pytest.mark.parametrize("name", ["c1", "cav12x12x12_r8_a2", "cav7x9x11_r6_a3"])
def test_pcg1_matches_reference_cg(name):
    """Uniform cavity diagonal: pcg1's iterates are CG's up to rounding, so its
    recurrence residuals follow the reference's recorded CG log."""
    pm, per_rank = golden_inputs(name)
    for s in (2, 3):
        _, rep = _solve_gpu(pm, per_rank, "pcg1", step=s)
        it_ref = int(get(name, 0, f"cg_{s}_rep")[0])
        ref = ref_history(get(name, 0, f"cg_{s}_log"), it_ref, TOL)
        assert abs(rep.iterations - it_ref) <= 1
        assert history_ok(rep.history, ref)[0], (rep.history, ref)


@pytest.mark.parametrize("dims,n_cpu,alpha", [((12, 12, 12), 4, 2), ((20, 18, 16), 6, 3)])
def test_bicgstab_solution_against_direct_solve(dims, n_cpu, alpha):
    """An independent check of BiCGStab (the reference has none): the GPU
    solution of the non-symmetric momentum system at tol 1e-12 equals SciPy's
    direct sparse solve of the gathered global matrix to 1e-9."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    _, asm, pm = cavity_case(dims, n_cpu, alpha)
    mom = momentum_ldu(asm, seed=4)

    def program(ctx):
        s = lrb.repartition(*mom[ctx.rank], pm, ctx)
        if not s.is_owner:
            return None
        rng = np.random.default_rng(100 + s.gpu_rank)
        b = rng.standard_normal(s.matrix.n_owned)
        x, rep = lrb.bicgstab_solve(s.matrix, s.halo, b, 1e-12, 2000, s.comm)
        g = lrb.gather_global(s.matrix, pm, s.comm)
        xs = s.comm.gather(x, 0)
        bs = s.comm.gather(b, 0)
        return (g, np.concatenate(xs), np.concatenate(bs), rep) if g is not None else None

    g, x, b, rep = lrb.run_world(n_cpu, program)[0]
    assert rep.converged
    A = sp.coo_matrix((g.vals, (g.rows, g.cols)), shape=(g.n_rows, g.n_cols)).tocsc()
    xd = spla.spsolve(A, b)
    assert np.linalg.norm(x - xd) <= 1e-9 * np.linalg.norm(xd)
    assert np.linalg.norm(A @ x - b) <= 1e-11 * np.linalg.norm(b)


@pytest.mark.parametrize("defer", ["0", "1"])
def test_pipecg_repeated_solves(defer, monkeypatch):
    """Regression (deferred variant): the reducer of phase k+1 published its
    scalars into the buffer that slow warps of the post-phase code of phase k
    were still reading, which split a CTA's control flow and deadlocked the
    second 68-iteration solve at 100^3 (tools/pipe_repro.py).  Repeated
    solves over timesteps must stay deterministic and equal the oracle's
    iteration counts within one."""
    monkeypatch.setenv("LRB_PIPE_DEFER", defer)
    monkeypatch.setenv("LRB_BARRIER_TIMEOUT_S", "20")
    _, asm, pm = cavity_case((100, 100, 100), 8, 8)
    steps = [2, 2, 3, 2, 3]

    def program(ctx):
        m, ifs = asm[ctx.rank]
        s = lrb.repartition(m, ifs, pm, ctx)
        out = []
        for st in steps:
            lrb.update(s, *lrb.perturb_coefficients(m, ifs, st), "direct")
            if s.is_owner:
                x, rep = lrb.cg_solve(s.matrix, s.halo, np.ones(s.matrix.n_owned), TOL, 2000, s.comm,
                                      method="pipecg", history=True)
                out.append((rep.iterations, rep.converged, tuple(rep.history), x.copy()))
        return out

    res = lrb.run_world(pm.n_cpu, program, timeout=600)[0]
    it2, it3 = res[0][0], res[2][0]
    for (it, conv, hist, x), st in zip(res, steps):
        assert conv and it == (it2 if st == 2 else it3)
    for a, b in ((0, 1), (0, 3), (2, 4)):   # same timestep, bit-identical
        assert res[a][2] == res[b][2] and np.array_equal(res[a][3], res[b][3])
