"""Stream-ordered C-ABI (lrb_update_segment_async / lrb_team_solve_async /
lrb_team_spmv_async): the GPU-resident plugin path of SURVEY §8(b).  Device
pointers in and out, a caller-owned CUDA stream, no host synchronisation
inside the calls.  Results must equal the synchronous drop-in path bit for
bit (same kernels, same inputs) and the oracle's scattered values."""

import numpy as np
import pytest

import paper_2510_08536_b200 as lrb
from helpers_b200 import cavity_case
from oracle import cavity as ocav
from oracle.pipeline import OraclePipeline
from paper_2510_08536_b200.repart import _pieces

pytestmark = pytest.mark.gpu

DIMS, N_CPU, ALPHA, STEP = (12, 12, 12), 8, 4, 3


def _setup():
    _, asm, pm = cavity_case(DIMS, N_CPU, ALPHA)

    def program(ctx):
        return lrb.repartition(*asm[ctx.rank], pm, ctx)

    systems = lrb.run_world(N_CPU, program)
    return asm, pm, systems


@pytest.mark.parametrize("src_kind", ["pinned", "device"])
def test_async_update_solve_matches_sync_path(src_kind):
    import torch
    asm, pm, systems = _setup()
    owners = [systems[ALPHA * k] for k in range(pm.n_gpu)]
    team = owners[0].team
    stream = torch.cuda.Stream()
    keep = []
    with torch.cuda.stream(stream):
        for r in range(N_CPU):
            s = systems[r]
            pieces = _pieces(*lrb.perturb_coefficients(*asm[r], STEP))
            ts = []
            for p in pieces:
                t = torch.from_numpy(np.ascontiguousarray(p, dtype=np.float64))
                t = t.pin_memory() if src_kind == "pinned" else t.to("cuda:0", non_blocking=False)
                ts.append(t)
            keep.append(ts)
            s.part.update_segment_async(s.segment, ts, stream.cuda_stream)
        b = [torch.ones(o.part.n, dtype=torch.float64, device="cuda:0") for o in owners]
        x = [torch.full((o.part.n,), float("nan"), dtype=torch.float64, device="cuda:0")
             for o in owners]
        rep = torch.zeros(64, dtype=torch.uint8).pin_memory()
        team.solve_async("pcg", b, x, 1e-6, 2000, streams=[stream.cuda_stream], report=rep)
        y = [torch.empty_like(v) for v in x]
        team.spmv_async(x, y, streams=[stream.cuda_stream])
    stream.synchronize()
    ra = team.report_from(rep)
    assert ra.status == 0 and ra.converged == 1 and ra.device_ms == -1.0
    xa = [v.cpu().numpy() for v in x]
    ya = [v.cpu().numpy() for v in y]

    # values: oracle, bit for bit
    probs = [ocav.perturb(p, STEP) for p in ocav.cavity_problems(DIMS, N_CPU)]
    pipe = OraclePipeline(probs, pm.offsets, ALPHA)
    for k, o in enumerate(owners):
        lv, nv = pipe.values[k]
        assert np.array_equal(o.matrix.local.vals, lv)
        assert np.array_equal(o.matrix.non_local.vals, nv)

    # the synchronous drop-in path on the same system: identical iterates
    xs, rs, _ = team.solve("pcg", [np.ones(o.part.n) for o in owners], 1e-6, 2000)
    assert rs.iterations == ra.iterations and rs.residual == ra.residual
    for k in range(pm.n_gpu):
        assert np.array_equal(xs[k], xa[k])
    ys = team.spmv(xs)
    for k in range(pm.n_gpu):
        assert np.array_equal(ys[k], ya[k])


def test_async_update_rejects_pageable():
    asm, pm, systems = _setup()
    s = systems[1]
    pieces = _pieces(*lrb.perturb_coefficients(*asm[1], STEP))

    class _Host:   # a pageable numpy array behind the tensor interface
        def __init__(self, a):
            self.a = np.ascontiguousarray(a, dtype=np.float64)

        def data_ptr(self):
            return self.a.ctypes.data

        def numel(self):
            return self.a.size

    with pytest.raises(ValueError, match="pageable"):
        s.part.update_segment_async(s.segment, [_Host(p) for p in pieces], 0)


def test_async_length_violation():
    import torch
    asm, pm, systems = _setup()
    s = systems[1]
    t = torch.zeros(5, dtype=torch.float64, device="cuda:0")
    with pytest.raises(ValueError, match="update pattern violation"):
        s.part.update_segment_async(s.segment, [t], 0)


def test_async_solve_split_device_ranks():
    """Two device ranks on one GPU (the cross-device peer protocol): the
    stream-ordered solve orders each device's inputs before every device's
    kernel (join_devices) and equals the synchronous solve bit for bit."""
    import torch

    from paper_2510_08536_b200.device import Team
    asm, pm, systems = _setup()
    owners = [systems[ALPHA * k] for k in range(pm.n_gpu)]
    parts = [o.part for o in owners]
    team = Team(parts, dev_ranks=list(range(len(parts))))
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    rng = np.random.default_rng(3)
    bh = [rng.standard_normal(p.n) for p in parts]
    b = [torch.from_numpy(v).to("cuda:0") for v in bh]
    x = [torch.zeros(p.n, dtype=torch.float64, device="cuda:0") for p in parts]
    rep = torch.zeros(64, dtype=torch.uint8).pin_memory()
    torch.cuda.synchronize()
    team.solve_async("pcg", b, x, 1e-8, 500, streams=[s0.cuda_stream, s1.cuda_stream], report=rep)
    s0.synchronize()
    s1.synchronize()
    ra = team.report_from(rep)
    xs, rs, _ = team.solve("pcg", bh, 1e-8, 500)
    assert ra.converged == 1 and ra.iterations == rs.iterations and ra.residual == rs.residual
    for k in range(len(parts)):
        assert np.array_equal(x[k].cpu().numpy(), xs[k])
