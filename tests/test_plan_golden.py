"""CPU tests of the native create path (lrb_plan_build_*) against the reference.

The plan is host-side integer work, so it is checked here without a GPU:
fused patterns, halo columns, scatter map, update pattern and the SELL-32
device layout must reproduce the reference's arrays exactly.  The SELL layout
is additionally checked by emulating the device SpMV in numpy and comparing
with the reference's spmv outputs bit for bit.
"""

import re

import numpy as np
import pytest

import paper_2510_08536_b200 as lrb
from golden_cases import case_config, case_meta, case_names, get, golden, matches, spmv_inputs
from helpers_b200 import golden_inputs, owner_buffer, owner_plan, sell_spmv
from oracle import cavity as ocav

CASES = case_names()
SMALL = [c for c in CASES if c not in ("c2",)]


@pytest.mark.parametrize("name", CASES)
def test_plan_matches_reference(name):
    pm, per_rank = golden_inputs(name)
    assert np.array_equal(pm.offsets, golden()[f"{name}__offsets"])
    counts = [lrb.repart._Source(m, ifs, pm, r).n_entries for r, (m, ifs) in enumerate(per_rank)]
    up = lrb.build_update_pattern(pm, counts)
    for k in range(pm.n_gpu):
        plan = owner_plan(pm, per_rank, k)
        loc_ptr, loc_col, nl_ptr, nl_col, halo = plan.csr()
        n = plan.n
        assert matches(name, k, "local_rows", np.repeat(np.arange(n), np.diff(loc_ptr)))
        assert matches(name, k, "local_cols", loc_col)
        assert matches(name, k, "nl_rows", np.repeat(np.arange(n), np.diff(nl_ptr)))
        assert matches(name, k, "nl_cols", nl_col)
        assert matches(name, k, "halo_cols", halo)
        to_local, index = plan.scatter()
        assert matches(name, k, "to_local", to_local)
        assert matches(name, k, "index", index)
        assert matches(name, k, "recv_offsets", up.recv_offsets[k])
        # values through the exported map equal the reference's scattered values
        buf = owner_buffer(per_rank, pm, k)
        lv = np.zeros(plan.nnz_local)
        nv = np.zeros(plan.nnz_nonlocal)
        lv[index[to_local]] = buf[to_local]
        nv[index[~to_local]] = buf[~to_local]
        assert matches(name, k, "vals_1_local", lv)
        assert matches(name, k, "vals_1_nl", nv)
        # halo owners resolve to the neighbour's send list (solver.py:69-77)
        hp, hi = plan.halo_owners()
        assert np.array_equal(hp, pm.col_owner_gpu(halo))
        assert np.array_equal(hi, halo - pm.gpu_offsets[hp])


@pytest.mark.parametrize("name", SMALL)
def test_sell_layout_reproduces_reference_spmv(name):
    pm, per_rank = golden_inputs(name)
    xs = spmv_inputs(name, pm.total_cells)
    if xs is None:
        pytest.skip("no spmv vectors recorded")
    for k in range(pm.n_gpu):
        plan = owner_plan(pm, per_rank, k)
        sp, col, src, dpos = plan.sell()
        buf = owner_buffer(per_rank, pm, k)
        vals = np.where(src >= 0, buf[np.maximum(src, 0)], 0.0)
        lo, hi = pm.gpu_range(k)
        _, _, _, _, halo = plan.csr()
        for i, x in enumerate(xs):
            y = sell_spmv(plan, vals, x[lo:hi], x[halo])
            assert np.array_equal(y, get(name, k, f"spmv_{i}")), (name, k, i)
        # diagonal slot of every row
        rows_with_diag = dpos >= 0
        assert rows_with_diag.all()


@pytest.mark.parametrize("dims,n", [((8, 1, 1), 4), ((6, 6, 6), 4), ((7, 9, 11), 6),
                                    ((12, 12, 12), 8), ((5, 13, 4), 3), ((1, 9, 1), 3),
                                    ((10, 1, 10), 5), ((32, 32, 32), 4)])
def test_product_generator_matches_oracle(dims, n):
    parts = lrb.decompose_slab(lrb.StructuredGrid(*dims), n)
    oracle = ocav.cavity_problems(dims, n)
    for p, o in zip(parts, oracle):
        m, ifs = lrb.assemble_poisson(p)
        assert m.n_cells == o.n
        assert np.array_equal(m.lower_addr, o.lower) and np.array_equal(m.upper_addr, o.upper)
        assert np.array_equal(m.diag, o.diag)
        assert [b.neighbor_rank for b in ifs] == [b.nbr for b in o.blocks]
        for b, ob in zip(ifs, o.blocks):
            assert np.array_equal(b.rows, ob.rows) and np.array_equal(b.cols_remote, ob.cols)
        for s in (2, 7):
            ms, _ = lrb.perturb_coefficients(m, ifs, s)
            assert np.array_equal(ms.diag, ocav.perturb(o, s).diag)
            out = np.empty_like(m.diag)
            lrb.perturb_diag_into(m.diag, s, out)
            assert np.array_equal(out, ms.diag)


def test_library_exports_every_header_symbol():
    import os
    from paper_2510_08536_b200 import _native
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "ldurepart_b200.h")).read()
    names = set(re.findall(r"\b(lrb_[a-z_]+)\s*\(", hdr))
    assert len(names) >= 30
    for nm in sorted(names):
        assert hasattr(_native.lib, nm), nm
    assert set(_native.EXPORTED) >= names


def test_plan_rejects_overlapping_ownership():
    pm = lrb.make_partition_map([2, 2], 2)
    good = lrb.SparsityPattern(np.array([0, 0, 1]), np.array([0, 2, 1]), np.array([0]),
                               np.array([2]), 0, 2)
    other = lrb.SparsityPattern(np.array([2, 3]), np.array([2, 3]), np.zeros(0, np.int64),
                                np.zeros(0, np.int64), 2, 4)
    with pytest.raises(ValueError, match="overlapping ownership"):
        lrb.fuse_patterns([good, other], pm, 0)


def test_lowlevel_api_matches_reference_chain():
    """extract / fuse / scatter-map helpers on the W1 chain (test_repart.py:22-171)."""
    grid = lrb.StructuredGrid(8, 1, 1)
    parts = lrb.decompose_slab(grid, 4)
    asm = [lrb.assemble_poisson(p) for p in parts]
    pm = lrb.make_partition_map([p.n_cells for p in parts], 2)
    sp = lrb.extract_sparsity(*asm[1], pm, 1)
    pairs = lambda r, c: set(zip(r.tolist(), c.tolist()))
    assert pairs(sp.local_rows, sp.local_cols) == {(2, 2), (2, 3), (3, 2), (3, 3)}
    assert pairs(sp.nonlocal_rows, sp.nonlocal_cols) == {(2, 1), (3, 4)}
    recv = [lrb.extract_sparsity(*asm[r], pm, r) for r in (0, 1)]
    local, nonlocal_ = lrb.fuse_patterns(recv, pm, 0)
    assert len(local[0]) == 10 and pairs(*nonlocal_) == {(3, 4)}
    sm = lrb.build_scatter_map(recv, local, nonlocal_, pm)
    assert sm.to_local[0] and (local[0][sm.index[0]], local[1][sm.index[0]]) == (0, 0)
    assert not sm.to_local[10]
    assert (nonlocal_[0][sm.index[10]], nonlocal_[1][sm.index[10]]) == (3, 4)
    counts = [lrb.extract_sparsity(*asm[r], pm, r).n_entries for r in range(4)]
    assert counts == [5, 6, 6, 5]
    up = lrb.build_update_pattern(pm, counts)
    assert up.segments(0) == [(0, 0, 5), (1, 5, 6)] and up.total(0) == 11
    with pytest.raises(ValueError, match="bijection"):
        lrb.ScatterMap(to_local=[True, True], index=[0, 0], n_local=2, n_nonlocal=0)
    with pytest.raises(ValueError, match="inconsistent interface"):
        lrb.extract_sparsity(asm[1][0], [lrb.InterfaceBlock(0, [0], [7], [-1.0])], pm, 1)


def test_plan_errors_map_to_reference_messages():
    with pytest.raises(ValueError, match="invalid ratio"):
        lrb.make_partition_map([1, 2, 3], 2)
    with pytest.raises(ValueError, match="empty part"):
        lrb.make_partition_map([1, 0], 1)
    with pytest.raises(ValueError, match=r"malformed LDU.*face 1"):
        lrb.LduMatrix(3, [0, 0], [1, 1], [1.0, 1.0, 1.0], [0.0, 0.0], [0.0, 0.0])
    with pytest.raises(ValueError, match="too many parts"):
        lrb.decompose_slab(lrb.StructuredGrid(4, 1, 1), 5)
    with pytest.raises(ValueError, match="row-major"):
        lrb.CooMatrix(2, 2, [1, 0], [0, 0], [1.0, 1.0])
    with pytest.raises(ValueError, match="duplicate"):
        lrb.coo_from_entries(2, 2, [0, 0], [1, 1], [1.0, 2.0])
    with pytest.raises(ValueError, match="out of range"):
        lrb.CooMatrix(2, 2, [0, 2], [0, 0], [1.0, 1.0])
