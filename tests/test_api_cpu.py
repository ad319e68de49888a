"""CPU tests of the drop-in API surface (no GPU): the reference's error
contracts and invariants (message substrings, frozen pattern
arrays, partition maps, LDU -> COO) and a seeded property test of the
world-free create pipeline (extract -> fuse -> scatter map) on random
partitioned systems: the scatter map is a bijection and moves every packed
coefficient to the slot of its (row, col) in the fused matrix.

The random generator mirrors the reference helpers' contract (a symmetric
pattern split into contiguous rank blocks, non-symmetric values); it is a
fresh implementation, seeded with default_rng(2024) like the reference's
acceptance test (test_acceptance.py:91-114).
"""

import numpy as np
import pytest

import paper_2510_08536_b200 as lrb
from helpers_b200 import chain_setup


# ---------------------------------------------------------------- partition map
def test_partition_map_ranges_and_owner():
    pm = lrb.make_partition_map([3, 2, 4, 1], 2)
    cpu = [c for r in range(pm.n_cpu) for c in range(*pm.cpu_range(r))]
    gpu = [c for k in range(pm.n_gpu) for c in range(*pm.gpu_range(k))]
    assert cpu == gpu == list(range(pm.total_cells))
    assert [lrb.gpu_owner(r, pm) for r in range(4)] == [0, 0, 1, 1]
    pm16 = lrb.make_partition_map([1] * 16, 4)
    assert [lrb.gpu_owner(r, pm16) for r in range(16)] == sorted(list(range(4)) * 4)
    with pytest.raises(ValueError, match="out of range"):
        lrb.gpu_owner(4, pm)


@pytest.mark.parametrize("cells,alpha,msg", [([1, 1, 1], 2, "invalid ratio"),
                                             ([2, 0, 2, 2], 2, "empty part")])
def test_partition_map_errors(cells, alpha, msg):
    with pytest.raises(ValueError, match=msg):
        lrb.make_partition_map(cells, alpha)


# --------------------------------------------------------------- LDU / COO types
def test_ldu_validation_names_the_face():
    with pytest.raises(ValueError, match="malformed LDU.*face 0"):
        lrb.LduMatrix(3, [1], [0], [1, 1, 1], [0], [0])
    with pytest.raises(ValueError, match="malformed LDU.*face 1"):
        lrb.LduMatrix(3, [0, 0], [2, 1], [1, 1, 1], [0, 0], [0, 0])
    with pytest.raises(ValueError, match="malformed LDU"):
        lrb.LduMatrix(3, [0, 0], [1, 1], [1, 1, 1], [0, 0], [0, 0])


def test_coo_contracts():
    with pytest.raises(ValueError, match="row-major"):
        lrb.CooMatrix(2, 2, [1, 0], [0, 0], [1.0, 1.0])
    with pytest.raises(ValueError, match="duplicate"):
        lrb.coo_from_entries(2, 2, [0, 0], [1, 1], [1.0, 2.0])
    c = lrb.coo_from_entries(2, 2, [1, 0], [0, 1], [2.0, 1.0])
    assert list(c.rows) == [0, 1] and list(c.cols) == [1, 0]   # sorted row-major
    with pytest.raises(ValueError):
        c.rows[0] = 1                                           # pattern frozen
    c.vals[0] = 5.0                                             # values writable


def _dense(m: lrb.LduMatrix):
    a = np.diag(np.asarray(m.diag, float))
    for f in range(m.n_faces):
        l, u = m.lower_addr[f], m.upper_addr[f]
        a[l, u] += m.upper_val[f]
        a[u, l] += m.lower_val[f]
    return a


@pytest.mark.parametrize("seed", range(5))
def test_ldu_to_coo_matches_dense_expansion(seed):
    rng = np.random.default_rng(seed)
    n = 12
    pairs = sorted({(i, j) for i, j in rng.integers(0, n, (30, 2)) if i < j})
    lo = np.array([p[0] for p in pairs], np.int64)
    up = np.array([p[1] for p in pairs], np.int64)
    m = lrb.LduMatrix(n, lo, up, rng.random(n), rng.random(len(pairs)), rng.random(len(pairs)))
    coo = lrb.ldu_to_coo(m)
    dense = np.zeros((n, n))
    dense[coo.rows, coo.cols] = coo.vals
    np.testing.assert_array_equal(dense, _dense(m))
    assert coo.nnz == n + 2 * len(pairs)


# --------------------------------------------------------------- cavity inputs
def test_cavity_generator_contracts():
    with pytest.raises(ValueError, match="too many parts"):
        lrb.decompose_slab(lrb.StructuredGrid(4, 4, 4), 8)
    parts = lrb.decompose_slab(lrb.StructuredGrid(6, 5, 4), 3)
    assert sum(p.n_cells for p in parts) == 6 * 5 * 4
    for p in parts:
        m, ifs = lrb.assemble_poisson(p)
        assert np.all(m.diag == 6.0)                       # uniform diagonal in 3D
        assert np.all(m.lower_val == -1.0) and np.all(m.upper_val == -1.0)
        for b in ifs:
            assert np.all(b.values == -1.0)
        m3, _ = lrb.perturb_coefficients(m, ifs, 3)
        assert np.all(m3.diag == 6.0 * 1.03) and m3.lower_val is m.lower_val
    with pytest.raises(ValueError):
        lrb.perturb_coefficients(m, ifs, 0)


# ------------------------------------------------------- create-path contracts
def test_inconsistent_interface_rejected():
    _, _, assembled, pm = chain_setup(alpha=2)
    m, _ = assembled[1]
    bad = [lrb.InterfaceBlock(0, rows=[0], cols_remote=[7], values=[-1.0])]
    with pytest.raises(ValueError, match="inconsistent interface"):
        lrb.extract_sparsity(m, bad, pm, 1)


def test_scatter_map_bijection_validated():
    with pytest.raises(ValueError, match="bijection"):
        lrb.ScatterMap(to_local=[True, True], index=[0, 0], n_local=2, n_nonlocal=0)


# ----------------------------------------------- random partitioned systems
def random_system(rng, n_ranks_choices=(2, 4, 6, 8), alphas=(1, 2)):
    """Symmetric random pattern over contiguous rank blocks, non-symmetric values."""
    n_ranks = int(rng.choice(n_ranks_choices))
    alpha = int(rng.choice([a for a in alphas if n_ranks % a == 0]))
    cells = rng.integers(1, 6, n_ranks)
    off = np.concatenate(([0], np.cumsum(cells)))
    total = int(off[-1])
    pairs = {(i, j) for i, j in rng.integers(0, total, (3 * total, 2)) if i < j}
    owner = np.searchsorted(off, np.arange(total), side="right") - 1
    per_rank, values = [], {}
    for r in range(n_ranks):
        lo_r = off[r]
        local = sorted((i, j) for i, j in pairs if owner[i] == r and owner[j] == r)
        n = int(cells[r])
        diag = 4.0 + rng.random(n)
        lower = np.array([i - lo_r for i, _ in local], np.int64)
        upper = np.array([j - lo_r for _, j in local], np.int64)
        lval, uval = -rng.random(len(local)), -rng.random(len(local))
        for c in range(n):
            values[(lo_r + c, lo_r + c)] = diag[c]
        for (i, j), lv, uv in zip(local, lval, uval):
            values[(i, j)] = uv
            values[(j, i)] = lv
        blocks = []
        for nb in range(n_ranks):
            if nb == r:
                continue
            cross = sorted({(i, j) for i, j in pairs if owner[i] == r and owner[j] == nb} |
                           {(j, i) for i, j in pairs if owner[j] == r and owner[i] == nb})
            if not cross:
                continue
            rows = np.array([i - lo_r for i, _ in cross], np.int64)
            cols = np.array([j - off[nb] for _, j in cross], np.int64)
            vals = -rng.random(len(cross))
            for (i, j), v in zip(cross, vals):
                values[(i, j)] = v
            blocks.append(lrb.InterfaceBlock(nb, rows, cols, vals))
        per_rank.append((lrb.LduMatrix(n, lower, upper, diag, lval, uval), blocks))
    return lrb.make_partition_map(list(cells), alpha), per_rank, values


@pytest.mark.parametrize("chunk", range(4))
def test_random_systems_scatter_is_a_value_preserving_bijection(chunk):
    rng = np.random.default_rng(2024 + chunk)
    for _ in range(25):
        pm, per_rank, values = random_system(rng)
        sps = [lrb.extract_sparsity(m, ifs, pm, r) for r, (m, ifs) in enumerate(per_rank)]
        for k in range(pm.n_gpu):
            src = range(pm.alpha * k, pm.alpha * (k + 1))
            received = [sps[r] for r in src]
            loc, nl = lrb.fuse_patterns(received, pm, k)
            sm = lrb.build_scatter_map(received, loc, nl, pm)
            buf = np.concatenate([lrb.pack_coefficients(*per_rank[r], r).values for r in src])
            assert len(buf) == sm.n_local + sm.n_nonlocal          # bijection: sizes
            out_l, out_n = np.full(sm.n_local, np.nan), np.full(sm.n_nonlocal, np.nan)
            out_l[sm.index[sm.to_local]] = buf[sm.to_local]
            out_n[sm.index[~sm.to_local]] = buf[~sm.to_local]
            assert not np.isnan(out_l).any() and not np.isnan(out_n).any()   # onto
            lr_, lc = np.asarray(loc[0]), np.asarray(loc[1])
            got = {(int(i), int(j)): v for i, j, v in zip(lr_, lc, out_l)}
            nr, nc = np.asarray(nl[0]), np.asarray(nl[1])
            got.update({(int(i), int(j)): v for i, j, v in zip(nr, nc, out_n)})
            lo, hi = pm.gpu_range(k)
            want = {key: v for key, v in values.items() if lo <= key[0] < hi}
            assert got == want


# ------------------------------------------------ wire formats
def test_matrix_market_round_trip_and_text(tmp_path):
    c = lrb.coo_from_entries(3, 4, [2, 0, 0, 1], [3, 1, 0, 2], [0.1, -1.0, 6.0, 1e-300])
    path = tmp_path / "m.mtx"
    lrb.write_matrix_market(c, path)
    text = path.read_text().splitlines()
    assert text[0] == lrb.MM_HEADER == "%%MatrixMarket matrix coordinate real general"
    assert text[1] == "3 4 4"
    # 1-based, row-major, 17 significant digits (the reference's export layout)
    assert text[2:] == ["1 1 6", "1 2 -1", "2 3 1e-300",
                        "3 4 0.10000000000000001"]
    back = lrb.read_matrix_market(path)
    assert (back.n_rows, back.n_cols) == (3, 4)
    np.testing.assert_array_equal(back.rows, c.rows)
    np.testing.assert_array_equal(back.cols, c.cols)
    np.testing.assert_array_equal(back.vals, c.vals)   # %.17g round-trips every double


def test_matrix_market_random_round_trip(tmp_path):
    rng = np.random.default_rng(11)
    pm, per_rank, values = random_system(rng)
    n = pm.total_cells
    keys = sorted(values)
    c = lrb.coo_from_entries(n, n, [k[0] for k in keys], [k[1] for k in keys],
                             [values[k] for k in keys])
    lrb.write_matrix_market(c, tmp_path / "r.mtx", block=7)
    back = lrb.read_matrix_market(tmp_path / "r.mtx")
    np.testing.assert_array_equal(back.vals, c.vals)
    np.testing.assert_array_equal(back.cols, c.cols)


def test_matrix_market_errors(tmp_path):
    (tmp_path / "a.mtx").write_text("hello\n")
    with pytest.raises(ValueError, match="not a Matrix Market file"):
        lrb.read_matrix_market(tmp_path / "a.mtx")
    (tmp_path / "b.mtx").write_text("%%MatrixMarket matrix array real general\n1 1\n1\n")
    with pytest.raises(ValueError, match="unsupported Matrix Market header"):
        lrb.read_matrix_market(tmp_path / "b.mtx")


def test_curves_csv(tmp_path):
    path = tmp_path / "c.csv"
    lrb.write_curves_csv(path, [(4, 0.5, 0.2), (1, 2.0, 0.2), (2, 1.0, 0.2)])
    assert path.read_text().splitlines()[0] == "n,t_as,t_ls"
    n, t_as, t_ls = lrb.read_curves_csv(path)
    assert n.tolist() == [1, 2, 4] and t_as.tolist() == [2.0, 1.0, 0.5] and t_ls.tolist() == [0.2] * 3
    with pytest.raises(ValueError, match="n = 1"):
        lrb.write_curves_csv(path, [(2, 1.0, 1.0)])
    with pytest.raises(ValueError, match="positive"):
        lrb.write_curves_csv(path, [(1, 0.0, 1.0)])


def test_dump_fixtures():
    """Known answers of the reference's tests/test_repart.py:297-313 (W1 chain,
    4 ranks, alpha 2): the sparsity dump of rank 1 and the scatter-map dump."""
    _, _, assembled, pm = chain_setup(4, 8, 2)
    sp = lrb.extract_sparsity(*assembled[1], pm, 1)
    assert lrb.dump_sparsity(sp) == ("rows 2 4\n"
                                     "local 2 2\nlocal 2 3\nlocal 3 2\nlocal 3 3\n"
                                     "nonlocal 2 1\nnonlocal 3 4\n")
    received = [lrb.extract_sparsity(*assembled[r], pm, r) for r in (0, 1)]
    local, nonlocal_ = lrb.fuse_patterns(received, pm, 0)
    sm = lrb.build_scatter_map(received, local, nonlocal_, pm)
    lines = lrb.dump_scatter(sm).splitlines()
    assert len(lines) == 11
    assert lines[0] == "0 -> local 0" and lines[10] == "10 -> nonlocal 0"
    for b, line in enumerate(lines):
        dest = "local" if sm.to_local[b] else "nonlocal"
        assert line == f"{b} -> {dest} {sm.index[b]}"
