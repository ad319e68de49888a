"""Verification helpers on the real device parts: the
owners' fused parts gathered into one global COO equal the global matrix the
ranks assembled (random partitioned systems, non-symmetric values), and a
Matrix Market export of it round-trips."""

import numpy as np
import pytest

import paper_2510_08536_b200 as lrb
from test_api_cpu import random_system

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [3, 8, 21])
def test_gather_global_is_the_assembled_matrix(seed, tmp_path):
    pm, per_rank, values = random_system(np.random.default_rng(seed))

    def program(ctx):
        s = lrb.repartition(*per_rank[ctx.rank], pm, ctx)
        if s.is_owner:
            return lrb.gather_global(s.matrix, pm, s.comm)
        return None

    res = lrb.run_world(len(per_rank), program)
    g = res[0]
    assert all(r is None for r in res[1:])
    got = {(int(i), int(j)): v for i, j, v in zip(g.rows, g.cols, g.vals)}
    assert got == values
    lrb.write_matrix_market(g, tmp_path / "g.mtx")
    back = lrb.read_matrix_market(tmp_path / "g.mtx")
    np.testing.assert_array_equal(back.vals, g.vals)
