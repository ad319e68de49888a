"""CPU tests of the collective context (the drop-in's World) and host logic."""

import numpy as np
import pytest

import paper_2510_08536_b200 as lrb
from helpers_b200 import chain_setup


def test_send_recv_and_ordered_allreduce():
    def program(ctx):
        v = ctx.allreduce_sum(float(ctx.rank) + 0.1)
        g = ctx.allgather(ctx.rank * 10)
        if ctx.rank == 0:
            ctx.send(1, np.arange(3.0))
        if ctx.rank == 1:
            return v, g, ctx.recv(0).tolist()
        return v, g, None

    res = lrb.run_world(4, program)
    expect = ((0.1 + 1.1) + 2.1) + 3.1
    assert all(r[0] == expect for r in res)
    assert res[1][1] == [0, 10, 20, 30] and res[1][2] == [0.0, 1.0, 2.0]


def test_split_active_group_ranks():
    _, _, asm, pm = chain_setup(4, alpha=2)

    def program(ctx):
        c = lrb.split_active(ctx, pm)
        return c.tag, c.group_rank, c.members

    res = lrb.run_world(4, program)
    assert res[0] == ("active", 0, (0, 2)) and res[2] == ("active", 1, (0, 2))
    assert res[1] == ("inactive", 0, (1, 3))


def test_mismatched_collective_participation_deadlocks():
    _, _, asm, pm = chain_setup(4, alpha=2)

    def program(ctx):
        sp = lrb.extract_sparsity(*asm[ctx.rank], pm, ctx.rank)
        if ctx.rank == 3:
            return None
        return len(lrb.exchange_patterns(sp, pm, ctx))

    with pytest.raises(lrb.DeadlockError):
        lrb.run_world(4, program)


def test_exchange_patterns_order():
    _, _, asm, pm = chain_setup(4, alpha=2)

    def program(ctx):
        sp = lrb.extract_sparsity(*asm[ctx.rank], pm, ctx.rank)
        return [(p.row_lo, p.row_hi) for p in lrb.exchange_patterns(sp, pm, ctx)]

    res = lrb.run_world(4, program)
    assert res == [[(0, 2), (2, 4)], [], [(4, 6), (6, 8)], []]


def test_rank_failure_is_attributed():
    def program(ctx):
        if ctx.rank == 2:
            raise ValueError("boom")
        ctx.barrier()

    with pytest.raises(lrb.RankFailedError) as err:
        lrb.run_world(3, program)
    assert err.value.rank == 2 and "boom" in str(err.value.cause)


def test_leader_call_delivers_results_and_errors():
    def program(ctx):
        c = ctx.comm
        out = c.leader_call(ctx.rank, lambda items: [sum(items) + i for i in range(len(items))])
        try:
            c.leader_call(ctx.rank, lambda items: 1 / 0)
        except ZeroDivisionError:
            return out
        return None

    assert lrb.run_world(3, program) == [3, 4, 5]


def test_update_pattern_and_packing():
    pm = lrb.make_partition_map([1] * 6, 3)
    up = lrb.build_update_pattern(pm, [7] * 6)
    assert up.recv_offsets[0].tolist() == [0, 7, 14, 21]
    _, _, asm, _ = chain_setup(4)
    assert lrb.pack_coefficients(*asm[1], 1).values.tolist() == [2, 2, -1, -1, -1, -1]
    m1, if1 = lrb.perturb_coefficients(*asm[1], 1)
    assert lrb.pack_coefficients(m1, if1, 1).values.tolist() == [2.02, 2.02, -1, -1, -1, -1]
    rev = list(reversed(asm[1][1]))
    assert lrb.pack_coefficients(asm[1][0], rev, 1).values.tolist() == \
        lrb.pack_coefficients(*asm[1], 1).values.tolist()
