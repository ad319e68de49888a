"""World-size-2 gloo tests of the multi-process (one process per GPU) host logic.

Runs on CPU: each process builds its owner plans natively (no GPU needed),
publishes its halo description over torch.distributed and checks that the
device halo tables (hpart/hidx, read straight from peer memory by the solve
kernels) equal the reference's send lists (solver.py:48-77, golden fixtures),
that blob exchange preserves rank order, and that timings reduce to the max.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out_dir):
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from golden_cases import get, matches
        from helpers_b200 import golden_inputs
        from paper_2510_08536_b200.dist import (ProcessLayout, allgather_bytes, allgather_obj,
                                                 halo_pairs, max_over_ranks)
        from paper_2510_08536_b200.repart import _owner_plan, _Source
        pm_all, per_rank = golden_inputs(case)
        lay = ProcessLayout(np.diff(pm_all.offsets), pm_all.alpha, world, rank)
        assert lay.cpu_ranks == list(range(lay.part_begin * pm_all.alpha,
                                           (lay.part_begin + lay.parts_per_proc) * pm_all.alpha))
        plans = {}
        for k in lay.parts:
            srcs = [_Source(*per_rank[r], lay.pm, r) for r in range(lay.pm.alpha * k,
                                                                     lay.pm.alpha * (k + 1))]
            plans[k] = _owner_plan(srcs, lay.pm, k)
        mine = {k: p.csr()[4] for k, p in plans.items()}
        halo = {}
        for d in allgather_obj(mine):
            halo.update(d)
        send = halo_pairs(lay, halo)
        ok = True
        for k, p in plans.items():
            hp, hi = p.halo_owners()
            for j in np.unique(hp):
                ok &= bool(np.array_equal(hi[hp == j], send[(int(j), k)]))
            # against the reference's own recv/send lists
            rnb = get(case, k, "halo_recv_nbrs")
            if rnb is not None:
                assert sorted(set(hp.tolist())) == rnb.tolist()
                snb = get(case, k, "halo_send_nbrs")
                cat = np.concatenate([send[(k, g)] for g in snb]) if len(snb) else \
                    np.zeros(0, np.int64)
                ok &= bool(matches(case, k, "halo_send_idx", cat))
        blobs = allgather_bytes(bytes([rank]) * 512)
        ok &= [b[0] for b in blobs] == list(range(world))
        ok &= max_over_ranks(float(rank) + 0.5) == world - 0.5
        with open(os.path.join(out_dir, f"r{rank}.txt"), "w") as fh:
            fh.write("ok" if ok else "FAIL")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["cav12x12x12_r8_a2", "cav12x12x12_r8_a1", "c2"])
def test_two_process_halo_tables_match_reference(case, tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert (tmp_path / f"r{r}.txt").read_text() == "ok"
