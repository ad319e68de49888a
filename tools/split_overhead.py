"""Cost of the cross-device team protocol, measured on ONE GPU.

    python tools/split_overhead.py [--n 200] [--ranks 8]

The same parts (n^3 cavity, ``ranks`` sources, alpha 1 -> ``ranks`` parts)
solved (Jacobi-PCG, timestep 2) by one team kernel, and by teams whose parts
are split into 2 / 4 / 8 "device ranks": separate kernels, each on its share
of the SMs, meeting at every team barrier through the peer-flag protocol with
halo values pushed into the readers' mirrors — the multi-GPU data path minus
the NVLink latency.  Iterates are bit-identical across the splits
(tests/test_gpu_halo.py), so the time difference is the protocol's cost.
Prints one JSON line per split with the solve's device time and its per-
iteration phase-release statistics."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import MAX_ITER, TOL, Problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200)
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--repeat", type=int, default=3)
    ap.add_argument("--method", default="pcg")
    args = ap.parse_args()
    import paper_2510_08536_b200 as lrb
    from paper_2510_08536_b200.device import Team
    prob = Problem(args.n, args.ranks, range(args.ranks))
    pm = lrb.make_partition_map(prob.cells, 1)
    holder = {}

    def program(ctx):
        s = lrb.repartition(*prob.base[ctx.rank], pm, ctx)
        lrb.update(s, *prob.produce(ctx.rank, 2), "direct")
        parts = s.comm.allgather(s.part)
        if s.comm.group_rank == 0:
            holder["parts"] = parts
        holder.setdefault("keep", []).append(s)
        return None

    lrb.run_world(args.ranks, program)
    parts = holder["parts"]
    for p in parts:
        p.sync()
    n_parts = len(parts)
    bs = [np.ones(p.n) for p in parts]
    ref_x = None
    for split in (1, 2, 4, 8):
        if split > n_parts:
            continue
        ranks = [i * split // n_parts for i in range(n_parts)]
        team = Team(parts, dev_ranks=ranks)
        team.profile(4 * MAX_ITER)
        ms, its = [], None
        for _ in range(args.repeat):
            xs, rep, hist = team.solve(args.method, bs, TOL, MAX_ITER, hist_cap=MAX_ITER)
            ms.append(rep.device_ms)
            its = rep.iterations
        ts = team.phase_times_ns().reshape(-1, 2)
        sync_us = (ts[1:, 1] - ts[1:, 0]) / 1e3
        if ref_x is None:
            ref_x = xs
        same = all(np.array_equal(a, b) for a, b in zip(xs, ref_x))
        print(json.dumps({"method": args.method, "device_ranks": split, "kernels": split,
                          "ctas_per_kernel": team.kernel_info(args.method)["grid"],
                          "iterations": its, "solve_ms": round(float(np.median(ms)), 4),
                          "us_per_iteration": round(float(np.median(ms)) * 1e3 / its, 2),
                          "barrier_last_arrival_to_release_us": round(float(np.median(sync_us)), 2),
                          "bit_identical_to_one_kernel": same}), flush=True)
        del team


if __name__ == "__main__":
    main()
