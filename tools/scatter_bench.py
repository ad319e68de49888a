#!/usr/bin/env python
"""Scatter (apply_scatter, update.py:105-112) timing on one B200.

    python tools/scatter_bench.py [--n 200] [--ranks 8] [--alpha 8] [--reps 20]

Prints one JSON line: device time of each part's whole-part scatter (CUDA
events on the part's stream; owner threads run concurrently, so with several
parts per GPU the per-part figures overlap) and algorithmic GB/s (20 B per
entry), plus a digest of the scattered values.  Under ncu, the first
``n_cpu`` scatter launches are the update's per-segment ones; the whole-part
launches follow (``--launch-skip n_cpu``).
"""
import argparse
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(args):
    import numpy as np
    import torch

    import bench
    import paper_2510_08536_b200 as lrb

    torch.cuda.set_device(0)
    prob = bench.Problem(args.n, args.ranks, range(args.ranks))
    pm = lrb.make_partition_map(prob.cells, args.alpha)
    out = {}

    def program(ctx):
        r = ctx.rank
        s = lrb.repartition(*prob.base[r], pm, ctx)
        lrb.update(s, *prob.produce(r, 3), "direct")
        ctx.barrier()
        if not s.is_owner:
            return None
        part = s.part
        part.sync()
        ms = []
        for i in range(args.reps + 3):
            t = part.apply_scatter_timed()
            if i >= 3:
                ms.append(t)
        part.sync()
        vals = s.matrix.local.vals
        return part.n_buf, ms, hashlib.sha256(vals.tobytes()).hexdigest()[:16]

    res = [x for x in lrb.run_world(args.ranks, program) if x is not None]
    n_buf = sum(r[0] for r in res)
    # parts are scattered one after another by their owner threads: report per part
    per = [float(np.median(r[1])) for r in res]
    out = {"parts": len(res),
           "ms_per_part": [round(x, 4) for x in per],
           "gbs_per_part": [round(20 * r[0] / (t * 1e-3) / 1e9, 1) for r, t in zip(res, per)],
           "entries": n_buf, "digest": [r[2] for r in res]}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200)
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--alpha", type=int, default=8)
    ap.add_argument("--reps", type=int, default=20)
    child(ap.parse_args())


if __name__ == "__main__":
    main()
