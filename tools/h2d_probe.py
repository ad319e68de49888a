"""Probe: host->device copy bandwidth on this box and through the update path.

    python tools/h2d_probe.py            (GPU box)
"""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def bw(nbytes, s):
    return nbytes / s / 1e9


def main():
    n = 56_000_000  # 446 MB of doubles (C3, 1 GPU)
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h.numpy()[:] = 1.0
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    print(f"torch pinned H2D 1 stream: {bw(5 * 8 * n, time.perf_counter() - t):.1f} GB/s")
    # 8 concurrent streams
    chunks = 8
    streams = [torch.cuda.Stream() for _ in range(chunks)]
    m = n // chunks
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * m:(i + 1) * m].copy_(h[i * m:(i + 1) * m], non_blocking=True)
    torch.cuda.synchronize()
    print(f"torch pinned H2D 8 streams: {bw(5 * 8 * m * chunks, time.perf_counter() - t):.1f} GB/s")
    pg = np.ones(n)
    t = time.perf_counter()
    d.copy_(torch.from_numpy(pg))
    torch.cuda.synchronize()
    print(f"torch pageable H2D: {bw(8 * n, time.perf_counter() - t):.1f} GB/s")
    t = time.perf_counter()
    h.numpy()[:] = pg
    print(f"host memcpy pageable->pinned 1 thread: {bw(8 * n, time.perf_counter() - t):.1f} GB/s")

    # through the drop-in update path (C3, 8 ranks -> 1 GPU)
    import paper_2510_08536_b200 as lrb
    from bench import Problem
    prob = Problem(200, 8, range(8))
    pm = lrb.make_partition_map(prob.cells, 8)
    times = []

    def program(ctx):
        r = ctx.rank
        s = lrb.repartition(*prob.base[r], pm, ctx)
        for step in range(2, 8):
            m, ifs = prob.produce(r, step)
            ctx.barrier()
            t0 = time.perf_counter()
            lrb.update(s, m, ifs, "direct")
            if s.is_owner:
                s.part.sync()
                times.append(time.perf_counter() - t0)
        if s.is_owner:
            return s.part.stats()

    res = lrb.run_world(8, program)
    nb = res[0]["h2d_bytes"] / 7
    print("update stats", res[0])
    print("update direct ms:", [round(1e3 * x, 2) for x in times],
          f"-> {bw(nb, np.median(times)):.1f} GB/s effective")

    # single-thread segment copies without the world
    part = None


if __name__ == "__main__":
    main()
