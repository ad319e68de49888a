"""Two processes sharing ONE GPU run the multi-process (CUDA IPC) team path.

    timeout 180 python tools/ipc_selftest.py

Process g owns GPU part g of a 16^3 cavity (4 ranks, alpha 2) on cuda:0; the
solve kernels of the two processes synchronise through the peer-memory flag
protocol exactly as on separate GPUs (contexts time-slice, so it is slow but
must be bit-identical to the single-process team).  Prints one JSON line.
"""
import json
import os
import socket
import sys
import time

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DIMS, NCPU, ALPHA = (16, 16, 16), 4, 2


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2510_08536_b200 as lrb
    from paper_2510_08536_b200.dist import DistributedOwner, ProcessLayout, allgather_obj
    parts = lrb.decompose_slab(lrb.StructuredGrid(*DIMS), NCPU)
    lay = ProcessLayout([p.n_cells for p in parts], ALPHA, world, rank)
    probs = {r: lrb.assemble_poisson(parts[r]) for r in lay.cpu_ranks}
    owner = DistributedOwner(lay, probs)
    for p in owner.parts:
        p.sync()
    dist.barrier()
    # 1) peer pointers: read the OTHER process's part (dinv = 1/diag after the
    #    initial scatter) through this process's team table (CUDA IPC mapping)
    other = 1 - rank
    n_other = parts[2 * other].n_cells + parts[2 * other + 1].n_cells
    diag = np.concatenate([lrb.assemble_poisson(parts[r])[0].diag for r in (2 * other, 2 * other + 1)])
    got = owner.team.read_vector(other, "dinv", n_other)
    peer_ok = bool(np.array_equal(got, 1.0 / diag))
    print(f"[rank {rank}] peer read ok={peer_ok}", file=sys.stderr, flush=True)
    dist.barrier()
    t0 = time.time()
    try:
        xs, rep, hist = owner.solve("pcg", [np.ones(p.n) for p in owner.parts], 1e-9, 500,
                                    hist_cap=500)
        err = None
    except Exception as exc:  # noqa: BLE001
        xs, rep, hist, err = [np.zeros(p.n) for p in owner.parts], None, [], repr(exc)
        print(f"[rank {rank}] solve failed: {err}; barrier state {owner.team.debug(world)}",
              file=sys.stderr, flush=True)
    dt = time.time() - t0
    mine = {"rank": rank, "peer_ok": peer_ok, "error": err, "seconds": dt,
            "debug": owner.team.debug(world).tolist(),
            "iterations": None if rep is None else rep.iterations,
            "x": np.concatenate(xs).tolist(), "hist": [float(h) for h in hist]}
    every = sorted(allgather_obj(mine), key=lambda d: d["rank"])
    if rank == 0:
        res = {"ranks": [{k: v for k, v in d.items() if k not in ("x", "hist")} for d in every],
               "peer_ok": all(d["peer_ok"] for d in every),
               "error": next((d["error"] for d in every if d["error"]), None),
               "iterations": every[0]["iterations"], "seconds": max(d["seconds"] for d in every),
               "x": [sum((d["x"] for d in every), [])], "hist": every[0]["hist"]}
        with open(out, "w") as fh:
            json.dump(res, fh)
    dist.barrier()
    dist.destroy_process_group()


def main():
    sys.path.insert(0, ROOT)
    out = os.path.join(ROOT, "gpurun_out", "ipc_selftest.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    mp.spawn(worker, args=(2, _port(), out), nprocs=2, join=True)
    res = json.load(open(out))
    if res.get("error"):
        print(json.dumps({k: v for k, v in res.items() if k not in ("x", "hist")}))
        sys.exit(2)
    # single-process reference run of the same team
    import paper_2510_08536_b200 as lrb
    parts = lrb.decompose_slab(lrb.StructuredGrid(*DIMS), NCPU)
    asm = [lrb.assemble_poisson(p) for p in parts]
    pm = lrb.make_partition_map([p.n_cells for p in parts], ALPHA)

    def program(ctx):
        s = lrb.repartition(*asm[ctx.rank], pm, ctx)
        if not s.is_owner:
            return None
        x, rep = lrb.cg_solve(s.matrix, s.halo, np.ones(s.matrix.n_owned), 1e-9, 500, s.comm,
                              method="pcg", history=True)
        pieces = s.comm.gather(x, 0)
        return (np.concatenate(pieces), rep) if pieces is not None else None

    x1, rep1 = lrb.run_world(NCPU, program)[0]
    same = bool(np.array_equal(np.asarray(res["x"][0]), x1)) and res["iterations"] == rep1.iterations
    print(json.dumps({"ipc_iterations": res["iterations"], "single_iterations": rep1.iterations,
                      "bit_identical": same, "ipc_seconds": res["seconds"]}))
    sys.exit(0 if same else 1)


if __name__ == "__main__":
    main()
