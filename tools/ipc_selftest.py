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
    t0 = time.time()
    xs, rep, hist = owner.solve("pcg", [np.ones(p.n) for p in owner.parts], 1e-9, 500,
                                hist_cap=500)
    dt = time.time() - t0
    xs_all = allgather_obj((rank, [x.copy() for x in xs], rep.iterations, list(hist)))
    if rank == 0:
        with open(out, "w") as fh:
            json.dump({"iterations": rep.iterations, "seconds": dt,
                       "x": [np.concatenate([np.concatenate(v[1]) for v in sorted(xs_all)]).tolist()],
                       "hist": list(hist)}, fh)
    dist.barrier()
    dist.destroy_process_group()


def main():
    sys.path.insert(0, ROOT)
    out = os.path.join(ROOT, "gpurun_out", "ipc_selftest.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    mp.spawn(worker, args=(2, _port(), out), nprocs=2, join=True)
    res = json.load(open(out))
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
