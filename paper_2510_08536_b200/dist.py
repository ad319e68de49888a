"""One process per GPU (torchrun): host orchestration of the multi-GPU path.

Process g owns GPU part(s) ``parts_per_proc*g ..`` and hosts their CPU source
ranks as threads.  ``torch.distributed`` (gloo, CPU) carries only create-time
plumbing — IPC blobs, halo descriptions — and the max-over-ranks of timings.
The data path (halo values, partial dot products) never touches NCCL: the
persistent solve kernels read neighbour vectors and exchange dot partials
through NVLink peer memory (csrc/kernels.cuh team_sync).

No update traffic crosses GPUs: a source's segment goes only to its owner
(repart.py:239-250), so ``update`` is process-local.
"""

from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .core import PartitionMap, make_partition_map
from .device import DevicePart, Team, device_count
from .repart import _owner_plan, _pieces, _Source, sparsity_fingerprint


class ProcessLayout:
    """Which GPU parts and CPU ranks live in process ``rank`` of ``world``."""

    def __init__(self, cells_per_rank, alpha: int, world: int, rank: int):
        self.pm: PartitionMap = make_partition_map(cells_per_rank, alpha)
        if self.pm.n_gpu % world:
            raise ValueError(f"{self.pm.n_gpu} GPU parts cannot be split over {world} processes")
        self.world, self.rank = world, rank
        self.parts_per_proc = self.pm.n_gpu // world
        self.part_begin = rank * self.parts_per_proc
        self.parts = list(range(self.part_begin, self.part_begin + self.parts_per_proc))
        a = self.pm.alpha
        self.cpu_ranks = list(range(self.part_begin * a, (self.part_begin + self.parts_per_proc) * a))

    def owner_of(self, cpu_rank: int) -> int:
        return cpu_rank // self.pm.alpha


def allgather_bytes(blob: bytes, group=None):
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, blob, group=group)
    return out


def allgather_obj(obj, group=None):
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


def plumbing_backend(world: int) -> str:
    """Process-group backend for the plumbing (blobs, barriers, timing): NCCL
    when every process has a GPU of its own (one process per GPU over NVLink),
    gloo when processes share a GPU (NCCL refuses duplicate devices) or there
    is no GPU (CPU tests)."""
    import torch
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    return "nccl" if n >= world > 1 else "gloo"


def init_plumbing(world: int, local_rank: int) -> str:
    """init_process_group for the multi-process path; returns the backend."""
    import torch
    import torch.distributed as dist
    backend = plumbing_backend(world)
    if backend == "nccl":
        dev = torch.device("cuda", local_rank)
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    return backend


def _dev():
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def max_over_ranks(value: float, group=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def halo_pairs(layout: ProcessLayout, halo_by_part):
    """Reference halo plan semantics across processes (solver.py:48-77):
    for every ordered pair (owner j -> needer k) the rows j sends, from the
    halo columns every part published.  Used by the tests to check the device
    halo tables (hpart/hidx) against the reference's send lists."""
    pm = layout.pm
    go = pm.gpu_offsets
    send = {}
    for k, halo in halo_by_part.items():
        owners = pm.col_owner_gpu(np.asarray(halo, dtype=np.int64))
        for j in np.unique(owners):
            send[(int(j), int(k))] = np.asarray(halo, np.int64)[owners == j] - go[j]
    return send


class DistributedOwner:
    """This process's owner part(s) and source ranks: create once, then
    update + solve per timestep through the C ABI with host buffers."""

    def __init__(self, layout: ProcessLayout, problems, group=None, n_threads=0, solve=True):
        """``problems``: {cpu_rank: (LduMatrix, [InterfaceBlock])} for this process.
        ``solve=False``: update-only owner (no solve team is connected)."""
        self.layout = layout
        pm = layout.pm
        self.fingerprints = {r: sparsity_fingerprint(*problems[r]) for r in layout.cpu_ranks}
        dev = (layout.rank % device_count())
        self.parts = []
        self.plans = []
        for k in layout.parts:
            srcs = [_Source(*problems[r], pm, r) for r in range(pm.alpha * k, pm.alpha * (k + 1))]
            plan = _owner_plan(srcs, pm, k)
            self.plans.append(plan)
            self.parts.append(DevicePart(plan, dev))
        self.team = None if not solve else Team.across_processes(self.parts, layout.part_begin, pm.n_gpu, layout.rank,
                                          layout.world, lambda b: allgather_bytes(b, group))
        self.pool = ThreadPoolExecutor(max(1, len(layout.cpu_ranks)))
        self.update(problems, "direct")

    def _batched(self, problems):
        """Direct update of each part's sources with one native call per part
        (lrb_update_segments), when every piece is pinned: no per-source
        Python in the update (C5 hosts 16 sources per part).  False: some
        piece is pageable, the per-source threads do it."""
        pm = self.layout.pm
        for r in self.layout.cpu_ranks:
            if sparsity_fingerprint(*problems[r]) != self.fingerprints[r]:
                raise RuntimeError(f"pattern drift on rank {r}")
        def one_part(i):
            k = self.layout.parts[i]
            ranks = range(pm.alpha * k, pm.alpha * (k + 1))
            return self.parts[i].update_segments([r % pm.alpha for r in ranks],
                                                 [_pieces(*problems[r]) for r in ranks])

        # parts in parallel (one host thread per part), sources of a part batched
        return all(list(self.pool.map(one_part, range(len(self.parts)))))

    def update(self, problems, mode="direct"):
        """Every local source rank copies its segment (threads; GIL released in C)."""
        pm = self.layout.pm

        def one(r):
            m, ifs = problems[r]
            if sparsity_fingerprint(m, ifs) != self.fingerprints[r]:
                raise RuntimeError(f"pattern drift on rank {r}")
            part = self.parts[self.layout.owner_of(r) - self.layout.part_begin]
            if mode == "direct":
                part.update_segment(r % pm.alpha, _pieces(m, ifs))
            else:
                part.stage_segment(r % pm.alpha, _pieces(m, ifs))

        if mode == "direct" and self._batched(problems):
            pass   # every part's sources in one native call each (pinned inputs)
        else:
            list(self.pool.map(one, self.layout.cpu_ranks))
        for p in self.parts:
            if mode == "direct":
                p.join()
            else:
                p.update_staged_from_stage()

    def solve(self, method, b_local, tol, max_iter, hist_cap=0, group=None):
        """One solve of the whole team.  A process barrier first bounds the launch
        skew between processes, so the kernels' cross-device barrier timeout
        (LRB_BARRIER_TIMEOUT_S) measures a missing peer, not a late launch."""
        import torch.distributed as dist
        if self.layout.world > 1:
            dist.barrier(group)
        bs = [None] * self.layout.pm.n_gpu
        for i, k in enumerate(self.layout.parts):
            bs[k] = b_local[i] if b_local is not None else None
        xs, rep, hist = self.team.solve(method, None if b_local is None else bs, tol, max_iter,
                                        want_x=True, hist_cap=hist_cap)
        return [xs[k] for k in self.layout.parts], rep, hist
