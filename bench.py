#!/usr/bin/env python
"""Benchmark: ms per timestep (matrix update + Krylov solve) on B200.

Workload (BASELINE.json configs[2], "C3"): 3D cavity 200^3 (8M cells),
``--rpg`` CPU assembly ranks per GPU (default 8) repartitioned onto N GPUs,
pressure Jacobi-PCG to 1e-6 with b = ones.  Timed window = timesteps
2..K+1 of the reference protocol (cli.py:181-272: step 1 is the creation
step and is excluded; cli.py:109-114), whatever ``--warmup`` is: the W
warm-up steps replay timestep 2 without advancing the physical timestep.
One timestep = update (all coefficients of every rank: H2D + gather-permute)
+ solve.  Every solve starts from x0 = 0 (solver.py:119), so a replayed step
is the same work as the first.

* ``value``  device-resident: coefficients already in the receive buffer in
  HBM, b resident; timed = scatter kernel + solve kernel (CUDA events).
* ``e2e``    through the public API (``update`` from pinned host LDU arrays by
  every rank thread, then ``cg_solve`` with b from host and x back to host).
  ``e2e_pageable``: the same with the reference generator's own pageable
  ``perturb_coefficients`` output (host copy into the pinned stage counted).
* ``--impl reference``: the UNMODIFIED reference package (``baseline/_ref``,
  pip-installed from /root/reference) on the host cores, the cli.run_case
  protocol with full solves on every timed step (no projection).

Other workloads: ``c1``/``c2`` (latency-bound sizes), ``c4`` (300^3 full
timestep: momentum update + 3 BiCGStab + pressure update + Jacobi-PCG) and
``c5`` (update-only stress: 200^3, 128 ranks -> 8 parts, alpha 16).

Inputs (1.5 GB PCG working set at N=1) are larger than L2, so no L2 flush is
needed between timed steps.
"""

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _impl_from_argv():
    for i, a in enumerate(sys.argv):
        if a == "--impl" and i + 1 < len(sys.argv):
            return sys.argv[i + 1]
        if a.startswith("--impl="):
            return a.split("=", 1)[1]
    return "ours"


# Set before numpy loads.  Our host side is C++ threads + CUDA (BLAS unused).
# The reference arm runs its fastest configuration: single-threaded OpenBLAS.
# Threaded dots were measured SLOWER for it (C1: 425 vs 45 ms/timestep with 8
# threads in the build container) and its SpMV (np.add.at, 92% of an
# iteration) and one-rank-at-a-time scheduler are single-core anyway.
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

sys.path.insert(0, ROOT)

METRIC = "ms/timestep (matrix update + CG solve) at 1/2/4/8 B200; % of HBM roofline"
WORKLOADS = {
    # name: (N, default rpg, method, description)
    "c3": (200, 8, "pipecg", "C3: 3D cavity 200^3 (8M cells), {n_cpu} CPU ranks -> {n_gpu} GPU(s) "
                             "(alpha {alpha}), pressure Jacobi-PCG (pipelined) to 1e-6, b=ones"),
    "c2": (100, 8, "pipecg", "C2: 3D cavity 100^3 (1M cells), {n_cpu} CPU ranks -> {n_gpu} GPU(s) "
                             "(alpha {alpha}), Jacobi-PCG (pipelined) to 1e-6"),
    # Jacobi-PCG in its pipelined form (one SpMV phase and one barrier per
    # iteration): the fastest solver at C1/C2, level with two-phase PCG at C3
    # (7.03 vs 7.06 ms/timestep) with half the team barriers — the ones that
    # cross NVLink on N > 1 GPUs.  At C3 its histories sit within 3.9e-11 of
    # the reference's CG logs with the same iteration counts
    # (tests/test_gpu_large.py).  --method pcg for the two-phase kernel; C4
    # keeps it for the pressure solve.
    "c1": (32, 4, "pipecg", "C1: 3D cavity 32^3, {n_cpu} CPU ranks -> {n_gpu} device(s) "
                            "(alpha {alpha}), Jacobi-PCG (pipelined) to 1e-6"),
    "c4": (300, 16, "pcg", "C4: 3D cavity {N}^3 ({cells} cells), {n_cpu} CPU ranks -> {n_gpu} GPU(s) "
                           "(alpha {alpha}), full timestep: momentum update + 3 BiCGStab (Ux, Uy, Uz) "
                           "+ pressure update + Jacobi-PCG, all to 1e-6"),
    "c5": (200, 16, None, "C5: value-update-only stress, 3D cavity 200^3 (8M cells), 128 CPU ranks -> "
                          "8 parts (alpha 16, 16 segments per part) on {n_gpu} GPU(s)"),
}
C5_RANKS = 128
TOL, MAX_ITER = 1e-6, 2000
PCIE_PINNED_GBS = 55.6     # measured pinned H2D on the pool's B200 boxes (tools/h2d_probe.py)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def step_plan(args):
    """(warm-up steps, timed steps): W replays of timestep 2, then 2..K+1."""
    return [2] * args.warmup, list(range(2, 2 + args.steps))


def gpus_used(args):
    """GPUs this run really uses: one process per GPU under torchrun; a
    single process (no torchrun) places every part on cuda:0, whatever
    --gpus says (its parts then emulate the GPU partition on one device)."""
    _, world, _ = dist_env()
    return world if world > 1 else 1


def timesteps_label(args):
    return f"2..{1 + args.steps}"


def warmup_label(args):
    return f"{args.warmup} replays of timestep 2 (the physical timestep does not advance)"


def host_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model,
            "openblas_num_threads": os.environ.get("OPENBLAS_NUM_THREADS")}


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:  # noqa: BLE001 - clocks are best effort
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[3:7])
                          if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def gpu_index(local_rank=0):
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    ids = [v for v in vis.split(",") if v.strip()]
    if ids and ids[local_rank % len(ids)].strip().isdigit():
        return int(ids[local_rank % len(ids)])
    return local_rank


# ---------------------------------------------------------------------------
# roofline accounting
# ---------------------------------------------------------------------------
def solve_bytes(n, nnz, h, iterations, checks, method):
    """Algorithmic HBM bytes of one solve: CG it 12nnz+4(n+1)+88n+8h, PCG +16n,
    true-residual check 12nnz+4(n+1)+16n+8h, init (b read, x r written) 24n.
    pcg1 (single reduction): it 12nnz+4(n+1)+8h + 88n (r, dinv, w, s_old and
    p, x read; p, x, r, s, w written), init + one SpMV 12nnz+4(n+1)+24n+8h.
    pipecg (pipelined): it 12nnz+4(n+1)+8h + 104n (w, dinv, z, s, p, x, r read;
    z, s, p, x, r, w written), init as pcg1 (the final x copy, 16n when the
    last iterate sits in the second buffer, is not counted)."""
    chk = 12 * nnz + 4 * (n + 1) + 16 * n + 8 * h
    if method == "pipecg":
        it = 12 * nnz + 4 * (n + 1) + 104 * n + 8 * h
        return iterations * it + checks * chk + 24 * n + 12 * nnz + 4 * (n + 1) + 24 * n + 8 * h
    if method == "pcg1":
        it = 12 * nnz + 4 * (n + 1) + 88 * n + 8 * h
        return iterations * it + checks * chk + 24 * n + 12 * nnz + 4 * (n + 1) + 24 * n + 8 * h
    it = 12 * nnz + 4 * (n + 1) + 88 * n + 8 * h + (16 * n if method == "pcg" else 0)
    return iterations * it + checks * chk + 24 * n


def bicgstab_bytes(n, nnz, h, iterations, checks):
    """Algorithmic bytes of one BiCGStab solve: per iteration
    2(12nnz+4(n+1)+8h)+152n, true-residual checks as CG, init 40n."""
    it = 2 * (12 * nnz + 4 * (n + 1) + 8 * h) + 152 * n
    chk = 12 * nnz + 4 * (n + 1) + 16 * n + 8 * h
    return iterations * it + checks * chk + 40 * n


def n_checks(history, iterations, tol):
    c = 0
    for it in range(1, iterations + 1):
        rec = history[it - 1] if it - 1 < len(history) else 0.0
        if rec <= tol or it % 10 == 0:
            c += 1
    return c


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def traffic_ratio(workload):
    """ncu DRAM bytes per algorithmic byte of a workload's dominant kernel
    (profiles/traffic.json, from one ncu --set full capture)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh).get(workload)
    except Exception:  # noqa: BLE001
        return None


# ---------------------------------------------------------------------------
# problem
# ---------------------------------------------------------------------------
class Problem:
    """Per-rank LDU inputs whose value arrays live in pinned host memory.

    Producer layout (the producer writes straight into pinned
    buffers in pack order): the value arrays of the ``group`` consecutive
    ranks that feed one GPU part are views into ONE pinned block, rank after
    rank, each as [diag | upper | lower | interface blocks by neighbour] —
    the reference's pack order (update.py:40-45) — so the update moves
    host-contiguous runs in few large copies.  The LduMatrix / InterfaceBlock
    objects handed to ``update`` are the reference's types as usual."""

    def __init__(self, N, n_cpu, ranks, pinned=True, group=1):
        import paper_2510_08536_b200 as lrb
        self.lrb = lrb
        grid = lrb.StructuredGrid(N, N, N)
        parts = lrb.decompose_slab(grid, n_cpu)
        self.cells = [p.n_cells for p in parts]
        self.base = {}
        self.live = {}
        for r in ranks:
            self.base[r] = lrb.assemble_poisson(parts[r])
            parts[r] = None   # drop the mesh (faces live on in the LDU matrix)
        if pinned:
            import torch
            ranks = sorted(self.base)
            blocks = {}
            for r in ranks:
                blocks.setdefault(r // group, []).append(r)
            for members in blocks.values():
                sizes = [self._pack_len(*self.base[r]) for r in members]
                flat = self._pin(torch, np.zeros(sum(sizes)))
                o = 0
                for r, n in zip(members, sizes):
                    self.live[r] = self._views(lrb, *self.base[r], flat[o:o + n])
                    o += n
        self.n_cells = grid.total_cells

    @staticmethod
    def _pack_len(m, ifs):
        return m.n_cells + 2 * m.n_faces + sum(len(b.values) for b in ifs)

    @staticmethod
    def _views(lrb, m, ifs, buf):
        """LduMatrix / InterfaceBlocks of the base values over buf, pack order."""
        n, f = m.n_cells, m.n_faces
        diag, upper, lower = buf[:n], buf[n:n + f], buf[n + f:n + 2 * f]
        diag[:], upper[:], lower[:] = m.diag, m.upper_val, m.lower_val
        mm = lrb.LduMatrix(m.n_cells, m.lower_addr, m.upper_addr, diag, lower, upper)
        o, ifp = n + 2 * f, []
        for b in sorted(ifs, key=lambda b: b.neighbor_rank):
            v = buf[o:o + len(b.values)]
            v[:] = b.values
            ifp.append(lrb.InterfaceBlock(b.neighbor_rank, b.rows, b.cols_remote, v))
            o += len(b.values)
        return mm, ifp, diag

    _pinned = []

    @classmethod
    def _pin(cls, torch, a):
        t = torch.empty(len(a), dtype=torch.float64, pin_memory=True)
        cls._pinned.append(t)          # keep the pinned tensor alive
        out = t.numpy()
        out[:] = a
        return out

    def produce(self, r, step):
        """Producer (outside the metric, like the reference's t_assemble):
        write step's diag into the pinned array of rank r."""
        m, ifs = self.base[r]
        mm, ifp, diag = self.live[r]
        self.lrb.perturb_diag_into(m.diag, step, diag)
        return mm, ifp

    def produce_pageable(self, r, step):
        """The reference generator's own output: fresh pageable numpy arrays
        (assembly.py:225-243), as a drop-in caller hands them to ``update``."""
        m, ifs = self.base[r]
        return self.lrb.perturb_coefficients(m, ifs, step)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch

    import paper_2510_08536_b200 as lrb
    from paper_2510_08536_b200 import _native

    rank, world, local_rank = dist_env()
    if args.workload == "c5":
        return run_c5(args)
    if world > 1:
        return run_ours_multi(args)
    if args.workload == "c4":
        return run_c4(args)
    N, _, method_default, desc = WORKLOADS[args.workload]
    method = args.method or method_default
    n_gpu = args.gpus
    n_cpu = args.rpg * n_gpu
    alpha = args.rpg
    torch.cuda.set_device(0)
    t0 = time.monotonic()
    prob = Problem(N, n_cpu, range(n_cpu), group=alpha)
    pm = lrb.make_partition_map(prob.cells, alpha)
    log(f"[bench] inputs {time.monotonic() - t0:.1f}s; n_cpu={n_cpu} alpha={alpha}")
    warm, timed = step_plan(args)
    seq = warm + timed
    W = len(warm)
    rec = {"e2e_ms": [], "wall_ms": [], "iters": [], "value_ms": [], "scatter_ms": [],
           "solve_ms": [], "kernel_ms": [], "checks": [], "launches": 0, "create_s": 0.0,
           "pg_ms": [], "pg_update_ms": []}
    sampler = ClockSampler(gpu_index())

    def program(ctx):
        r = ctx.rank
        m0, if0 = prob.base[r]
        tc = time.monotonic()
        system = lrb.repartition(m0, if0, pm, ctx)
        lrb.capture_device_base(system)   # the base coefficients, for the GPU-producer leg
        ctx.barrier()
        if r == 0:
            rec["create_s"] = time.monotonic() - tc
        b = Problem._pin(torch, np.ones(system.matrix.n_owned)) if system.is_owner else None
        # ---------------- e2e: public API, pinned host buffers ---------------
        for i, step in enumerate(seq):
            m_s, if_s = prob.produce(r, step)
            ctx.barrier()
            if r == 0:
                if i == W:
                    sampler.__enter__()
                    rec["l0"] = _native.lrb_launch_count()
                system.part.mark()
                tw = time.perf_counter()
            lrb.update(system, m_s, if_s, args.mode)
            tu = time.perf_counter()
            if system.is_owner:
                x, rep = lrb.cg_solve(system.matrix, system.halo, b, TOL, MAX_ITER, system.comm,
                                      method=method)
            if r == 0:
                system.part.mark()
                te = time.perf_counter()
                wall = (te - tw) * 1e3
                if i >= W:
                    rec["e2e_ms"].append(system.part.elapsed_ms())
                    rec["wall_ms"].append(wall)
                    rec["iters"].append(rep.iterations)
                    rec.setdefault("e2e_update_wall_ms", []).append((tu - tw) * 1e3)
                    rec.setdefault("e2e_solve_wall_ms", []).append((te - tu) * 1e3)
                    rec.setdefault("e2e_solve_kernel_ms", []).append(rep.device_ms)
                if i == len(seq) - 1:
                    rec["launches"] = _native.lrb_launch_count() - rec["l0"]
        ctx.barrier()
        if r == 0:
            sampler.__exit__()
        # ---------------- e2e, pageable drop-in inputs ------------------------
        if not args.no_pageable:
            for i, step in enumerate([2] + timed):
                m_s, if_s = prob.produce_pageable(r, step)
                ctx.barrier()
                if r == 0:
                    tw = time.perf_counter()
                lrb.update(system, m_s, if_s, args.mode)
                if system.is_owner:
                    tu = time.perf_counter()
                    x, rep = lrb.cg_solve(system.matrix, system.halo, b, TOL, MAX_ITER,
                                          system.comm, method=method)
                if r == 0 and i >= 1:
                    te = time.perf_counter()
                    rec["pg_ms"].append((te - tw) * 1e3)
                    rec["pg_update_ms"].append((tu - tw) * 1e3)
                del m_s, if_s
            ctx.barrier()
        # ---------------- e2e with the producer on the GPU ------
        for i, step in enumerate([2] + timed):
            ctx.barrier()
            if r == 0:
                system.part.mark()
                tw = time.perf_counter()
            lrb.update_on_device(system, step)
            if system.is_owner:
                x, rep = lrb.cg_solve(system.matrix, system.halo, b, TOL, MAX_ITER, system.comm,
                                      method=method)
            if r == 0:
                system.part.mark()
                te = time.perf_counter()
                if i >= 1:
                    rec.setdefault("dev_asm_ms", []).append(system.part.elapsed_ms())
                    rec.setdefault("dev_asm_wall_ms", []).append((te - tw) * 1e3)
                    rec.setdefault("dev_asm_iters", []).append(rep.iterations)
        ctx.barrier()
        # ---------------- value: device-resident (HBM) inputs ---------------
        for i, step in enumerate(seq):
            m_s, if_s = prob.produce(r, step)
            lrb.update(system, m_s, if_s, "direct")     # untimed: coefficients -> HBM
            ctx.barrier()
            if r == 0:
                part, team = system.part, system.team
                others = [q for q in team.parts if q is not part]   # parts on the same GPU
                for q in team.parts:
                    q.sync()
                t_sc = part.apply_scatter_timed(others)
                _, rep, hist = team.solve(method, None, TOL, MAX_ITER, want_x=False,
                                          hist_cap=MAX_ITER)
                part.sync()
                if i >= W:
                    rec["scatter_ms"].append(t_sc)
                    rec["kernel_ms"].append(rep.device_ms)
                    rec["value_ms"].append(t_sc + rep.device_ms)
                    rec["checks"].append(n_checks(hist, rep.iterations, TOL))
                    rec.setdefault("value_iters", []).append(rep.iterations)
            ctx.barrier()
        if r == 0:
            # every part of the team is on this GPU: the work of all of them
            ps = [q.plan for q in system.team.parts]
            rec["plan"] = (sum(p.n for p in ps), sum(p.nnz_local + p.nnz_nonlocal for p in ps),
                           sum(p.n_halo for p in ps), sum(p.n_buf for p in ps))
            rec["kernel_info"] = system.team.kernel_info(method)
        return None

    lrb.run_world(n_cpu, program)
    log(f"[bench] ours done ({time.monotonic() - t0:.1f}s)")
    line = finish_line(args, rec, method,
                       desc.format(n_cpu=n_cpu, alpha=alpha, N=N, cells=f"{N ** 3 / 1e6:.3g}M",
                                   n_gpu=n_gpu if n_gpu == 1 else f"{n_gpu} parts on 1"),
                       N, n_cpu, alpha, sampler)
    if rec.get("dev_asm_ms"):
        line["e2e_device_producer"] = {
            "value": round(float(np.mean(rec["dev_asm_ms"])), 4), "unit": "ms/timestep",
            "wall_ms": round(float(np.mean(rec["dev_asm_wall_ms"])), 4),
            "h2d_bytes_per_step": int(8 * rec["plan"][0]), "d2h_bytes_per_step": int(8 * rec["plan"][0]),
            "iterations_equal_e2e": rec["dev_asm_iters"] == rec["iters"],
            "what": "update_on_device (perturb_coefficients produced on the GPU from the base "
                    "captured at repartition, fused with the scatter; SURVEY §8 f3) + cg_solve "
                    "with b from and x to pinned host memory; no coefficient crosses PCIe"}
    if rec["pg_ms"]:
        line["e2e_pageable"] = {
            "value": round(float(np.mean(rec["pg_ms"])), 4), "unit": "ms/timestep",
            "update_wall_ms": round(float(np.mean(rec["pg_update_ms"])), 4),
            "timer": "host wall clock around update + cg_solve of rank 0 (synchronous API)",
            "inputs": "perturb_coefficients output (pageable numpy, as the reference's own "
                      "generator returns it: a fresh diagonal, the same off-diagonal arrays "
                      "every step); the fresh pieces are host-copied into the part's pinned "
                      "stage inside the update, reused >= 4 MB arrays are page-locked in place "
                      "from their second update on (first update, untimed warm-up)"}
    return line


def run_ours_multi(args):
    """torchrun: one process per GPU; each hosts its part's rpg source ranks as
    threads; the solve kernels of all GPUs synchronise through NVLink peer
    memory (CUDA IPC).  gloo carries only create-time blobs and the
    max-over-ranks of the timings."""
    import torch
    import torch.distributed as dist

    from paper_2510_08536_b200 import _native
    from paper_2510_08536_b200.dist import DistributedOwner, ProcessLayout, max_over_ranks

    rank, world, local_rank = dist_env()
    # one GPU per process; on a 1-GPU box the ranks share it (time-sliced,
    # correctness only — the protocol is the same as over NVLink)
    local_rank = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    from paper_2510_08536_b200.dist import init_plumbing
    backend = init_plumbing(world, local_rank)
    N, _, method_default, desc = WORKLOADS[args.workload]
    method = args.method or method_default
    n_gpu = world
    n_cpu = args.rpg * n_gpu
    alpha = args.rpg
    t0 = time.monotonic()
    import paper_2510_08536_b200 as lrb
    parts_all = lrb.decompose_slab(lrb.StructuredGrid(N, N, N), n_cpu)
    layout = ProcessLayout([p.n_cells for p in parts_all], alpha, world, rank)
    del parts_all
    prob = Problem(N, n_cpu, layout.cpu_ranks, group=alpha)
    owner = DistributedOwner(layout, {r: prob.base[r] for r in layout.cpu_ranks})
    dist.barrier()
    create_s = max_over_ranks(time.monotonic() - t0)
    b = [Problem._pin(torch, np.ones(p.n)) for p in owner.parts]
    warm, timed = step_plan(args)
    seq = warm + timed
    W = len(warm)
    rec = {"e2e_ms": [], "wall_ms": [], "value_ms": [], "scatter_ms": [], "kernel_ms": [],
           "checks": [], "value_iters": [], "launches": 0, "create_s": create_s,
           "kernel_ms_rank": []}
    sampler = ClockSampler(gpu_index(local_rank))
    part = owner.parts[0]
    for i, step in enumerate(seq):
        live = {r: prob.produce(r, step) for r in layout.cpu_ranks}
        torch.cuda.synchronize()
        dist.barrier()
        if i == W:
            sampler.__enter__()
            l0 = _native.lrb_launch_count()
        part.mark()
        tw = time.perf_counter()
        owner.update(live, args.mode)
        xs, rep, _ = owner.solve(method, b, TOL, MAX_ITER)
        part.mark()
        wall = (time.perf_counter() - tw) * 1e3
        torch.cuda.synchronize()
        e2e = max_over_ranks(part.elapsed_ms())
        wall = max_over_ranks(wall)
        if i >= W:
            rec["e2e_ms"].append(e2e)
            rec["wall_ms"].append(wall)
    rec["launches"] = _native.lrb_launch_count() - l0
    dist.barrier()
    sampler.__exit__()
    for i, step in enumerate(seq):
        owner.update({r: prob.produce(r, step) for r in layout.cpu_ranks}, "direct")
        for p in owner.parts:
            p.sync()
        dist.barrier()
        t_sc = owner.parts[0].apply_scatter_timed(owner.parts[1:])
        _, rep, hist = owner.team.solve(method, None, TOL, MAX_ITER, want_x=False,
                                        hist_cap=MAX_ITER)
        t_sc = max_over_ranks(t_sc)
        kms = max_over_ranks(rep.device_ms)
        if i >= W:
            rec["scatter_ms"].append(t_sc)
            rec["kernel_ms"].append(kms)
            rec["kernel_ms_rank"].append(rep.device_ms)
            rec["value_ms"].append(t_sc + kms)
            rec["checks"].append(n_checks(hist, rep.iterations, TOL))
            rec["value_iters"].append(rep.iterations)
    p0 = owner.plans[0]
    # roofline on the max-loaded GPU: the largest part
    sizes = max_over_ranks(float(p0.n))
    rec["plan"] = (p0.n, p0.nnz_local + p0.nnz_nonlocal, p0.n_halo, p0.n_buf)
    rec["kernel_info"] = owner.team.kernel_info(method)
    rec["e2e_update_wall_ms"] = [0.0]
    rec["e2e_solve_wall_ms"] = [0.0]
    rec["e2e_solve_kernel_ms"] = [0.0]
    # per-device evidence: every rank's mean solve-kernel time and launch count
    from paper_2510_08536_b200.dist import allgather_obj
    per_dev = allgather_obj({"rank": rank, "device": torch.cuda.current_device(),
                             "solve_kernel_ms": round(float(np.mean(rec["kernel_ms_rank"])), 4),
                             "launches": int(rec["launches"]), "rows": int(p0.n)})
    line = finish_line(args, rec, method,
                       desc.format(n_cpu=n_cpu, n_gpu=n_gpu, alpha=alpha, N=N,
                                   cells=f"{N ** 3 / 1e6:.3g}M"), N, n_cpu, alpha, sampler)
    line["config"]["max_part_rows"] = int(sizes)
    line["config"]["parallelism"] = f"{n_gpu} GPU parts, NVLink peer-memory halo + reductions"
    line["per_device"] = per_dev
    line["devices_ran_solve"] = sum(1 for d in per_dev if d["launches"] > 0)
    line["plumbing"] = (f"torch.distributed {backend}: create-time blobs, barriers, max-over-ranks "
                        "timing; the solve's halo and reductions move by NVLink peer stores "
                        "inside the kernels (no collective on the data path)")
    dist.barrier()
    dist.destroy_process_group()
    return line if rank == 0 else None


def kernel_name(info, method):
    """The solve kernel that ran (lrb_team_kernel_info): streaming or classic."""
    jac = "true" if method in ("pcg", "pcg1", "pipecg") else "false"
    if info and info.get("streaming") and method == "pipecg":
        return (f"team_pipecg_stream_kernel (pipelined Jacobi-PCG, one barrier per iteration, bulk-copy "
                f"ring: {info['stages']} x {info['stage_bytes']} B stages, {info['grid']} x {info['block']} threads)")
    if info and info.get("streaming") and method == "pcg1":
        return (f"team_pcg1_stream_kernel (single-reduction Jacobi-PCG, bulk-copy ring: {info['stages']} x "
                f"{info['stage_bytes']} B stages, {info['grid']} x {info['block']} threads)")
    if info and info.get("streaming"):
        return (f"team_cg_stream_kernel<JAC={jac}> (persistent, bulk-copy ring: {info['stages']} x "
                f"{info['stage_bytes']} B stages, {info['grid']} x {info['block']} threads)")
    return f"team_cg_kernel<JAC={jac}> (persistent, classic per-thread gathers)"


def finish_line(args, rec, method, desc, N, n_cpu, alpha, sampler):
    n, nnz, h, n_buf = rec["plan"]
    value = float(np.mean(rec["value_ms"]))
    peak, peak_kind = measured_peak()
    alg = [solve_bytes(n, nnz, h, it, ck, method) for it, ck in zip(rec["value_iters"],
                                                                    rec["checks"])]
    achieved = float(np.mean([b / (ms * 1e-3) / 1e9 for b, ms in zip(alg, rec["kernel_ms"])]))
    scatter_gbs = float(np.mean([20 * n_buf / (ms * 1e-3) / 1e9 for ms in rec["scatter_ms"]]))
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "ms/timestep",
        "n_gpus": gpus_used(args), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(value, 4), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference cavity generator, "
                                                    "closed form)",
        "config": {"workload": desc, "n_cells": N ** 3, "n_cpu": n_cpu, "alpha": alpha,
                   "mode": args.mode, "method": method, "tol": TOL,
                   "timesteps": timesteps_label(args), "warmup": warmup_label(args),
                   "l2": "inputs larger than L2 (no flush needed)" if N >= 100 else
                         "L2-resident (latency-bound)"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                     "kernel": kernel_name(rec.get("kernel_info"), method),
                     "kernel_geometry": rec.get("kernel_info"),
                     "peak_kind": peak_kind,
                     "alg_bytes_per_launch": int(np.mean(alg)),
                     "kernel_ms": round(float(np.mean(rec["kernel_ms"])), 4)},
        "e2e": {"value": round(float(np.mean(rec["e2e_ms"])), 4), "unit": "ms/timestep",
                "h2d_bytes_per_step": int(8 * n_buf + 8 * n),
                "d2h_bytes_per_step": int(8 * n),
                "wall_ms": round(float(np.mean(rec["wall_ms"])), 4),
                "update_wall_ms": round(float(np.mean(rec["e2e_update_wall_ms"])), 4),
                "solve_wall_ms": round(float(np.mean(rec["e2e_solve_wall_ms"])), 4),
                "solve_kernel_ms": round(float(np.mean(rec["e2e_solve_kernel_ms"])), 4)},
        "breakdown": {"scatter_ms": round(float(np.mean(rec["scatter_ms"])), 4),
                      "scatter_gbs": round(scatter_gbs, 1),
                      "solve_kernel_ms": round(float(np.mean(rec["kernel_ms"])), 4),
                      "iterations": rec["value_iters"], "create_s": round(rec["create_s"], 2)},
        "gpu_launches": int(rec["launches"]),
        "clocks": sampler.summary(),
    }
    # the capture of this workload's solve kernel: "<workload>_<method>", or
    # "<workload>" for two-phase PCG
    t = traffic_ratio(f"{args.workload}_{method}") or (traffic_ratio(args.workload) if method == "pcg" else None)
    if t:
        # ncu DRAM bytes per algorithmic byte of the solve kernel, applied to this
        # run's launches (same kernel, same config)
        line["roofline"]["traffic"] = int(t["dram_bytes_per_alg_byte"] *
                                          line["roofline"]["alg_bytes_per_launch"])
        line["roofline"]["traffic_note"] = t.get("note")
        dram_gbs = line["roofline"]["traffic"] / (line["roofline"]["kernel_ms"] * 1e-3) / 1e9
        line["roofline"]["dram_achieved"] = round(dram_gbs, 1)
        line["roofline"]["dram_frac"] = round(dram_gbs / line["roofline"]["peak"], 4)
    ts = traffic_ratio(args.workload + "_scatter")
    if ts:
        # the whole-part scatter's DRAM bytes per algorithmic byte (ncu), applied
        # to this run's scatter time
        sd = scatter_gbs * ts["dram_bytes_per_alg_byte"]
        line["breakdown"]["scatter_dram_gbs"] = round(sd, 1)
        line["breakdown"]["scatter_dram_frac"] = round(sd / line["roofline"]["peak"], 4)
        line["breakdown"]["scatter_traffic_note"] = ts.get("note")
    return line


# ---------------------------------------------------------------------------
# C4: full timestep (momentum BiCGStab x 3 + pressure Jacobi-PCG), one GPU
# ---------------------------------------------------------------------------
MOM_RHS = 3


def momentum_eps(m, seed):
    rng = np.random.default_rng(seed)
    return 0.05 * rng.random(m.n_faces), 0.05 * rng.random(m.n_faces)


def momentum_values_into(eps_u, eps_l, step, upper, lower):
    """Non-symmetric, diagonally dominant momentum coefficients of a timestep
    (upper -1+eps, lower -1-eps, diag 6.5), eps scaled by the step;
    written in place into the (pinned) arrays the update reads."""
    f = 1.0 + step / 100.0
    np.multiply(eps_u, f, out=upper)
    upper -= 1.0
    np.multiply(eps_l, -f, out=lower)
    lower -= 1.0


def momentum_rhs(n, k):
    i = np.arange(n, dtype=np.float64)
    return np.ones(n) if k == 0 else (1.0 + np.mod(i, 3.0 + k)) * (0.5 ** k)


def run_c4(args):
    import torch

    import paper_2510_08536_b200 as lrb
    from paper_2510_08536_b200 import _native

    N = args.n or WORKLOADS["c4"][0]
    n_cpu = args.rpg * args.gpus
    alpha = args.rpg
    torch.cuda.set_device(0)
    t0 = time.monotonic()
    prob = Problem(N, n_cpu, range(n_cpu), group=alpha)
    pm = lrb.make_partition_map(prob.cells, alpha)
    mom = {}
    # momentum LDU on the same addressing; its value arrays (interface blocks
    # included) are pinned views in pack order, one block per GPU part
    flat = Problem._pin(torch, np.zeros(sum(Problem._pack_len(*prob.base[r]) for r in range(n_cpu))))
    o = 0
    for r in range(n_cpu):
        m, ifs = prob.base[r]
        n = Problem._pack_len(m, ifs)
        mm, ifp, dg = Problem._views(lrb, m, ifs, flat[o:o + n])
        o += n
        dg[:] = 6.5
        eu, el = momentum_eps(m, r)
        mom[r] = (mm, ifp, eu, el, mm.upper_val, mm.lower_val)
    log(f"[bench c4] inputs {time.monotonic() - t0:.1f}s; N={N} n_cpu={n_cpu} alpha={alpha}")
    warm, timed = step_plan(args)
    seq = warm + timed
    W = len(warm)
    rec = {"e2e_ms": [], "value_ms": [], "kernel_ms": [], "alg": [], "iters_p": [], "iters_m": [],
           "launches": 0, "create_s": 0.0, "press_ms": [], "press_alg": []}
    sampler = ClockSampler(gpu_index())

    def produce_mom(r, step):
        mm, ifs, eu, el, up, lo = mom[r]
        momentum_values_into(eu, el, step, up, lo)
        return mm, ifs

    def program(ctx):
        r = ctx.rank
        tc = time.monotonic()
        sm = lrb.repartition(*produce_mom(r, 1), pm, ctx)    # momentum system
        sp = lrb.repartition(*prob.base[r], pm, ctx)          # pressure system
        ctx.barrier()
        if r == 0:
            rec["create_s"] = time.monotonic() - tc
        bs = [Problem._pin(torch, momentum_rhs(sm.matrix.n_owned, k)) for k in range(MOM_RHS)] \
            if sm.is_owner else None
        bp = Problem._pin(torch, np.ones(sp.matrix.n_owned)) if sp.is_owner else None
        # ---------------- e2e: public API, host buffers ----------------------
        for i, step in enumerate(seq):
            m_s, if_s = produce_mom(r, step)
            p_s, pif_s = prob.produce(r, step)
            ctx.barrier()
            if r == 0:
                if i == W:
                    sampler.__enter__()
                    rec["l0"] = _native.lrb_launch_count()
                tw = time.perf_counter()
            lrb.update(sm, m_s, if_s, "direct")
            its = []
            if sm.is_owner:
                for k in range(MOM_RHS):
                    _, rep = lrb.bicgstab_solve(sm.matrix, sm.halo, bs[k], TOL, MAX_ITER, sm.comm)
                    its.append(rep.iterations)
            lrb.update(sp, p_s, pif_s, "direct")
            if sp.is_owner:
                _, rep = lrb.cg_solve(sp.matrix, sp.halo, bp, TOL, MAX_ITER, sp.comm, method="pcg")
            if r == 0:
                # the API calls are synchronous (x lands on the host): wall clock
                if i >= W:
                    rec["e2e_ms"].append((time.perf_counter() - tw) * 1e3)
                    rec["iters_m"].append(its)
                    rec["iters_p"].append(rep.iterations)
                if i == len(seq) - 1:
                    rec["launches"] = _native.lrb_launch_count() - rec["l0"]
        ctx.barrier()
        if r == 0:
            sampler.__exit__()
        # ---------------- value: device-resident (HBM) inputs ---------------
        for i, step in enumerate(seq):
            lrb.update(sm, *produce_mom(r, step), "direct")   # untimed: coefficients -> HBM
            lrb.update(sp, *prob.produce(r, step), "direct")
            ctx.barrier()
            if r == 0:
                tot = 0.0
                kms = 0.0
                alg = 0
                alg_k = {"scatter": 0, "bicgstab": 0, "pcg": 0}
                pln = sm.part.plan
                n, nnz, h = pln.n, pln.nnz_local + pln.nnz_nonlocal, pln.n_halo
                for part, team, method, rhs in ((sm.part, sm.team, "bicgstab", bs),
                                                (sp.part, sp.team, "pcg", [bp])):
                    part.sync()
                    tot += part.apply_scatter_timed()
                    alg += 20 * pln.n_buf
                    alg_k["scatter"] += 20 * pln.n_buf
                    for b in rhs:
                        _, rep, hist = team.solve(method, [b], TOL, MAX_ITER, want_x=False,
                                                  hist_cap=MAX_ITER)
                        tot += rep.device_ms
                        kms += rep.device_ms
                        ck = n_checks(hist, rep.iterations, TOL)
                        a = (bicgstab_bytes(n, nnz, h, rep.iterations, ck) if method == "bicgstab"
                             else solve_bytes(n, nnz, h, rep.iterations, ck, "pcg"))
                        alg += a
                        alg_k[method] += a
                        if method == "pcg" and i >= W:
                            rec["press_ms"].append(rep.device_ms)
                            rec["press_alg"].append(a)
                if i >= W:
                    rec["value_ms"].append(tot)
                    rec["kernel_ms"].append(kms)
                    rec["alg"].append(alg)
                    rec.setdefault("alg_k", []).append(alg_k)
            ctx.barrier()
        if r == 0:
            p = sp.part.plan
            rec["plan"] = (p.n, p.nnz_local + p.nnz_nonlocal, p.n_halo, p.n_buf)
            rec["kinfo"] = {"bicgstab": sm.team.kernel_info("bicgstab"),
                            "pcg": sp.team.kernel_info("pcg")}
        return None

    lrb.run_world(n_cpu, program)
    log(f"[bench c4] done ({time.monotonic() - t0:.1f}s)")
    n, nnz, h, n_buf = rec["plan"]
    peak, peak_kind = measured_peak()
    value = float(np.mean(rec["value_ms"]))
    achieved = float(np.mean([a / (ms * 1e-3) / 1e9 for a, ms in zip(rec["alg"], rec["value_ms"])]))
    p_ach = float(np.mean([a / (ms * 1e-3) / 1e9 for a, ms in zip(rec["press_alg"],
                                                                 rec["press_ms"])]))
    desc = WORKLOADS["c4"][3].format(N=N, cells=f"{N ** 3 / 1e6:.3g}M", n_cpu=n_cpu, n_gpu=args.gpus,
                                      alpha=alpha)
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "ms/timestep", "n_gpus": gpus_used(args),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value, 4),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference cavity generator; momentum LDU per SURVEY §8d)",
        "config": {"workload": desc, "n_cells": N ** 3, "n_cpu": n_cpu, "alpha": alpha, "mode": "direct",
                   "method": "bicgstab x3 + pcg", "tol": TOL, "timesteps": timesteps_label(args),
                   "warmup": warmup_label(args), "l2": "inputs larger than L2 (no flush needed)"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None, "peak_kind": peak_kind,
                     "kernel": "whole timestep: 2 scatters + 3 team_bicgstab_stream_kernel + "
                               "team_cg_stream_kernel<JAC=true>",
                     "kernel_geometry": rec.get("kinfo"),
                     "alg_bytes_per_launch": int(np.mean(rec["alg"])),
                     "kernel_ms": round(float(np.mean(rec["kernel_ms"])), 4),
                     "pressure_pcg_achieved": round(p_ach, 1),
                     "pressure_pcg_frac": round(p_ach / peak, 4)},
        "e2e": {"value": round(float(np.mean(rec["e2e_ms"])), 4), "unit": "ms/timestep",
                "timer": "host wall clock around the synchronous API calls of rank 0",
                "h2d_bytes_per_step": int(2 * 8 * n_buf + 8 * n * (MOM_RHS + 1)),
                "d2h_bytes_per_step": int(8 * n * (MOM_RHS + 1))},
        "breakdown": {"iterations_momentum": rec["iters_m"], "iterations_pressure": rec["iters_p"],
                      "create_s": round(rec["create_s"], 2)},
        "gpu_launches": int(rec["launches"]),
        "clocks": sampler.summary(),
    }
    tb, tp = traffic_ratio("c4_bicgstab"), traffic_ratio("c4_pcg")
    if tb and tp:
        # ncu DRAM bytes per algorithmic byte of each solve kernel at 300^3; the
        # scatters are counted at their algorithmic bytes (DRAM/alg ~1 for a
        # whole-part launch, profiles/r2_c3_scatter_summary.md)
        ak = {k: float(np.mean([a[k] for a in rec["alg_k"]])) for k in rec["alg_k"][0]}
        traffic = (tb["dram_bytes_per_alg_byte"] * ak["bicgstab"] +
                   tp["dram_bytes_per_alg_byte"] * ak["pcg"] + ak["scatter"])
        line["roofline"]["traffic"] = int(traffic)
        line["roofline"]["traffic_note"] = "; ".join([tb.get("note", ""), tp.get("note", "")])
        dram = traffic / (value * 1e-3) / 1e9
        line["roofline"]["dram_achieved"] = round(dram, 1)
        line["roofline"]["dram_frac"] = round(dram / peak, 4)
    return line


# ---------------------------------------------------------------------------
# C5: value-update-only stress (BASELINE.json configs[4]): 200^3, 128 ranks ->
# 8 parts (alpha 16); the 8 parts are spread over the N GPUs (strong scaling)
# ---------------------------------------------------------------------------
def run_c5(args):
    import torch

    import paper_2510_08536_b200 as lrb
    from paper_2510_08536_b200 import _native
    from paper_2510_08536_b200.dist import DistributedOwner, ProcessLayout, max_over_ranks

    rank, world, local_rank = dist_env()
    N, alpha = WORKLOADS["c5"][0], WORKLOADS["c5"][1]
    n_cpu = C5_RANKS
    torch.cuda.set_device(local_rank % torch.cuda.device_count())
    if world > 1:
        from paper_2510_08536_b200.dist import init_plumbing
        init_plumbing(world, local_rank % torch.cuda.device_count())
    t0 = time.monotonic()
    cells = [p.n_cells for p in lrb.decompose_slab(lrb.StructuredGrid(N, N, N), n_cpu)]
    layout = ProcessLayout(cells, alpha, world, rank)
    prob = Problem(N, n_cpu, layout.cpu_ranks, group=alpha)
    owner = DistributedOwner(layout, {r: prob.base[r] for r in layout.cpu_ranks}, solve=False)
    create_s = time.monotonic() - t0
    for p in owner.parts:   # the pristine base, for the GPU-producer leg
        p.capture_base()
    mx = (lambda v: max_over_ranks(v)) if world > 1 else (lambda v: v)
    sync = (lambda: torch.distributed.barrier()) if world > 1 else (lambda: None)
    log(f"[bench c5] create {create_s:.1f}s; parts {layout.parts} ranks "
        f"{layout.cpu_ranks[0]}..{layout.cpu_ranks[-1]}")
    warm, timed = step_plan(args)
    seq = warm + timed
    W = len(warm)
    rec = {"e2e": [], "pg": [], "value": [], "launches": 0}
    sampler = ClockSampler(gpu_index(local_rank))

    def timed_update(live, mode):
        torch.cuda.synchronize()
        sync()
        for p in owner.parts:
            p.mark()
        tw = time.perf_counter()
        owner.update(live, mode)
        for p in owner.parts:
            p.mark()
        for p in owner.parts:
            p.sync()
        wall = (time.perf_counter() - tw) * 1e3
        ev = max(p.elapsed_ms() for p in owner.parts)
        return mx(ev), mx(wall)

    for i, step in enumerate(seq):   # e2e: pinned producer, direct mode
        live = {r: prob.produce(r, step) for r in layout.cpu_ranks}
        if i == W:
            sampler.__enter__()
            l0 = _native.lrb_launch_count()
        ev, wall = timed_update(live, args.mode)
        if i >= W:
            rec["e2e"].append((ev, wall))
    rec["launches"] = _native.lrb_launch_count() - l0
    sampler.__exit__()
    if not args.no_pageable:
        for i, step in enumerate([2] + timed):   # pageable drop-in inputs
            live = {r: prob.produce_pageable(r, step) for r in layout.cpu_ranks}
            ev, wall = timed_update(live, args.mode)
            if i >= 1:
                rec["pg"].append((ev, wall))
            del live
    # GPU-side producer: the timestep's coefficients made on the
    # device from the base captured after create, fused with the scatter
    for i, step in enumerate([2] + timed):
        torch.cuda.synchronize()
        sync()
        for p in owner.parts:
            p.mark()
        for p in owner.parts:
            p.update_perturb(1.0 + step / 100.0)
        for p in owner.parts:
            p.mark()
        ms = mx(max(p.elapsed_ms() for p in owner.parts))
        if i >= 1:
            rec.setdefault("dev", []).append(ms)
    for i, step in enumerate(seq):   # value: receive buffers already in HBM
        owner.update({r: prob.produce(r, step) for r in layout.cpu_ranks}, "direct")
        for p in owner.parts:
            p.sync()
        sync()
        ms = mx(owner.parts[0].apply_scatter_timed(owner.parts[1:]))
        if i >= W:
            rec["value"].append(ms)
    n_buf = sum(p.n_buf for p in owner.parts)
    n_rows = sum(p.n for p in owner.parts)
    n_buf_all = int(mx(float(n_buf))) if world == 1 else None
    peak, peak_kind = measured_peak()
    value = float(np.mean(rec["value"]))
    e2e = float(np.mean([e for e, _ in rec["e2e"]]))
    scat_gbs = 20 * n_buf / (value * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "ms/timestep", "n_gpus": gpus_used(args),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value, 4),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference cavity generator, closed form)",
        "config": {"workload": WORKLOADS["c5"][3].format(n_gpu=world), "n_cells": N ** 3,
                   "n_cpu": n_cpu, "alpha": alpha, "mode": args.mode, "method": "update only",
                   "timesteps": timesteps_label(args), "warmup": warmup_label(args),
                   "parts_per_gpu": len(layout.parts),
                   "l2": "inputs larger than L2 (no flush needed)"},
        "roofline": {"bound": "hbm", "achieved": round(scat_gbs, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(scat_gbs / peak, 4), "traffic": None, "peak_kind": peak_kind,
                     "kernel": "scatter_rows_kernel (gather-permute, 20 B/entry), one launch per "
                               "part (device-resident) / per segment (update path)",
                     "alg_bytes_per_launch": int(20 * n_buf / max(1, len(owner.parts))),
                     "kernel_ms": round(value / max(1, len(owner.parts)), 4)},
        "e2e": {"value": round(e2e, 4), "unit": "ms/timestep",
                "h2d_bytes_per_step": int(8 * n_buf), "d2h_bytes_per_step": 0,
                "wall_ms": round(float(np.mean([w for _, w in rec["e2e"]])), 4),
                "link_gbs": round(8 * n_buf / (e2e * 1e-3) / 1e9, 1),
                "link_peak_gbs": PCIE_PINNED_GBS,
                "link_frac": round(8 * n_buf / (e2e * 1e-3) / 1e9 / PCIE_PINNED_GBS, 4)},
        "breakdown": {"entries_per_step": int(n_buf), "rows": int(n_rows),
                      "segments": len(layout.cpu_ranks), "create_s": round(create_s, 2),
                      "scatter_gbs": round(scat_gbs, 1)},
        "gpu_launches": int(rec["launches"]),
        "clocks": sampler.summary(),
    }
    if n_buf_all is not None:
        line["breakdown"]["entries_all_parts"] = n_buf_all
    if rec.get("dev"):
        line["e2e_device_producer"] = {
            "value": round(float(np.mean(rec["dev"])), 4), "unit": "ms/timestep",
            "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
            "what": "lrb_update_perturb per part (perturb_coefficients produced on the GPU from the "
                    "base captured after create, fused with the scatter; SURVEY §8 f3)"}
    if rec["pg"]:
        pg = float(np.mean([e for e, _ in rec["pg"]]))
        line["e2e_pageable"] = {"value": round(pg, 4), "unit": "ms/timestep",
                                "link_gbs": round(8 * n_buf / (pg * 1e-3) / 1e9, 1),
                                "inputs": "perturb_coefficients output (pageable numpy); host "
                                          "copy into the pinned stage counted"}
    # the same kernel's whole-part DRAM/algorithmic ratio from ncu at C3 (the 8
    # concurrent part launches move 1.1 GB, well past L2, like the C3 launch)
    t = traffic_ratio("c5") or traffic_ratio("c3_scatter")
    if t:
        line["roofline"]["traffic"] = int(t["dram_bytes_per_alg_byte"] *
                                          line["roofline"]["alg_bytes_per_launch"])
        line["roofline"]["traffic_note"] = t.get("note")
        dram = line["roofline"]["traffic"] / (line["roofline"]["kernel_ms"] * 1e-3) / 1e9
        line["roofline"]["dram_achieved"] = round(dram, 1)
        line["roofline"]["dram_frac"] = round(dram / peak, 4)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return line if rank == 0 else None


# ---------------------------------------------------------------------------
# reference arm: the UNMODIFIED reference package on the host cores
# ---------------------------------------------------------------------------
def load_reference():
    """The reference installed with pip into baseline/_ref (git-ignored; it
    travels to the GPU box with the snapshot)."""
    if not os.path.isdir(os.path.join(REF_DIR, "ldurepart")):
        return None
    sys.path.insert(0, REF_DIR)
    import ldurepart
    if not os.path.abspath(ldurepart.__file__).startswith(os.path.abspath(REF_DIR)):
        raise RuntimeError(f"ldurepart imported from {ldurepart.__file__}, not baseline/_ref")
    return ldurepart


def reference_steps(args, ref, N, n_cpu, alpha, solve=True, warm_max_iter=2):
    """The reference's cli.run_case protocol (cli.py:181-272) through its own
    public API — repartition once, then per timestep perturb_coefficients ->
    update -> cg_solve on the owners — inside its deterministic World.  Per
    phase the time is the max over ranks (cli.py:260-262); the producer
    (perturb_coefficients, the reference's t_assemble) is not part of the
    metric, as in our arm.  cli.run_case itself cannot be called: its World
    uses the default 120 s watchdog (transport.py:133,324) and it always solves
    the unperturbed creation step first (cli.py:233), minutes at 200^3.
    Warm-up replays of timestep 2 run cg_solve with max_iter=warm_max_iter."""
    warm, timed = step_plan(args)
    seq = warm + timed
    W = len(warm)
    grid = ref.StructuredGrid(N, N, N)
    parts = ref.decompose_slab(grid, n_cpu)
    pm = ref.make_partition_map([p.n_cells for p in parts], alpha)
    clock = time.perf_counter

    def program(ctx):
        base_m, base_if = ref.assemble_poisson(parts[ctx.rank])
        t0 = clock()
        system = ref.repartition(base_m, base_if, pm, ctx)
        st = {"create": clock() - t0, "update": [], "solve": [], "iters": [], "wall": []}
        b = np.ones(system.matrix.n_owned) if system.is_owner else None
        for i, step in enumerate(seq):
            m_s, if_s = ref.perturb_coefficients(base_m, base_if, step)
            ctx.barrier()
            tw = clock()
            t0 = clock()
            ref.update(system, m_s, if_s, args.mode)
            t_up = clock() - t0
            t_solve, its = 0.0, None
            if solve and system.is_owner:
                t0 = clock()
                _, rep = ref.cg_solve(system.matrix, system.halo, b, TOL,
                                      warm_max_iter if i < W else MAX_ITER, system.comm)
                t_solve = clock() - t0
                its = rep.iterations
            ctx.barrier()
            if i >= W:
                st["update"].append(t_up)
                st["solve"].append(t_solve)
                st["iters"].append(its)
                st["wall"].append(clock() - tw)
        return st

    t0 = time.monotonic()
    res = ref.run_world(n_cpu, program, timeout=1e7)
    wall = time.monotonic() - t0
    t_up = [max(r["update"][s] for r in res) for s in range(len(timed))]
    t_so = [max(r["solve"][s] for r in res) for s in range(len(timed))]
    return {"step_ms": [(u + s) * 1e3 for u, s in zip(t_up, t_so)],
            "update_ms": [u * 1e3 for u in t_up], "solve_ms": [s * 1e3 for s in t_so],
            "iterations": res[0]["iters"], "create_s": max(r["create"] for r in res),
            "world_wall_ms": [w * 1e3 for w in res[0]["wall"]],
            "wall_s": wall, "timed": timed}


def port_steps(args, N, n_cpu, alpha):
    """Fallback when baseline/_ref is absent: the oracle/ numpy port of the
    same path, full solves on every timed step (no projection)."""
    from oracle import cavity as ocav
    from oracle import krylov
    from oracle.pipeline import OraclePipeline
    warm, timed = step_plan(args)
    probs = ocav.cavity_problems((N, N, N), n_cpu)
    offsets = np.concatenate(([0], np.cumsum([p.n for p in probs]))).astype(np.int64)
    t0 = time.monotonic()
    pipe = OraclePipeline(probs, offsets, alpha)
    create = time.monotonic() - t0
    out = {"step_ms": [], "update_ms": [], "solve_ms": [], "iterations": [], "create_s": create,
           "timed": timed}
    for i, step in enumerate(warm + timed):
        ps = [ocav.perturb(p, step) for p in probs]
        ts = time.perf_counter()
        pipe.update(ps)
        t_up = time.perf_counter() - ts
        ts = time.perf_counter()
        _, rep = krylov.cg(pipe.system, pipe.rhs_ones(), TOL,
                           2 if i < len(warm) else MAX_ITER, jacobi=False)
        its = rep.iterations
        t_so = time.perf_counter() - ts
        if i >= len(warm):
            out["step_ms"].append((t_up + t_so) * 1e3)
            out["update_ms"].append(t_up * 1e3)
            out["solve_ms"].append(t_so * 1e3)
            out["iterations"].append(its)
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    wl = args.workload
    N = args.n or WORKLOADS[wl][0]
    if wl == "c5":
        n_cpu, alpha, n_gpu = C5_RANKS, WORKLOADS["c5"][1], args.gpus
    else:
        n_gpu = args.gpus
        n_cpu, alpha = args.rpg * n_gpu, args.rpg
    ref = load_reference()
    if ref is not None:
        kind = "reference"
        res = reference_steps(args, ref, N, n_cpu, alpha, solve=(wl != "c5"))
        what = (f"unmodified reference ldurepart {getattr(ref, '__version__', '')} "
                f"(baseline/_ref, pip-installed from /root/reference)")
    else:
        kind = "port"
        res = port_steps(args, N, n_cpu, alpha)
        what = "oracle/ numpy port of the reference path (baseline/_ref absent)"
    value = float(np.mean(res["step_ms"]))
    hi = host_info()
    steps_txt = f"timesteps {res['timed'][0]}..{res['timed'][-1]}"
    if wl == "c4":
        note = "pressure update + CG only: the reference has no BiCGStab (SPEC.md:468)"
    elif wl == "c5":
        note = "update only"
    else:
        note = "update + CG (the reference's solver; its iterates equal Jacobi-PCG's on the " \
               "uniform-diagonal cavity, SURVEY App. B)"
    sample = (f"{what}: cli.run_case protocol, {N}^3, {n_cpu} ranks, alpha {alpha}, "
              f"deterministic World; repartition once ({res['create_s']:.1f}s, excluded), "
              f"{args.warmup} warm-up replays of timestep 2 (cg_solve max_iter=2), then {steps_txt} "
              f"each run in full ({note}); per phase the max over ranks (cli.py:260-262)")
    cores = int(hi["openblas_num_threads"] or 1)
    if wl == "c5":
        desc = WORKLOADS["c5"][3].format(n_gpu=n_gpu)
    else:
        desc = WORKLOADS[wl][3].format(n_cpu=n_cpu, n_gpu=n_gpu, alpha=alpha, N=N,
                                       cells=f"{N ** 3 / 1e6:.3g}M")
    config = {"workload": desc, "n_cells": N ** 3, "n_cpu": n_cpu, "alpha": alpha,
              "mode": args.mode, "method": WORKLOADS[wl][2] or "update only", "tol": TOL,
              "timesteps": timesteps_label(args), "warmup": warmup_label(args),
              "l2": "inputs larger than L2 (no flush needed)" if N >= 100 else
                    "L2-resident (latency-bound)"}
    if wl == "c5":
        config.pop("tol")
        config["parts_per_gpu"] = 8 // max(1, args.gpus) if 8 % max(1, args.gpus) == 0 else None
    if wl == "c4":
        config["method"] = "bicgstab x3 + pcg"
    cpu = {"value": round(value, 2), "unit": "ms/timestep", "cores": cores, "kind": kind,
           "sample": sample, "host": hi,
           "cores_note": ("the reference's rank code is single-core: one rank thread runs at a time "
                          "(transport.py:206-219) and its SpMV (np.add.at, 92% of a CG iteration, "
                          "SURVEY §3) is single-threaded; OpenBLAS threads for its dots were measured "
                          "slower (C1: 425 vs 45 ms/timestep at 8 threads), so 1 is its fastest "
                          "configuration")}
    return {
        "metric": METRIC, "value": round(value, 2), "unit": "ms/timestep", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value, 2),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference cavity generator)", "impl": "reference",
        "config": config,
        "cpu_baseline": cpu,
        "e2e": {"value": round(value, 2), "unit": "ms/timestep", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "breakdown": {"update_ms": [round(v, 2) for v in res["update_ms"]],
                      "solve_ms": [round(v, 2) for v in res["solve_ms"]],
                      "iterations": res["iterations"], "create_s": round(res["create_s"], 2),
                      # whole-world wall time of each step (barrier to barrier on rank 0):
                      # the deterministic scheduler runs one rank at a time, so this is the
                      # serialised cost; value is the reference's own max-over-ranks metric
                      "world_wall_ms": [round(v, 2) for v in res.get("world_wall_ms", [])]},
    }


def cpu_baseline(args):
    """Bounded sample for our line: the reference arm on timestep 2 only (its
    heaviest timestep), in a subprocess so it gets the host's BLAS threads."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
           "--warmup", "3", "--workload", args.workload, "--gpus", str(args.gpus),
           "--mode", args.mode]
    if args.workload != "c5":
        cmd += ["--rpg", str(args.rpg)]
    if args.n:
        cmd += ["--n", str(args.n)]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, env=env,
                             timeout=args.cpu_budget_s).stdout
        line = json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])
    except Exception as exc:  # noqa: BLE001 - reported, not hidden
        return {"value": None, "unit": "ms/timestep", "cores": None, "kind": None,
                "sample": f"cpu baseline failed: {type(exc).__name__}: {exc}"}
    cb = dict(line["cpu_baseline"])
    cb["sample"] = "timestep 2 only (bounded sample) — " + cb["sample"]
    return cb


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c3")
    ap.add_argument("--rpg", type=int, default=None, help="CPU ranks per GPU (alpha)")
    ap.add_argument("--n", type=int, default=None, help="cavity edge (c4; default 300)")
    ap.add_argument("--mode", choices=("direct", "staged"), default="direct")
    ap.add_argument("--method", choices=("cg", "pcg", "pcg1", "pipecg"), default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pageable", action="store_true",
                    help="skip the pageable-input e2e leg")
    ap.add_argument("--cpu-budget-s", type=float, default=600.0,
                    help="time limit of the cpu_baseline subprocess")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.rpg is None:
        args.rpg = WORKLOADS[args.workload][1]
    if args.impl == "reference":
        line = run_reference(args)
    else:
        line = run_ours(args)
        rank, world, _ = dist_env()
        if line is not None and rank == 0 and world == 1:
            if args.no_cpu_baseline:
                line["cpu_baseline"] = None
                line["cpu_baseline_note"] = "skipped (--no-cpu-baseline)"
            else:
                if args.workload == "c4":   # 300^3: the reference's create alone is ~1.5 min
                    args.cpu_budget_s = max(args.cpu_budget_s, 1500.0)
                line["cpu_baseline"] = cpu_baseline(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
