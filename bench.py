#!/usr/bin/env python
"""Benchmark: ms per timestep (matrix update + Krylov solve) on B200.

Workload (BASELINE.json configs[2], "C3"): 3D cavity 200^3 (8M cells),
``--rpg`` CPU assembly ranks per GPU (default 8) repartitioned onto N GPUs,
pressure Jacobi-PCG to 1e-6 with b = ones, timesteps 2.. of the reference
protocol (cli.py:181-272; step 1 = creation, excluded).  One timestep =
update (all coefficients of every rank: H2D + gather-permute) + solve.

* ``value``  device-resident: coefficients already in the receive buffer in
  HBM, b resident; timed = scatter kernel + solve kernel (CUDA events).
* ``e2e``    through the public API (``update`` from pinned host LDU arrays by
  every rank thread, then ``cg_solve`` with b from host and x back to host).
* ``--impl reference``: the reference CPU path (oracle port, oracle/) on the
  host cores, bounded sample scaled to a full timestep.

Inputs (1.5 GB PCG working set at N=1) are larger than L2, so no L2 flush is
needed between timed steps.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms/timestep (matrix update + CG solve) at 1/2/4/8 B200; % of HBM roofline"
WORKLOADS = {
    # name: (N, default rpg, method, description)
    "c3": (200, 8, "pcg", "C3: 3D cavity 200^3 (8M cells), {n_cpu} CPU ranks -> {n_gpu} GPU(s) "
                          "(alpha {alpha}), pressure Jacobi-PCG to 1e-6, b=ones"),
    "c2": (100, 8, "pcg", "C2: 3D cavity 100^3 (1M cells), {n_cpu} CPU ranks -> {n_gpu} GPU(s) "
                          "(alpha {alpha}), Jacobi-PCG to 1e-6"),
    "c1": (32, 4, "pcg", "C1: 3D cavity 32^3, {n_cpu} CPU ranks -> {n_gpu} device(s) "
                         "(alpha {alpha}), Jacobi-PCG to 1e-6"),
    "c4": (300, 16, "pcg", "C4: 3D cavity {N}^3 ({cells} cells), {n_cpu} CPU ranks -> {n_gpu} GPU(s) "
                           "(alpha {alpha}), full timestep: momentum update + 3 BiCGStab (Ux, Uy, Uz) "
                           "+ pressure update + Jacobi-PCG, all to 1e-6"),
}
TOL, MAX_ITER = 1e-6, 2000


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


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


# ---------------------------------------------------------------------------
# roofline accounting
# ---------------------------------------------------------------------------
def solve_bytes(n, nnz, h, iterations, checks, method):
    """Algorithmic HBM bytes of one solve: CG it 12nnz+4(n+1)+88n+8h, PCG +16n,
    true-residual check 12nnz+4(n+1)+16n+8h, init (b read, x r written) 24n.
    pcg1 (single reduction): it 12nnz+4(n+1)+8h + 88n (r, dinv, w, s_old and
    p, x read; p, x, r, s, w written), init + one SpMV 12nnz+4(n+1)+24n+8h."""
    chk = 12 * nnz + 4 * (n + 1) + 16 * n + 8 * h
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


# ---------------------------------------------------------------------------
# problem
# ---------------------------------------------------------------------------
class Problem:
    """Per-rank LDU inputs whose value arrays live in pinned host memory."""

    def __init__(self, N, n_cpu, ranks, pinned=True):
        import paper_2510_08536_b200 as lrb
        self.lrb = lrb
        grid = lrb.StructuredGrid(N, N, N)
        parts = lrb.decompose_slab(grid, n_cpu)
        self.cells = [p.n_cells for p in parts]
        self.base = {}
        self.live = {}
        for r in ranks:
            m, ifs = lrb.assemble_poisson(parts[r])
            self.base[r] = (m, ifs)
            if pinned:
                import torch
                pin = lambda a: self._pin(torch, a)  # noqa: E731
                diag = pin(m.diag)
                mm = lrb.LduMatrix(m.n_cells, m.lower_addr, m.upper_addr, diag,
                                   pin(m.lower_val), pin(m.upper_val))
                ifp = [lrb.InterfaceBlock(b.neighbor_rank, b.rows, b.cols_remote, pin(b.values))
                       for b in ifs]
                self.live[r] = (mm, ifp, diag)
            parts[r] = None   # drop the mesh (faces live on in the LDU matrix)
        self.n_cells = grid.total_cells

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


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch

    import paper_2510_08536_b200 as lrb
    from paper_2510_08536_b200 import _native

    rank, world, local_rank = dist_env()
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
    prob = Problem(N, n_cpu, range(n_cpu))
    pm = lrb.make_partition_map(prob.cells, alpha)
    log(f"[bench] inputs {time.monotonic() - t0:.1f}s; n_cpu={n_cpu} alpha={alpha}")
    n_steps = args.warmup + args.steps
    steps = list(range(2, 2 + n_steps))
    rec = {"e2e_ms": [], "wall_ms": [], "iters": [], "value_ms": [], "scatter_ms": [],
           "solve_ms": [], "kernel_ms": [], "checks": [], "launches": 0, "create_s": 0.0}
    sampler = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))

    def program(ctx):
        r = ctx.rank
        m0, if0 = prob.base[r]
        tc = time.monotonic()
        system = lrb.repartition(m0, if0, pm, ctx)
        ctx.barrier()
        if r == 0:
            rec["create_s"] = time.monotonic() - tc
        b = Problem._pin(torch, np.ones(system.matrix.n_owned)) if system.is_owner else None
        # ---------------- e2e: public API, host buffers ----------------------
        for i, step in enumerate(steps):
            m_s, if_s = prob.produce(r, step)
            ctx.barrier()
            if r == 0:
                if i == args.warmup:
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
                if i >= args.warmup:
                    rec["e2e_ms"].append(system.part.elapsed_ms())
                    rec["wall_ms"].append(wall)
                    rec["iters"].append(rep.iterations)
                    rec.setdefault("e2e_update_wall_ms", []).append((tu - tw) * 1e3)
                    rec.setdefault("e2e_solve_wall_ms", []).append((te - tu) * 1e3)
                    rec.setdefault("e2e_solve_kernel_ms", []).append(rep.device_ms)
                if i == n_steps - 1:
                    rec["launches"] = _native.lrb_launch_count() - rec["l0"]
        ctx.barrier()
        if r == 0:
            sampler.__exit__()
        # ---------------- value: device-resident (HBM) inputs ---------------
        for i, step in enumerate(steps):
            m_s, if_s = prob.produce(r, step)
            lrb.update(system, m_s, if_s, "direct")     # untimed: coefficients -> HBM
            ctx.barrier()
            if r == 0:
                part, team = system.part, system.team
                part.sync()
                part.mark()
                part.apply_scatter()
                part.mark()
                _, rep, hist = team.solve(method, None, TOL, MAX_ITER, want_x=False,
                                          hist_cap=MAX_ITER)
                t_sc = part.elapsed_ms()
                part.mark()
                part.sync()
                if i >= args.warmup:
                    rec["scatter_ms"].append(t_sc)
                    rec["kernel_ms"].append(rep.device_ms)
                    rec["value_ms"].append(t_sc + rep.device_ms)
                    rec["checks"].append(n_checks(hist, rep.iterations, TOL))
                    rec.setdefault("value_iters", []).append(rep.iterations)
            ctx.barrier()
        if r == 0:
            p = system.part.plan
            rec["plan"] = (p.n, p.nnz_local + p.nnz_nonlocal, p.n_halo, p.n_buf)
            rec["kernel_info"] = system.team.kernel_info(method)
        return None

    lrb.run_world(n_cpu, program)
    log(f"[bench] ours done ({time.monotonic() - t0:.1f}s)")
    return finish_line(args, rec, method, desc.format(n_cpu=n_cpu, n_gpu=n_gpu, alpha=alpha, N=N, cells=f"{N ** 3 / 1e6:.3g}M"), N,
                       n_cpu, alpha, sampler)


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
    dist.init_process_group("gloo")
    # one GPU per process; on a 1-GPU box the ranks share it (time-sliced,
    # correctness only — the protocol is the same as over NVLink)
    local_rank = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
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
    prob = Problem(N, n_cpu, layout.cpu_ranks)
    owner = DistributedOwner(layout, {r: prob.base[r] for r in layout.cpu_ranks})
    dist.barrier()
    create_s = max_over_ranks(time.monotonic() - t0)
    b = [Problem._pin(torch, np.ones(p.n)) for p in owner.parts]
    n_steps = args.warmup + args.steps
    steps = list(range(2, 2 + n_steps))
    rec = {"e2e_ms": [], "wall_ms": [], "value_ms": [], "scatter_ms": [], "kernel_ms": [],
           "checks": [], "value_iters": [], "launches": 0, "create_s": create_s}
    sampler = ClockSampler(local_rank)
    part = owner.parts[0]
    for i, step in enumerate(steps):
        live = {r: prob.produce(r, step) for r in layout.cpu_ranks}
        torch.cuda.synchronize()
        dist.barrier()
        if i == args.warmup:
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
        if i >= args.warmup:
            rec["e2e_ms"].append(e2e)
            rec["wall_ms"].append(wall)
    rec["launches"] = _native.lrb_launch_count() - l0
    dist.barrier()
    sampler.__exit__()
    for i, step in enumerate(steps):
        owner.update({r: prob.produce(r, step) for r in layout.cpu_ranks}, "direct")
        for p in owner.parts:
            p.sync()
        dist.barrier()
        part.mark()
        for p in owner.parts:
            p.apply_scatter()
        part.mark()
        _, rep, hist = owner.team.solve(method, None, TOL, MAX_ITER, want_x=False,
                                        hist_cap=MAX_ITER)
        t_sc = max_over_ranks(part.elapsed_ms())
        kms = max_over_ranks(rep.device_ms)
        if i >= args.warmup:
            rec["scatter_ms"].append(t_sc)
            rec["kernel_ms"].append(kms)
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
    line = finish_line(args, rec, method, desc.format(n_cpu=n_cpu, n_gpu=n_gpu, alpha=alpha, N=N, cells=f"{N ** 3 / 1e6:.3g}M"), N,
                       n_cpu, alpha, sampler)
    line["config"]["max_part_rows"] = int(sizes)
    line["config"]["parallelism"] = f"{n_gpu} GPU parts, NVLink peer-memory halo + reductions"
    dist.barrier()
    dist.destroy_process_group()
    return line if rank == 0 else None


def kernel_name(info, method):
    """The solve kernel that ran (lrb_team_kernel_info): streaming or classic."""
    jac = "true" if method in ("pcg", "pcg1") else "false"
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
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(value, 4), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference cavity generator, "
                                                    "closed form)",
        "config": {"workload": desc, "n_cells": N ** 3, "n_cpu": n_cpu, "alpha": alpha,
                   "mode": args.mode, "method": method, "tol": TOL,
                   "timesteps": f"{2 + args.warmup}..{1 + args.warmup + args.steps}",
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
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as fh:
                t = json.load(fh).get(args.workload)
            if t:
                # ncu DRAM bytes per algorithmic byte of the solve kernel, applied
                # to this run's launches (same kernel, same config)
                line["roofline"]["traffic"] = int(t["dram_bytes_per_alg_byte"] *
                                                  line["roofline"]["alg_bytes_per_launch"])
                line["roofline"]["traffic_note"] = t.get("note")
                # the same kernel time against the bytes DRAM actually moved
                dram_gbs = line["roofline"]["traffic"] / (line["roofline"]["kernel_ms"] * 1e-3) / 1e9
                line["roofline"]["dram_achieved"] = round(dram_gbs, 1)
                line["roofline"]["dram_frac"] = round(dram_gbs / line["roofline"]["peak"], 4)
        except Exception:  # noqa: BLE001
            pass
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
    prob = Problem(N, n_cpu, range(n_cpu))
    pm = lrb.make_partition_map(prob.cells, alpha)
    mom = {}
    for r in range(n_cpu):   # momentum LDU on the same addressing, pinned value arrays
        m, ifs = prob.base[r]
        eu, el = momentum_eps(m, r)
        up = Problem._pin(torch, np.zeros(m.n_faces))
        lo = Problem._pin(torch, np.zeros(m.n_faces))
        dg = Problem._pin(torch, np.full(m.n_cells, 6.5))
        mm = lrb.LduMatrix(m.n_cells, m.lower_addr, m.upper_addr, dg, lo, up)
        mom[r] = (mm, ifs, eu, el, up, lo)
    log(f"[bench c4] inputs {time.monotonic() - t0:.1f}s; N={N} n_cpu={n_cpu} alpha={alpha}")
    n_steps = args.warmup + args.steps
    steps = list(range(2, 2 + n_steps))
    rec = {"e2e_ms": [], "value_ms": [], "kernel_ms": [], "alg": [], "iters_p": [], "iters_m": [],
           "launches": 0, "create_s": 0.0}
    sampler = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))

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
        for i, step in enumerate(steps):
            m_s, if_s = produce_mom(r, step)
            p_s, pif_s = prob.produce(r, step)
            ctx.barrier()
            if r == 0:
                if i == args.warmup:
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
                if i >= args.warmup:
                    rec["e2e_ms"].append((time.perf_counter() - tw) * 1e3)
                    rec["iters_m"].append(its)
                    rec["iters_p"].append(rep.iterations)
                if i == n_steps - 1:
                    rec["launches"] = _native.lrb_launch_count() - rec["l0"]
        ctx.barrier()
        if r == 0:
            sampler.__exit__()
        # ---------------- value: device-resident (HBM) inputs ---------------
        for i, step in enumerate(steps):
            lrb.update(sm, *produce_mom(r, step), "direct")   # untimed: coefficients -> HBM
            lrb.update(sp, *prob.produce(r, step), "direct")
            ctx.barrier()
            if r == 0:
                tot = 0.0
                kms = 0.0
                alg = 0
                pln = sm.part.plan
                n, nnz, h = pln.n, pln.nnz_local + pln.nnz_nonlocal, pln.n_halo
                for part, team, method, rhs in ((sm.part, sm.team, "bicgstab", bs), (sp.part, sp.team, "pcg",
                                                                                     [bp])):
                    part.sync()
                    part.mark()
                    part.apply_scatter()
                    part.mark()
                    tot += part.elapsed_ms()
                    alg += 20 * pln.n_buf
                    for b in rhs:
                        _, rep, hist = team.solve(method, [b], TOL, MAX_ITER, want_x=False, hist_cap=MAX_ITER)
                        tot += rep.device_ms
                        kms += rep.device_ms
                        ck = n_checks(hist, rep.iterations, TOL)
                        alg += (bicgstab_bytes(n, nnz, h, rep.iterations, ck) if method == "bicgstab"
                                else solve_bytes(n, nnz, h, rep.iterations, ck, "pcg"))
                if i >= args.warmup:
                    rec["value_ms"].append(tot)
                    rec["kernel_ms"].append(kms)
                    rec["alg"].append(alg)
            ctx.barrier()
        if r == 0:
            p = sp.part.plan
            rec["plan"] = (p.n, p.nnz_local + p.nnz_nonlocal, p.n_halo, p.n_buf)
            rec["kinfo"] = {"bicgstab": sm.team.kernel_info("bicgstab"), "pcg": sp.team.kernel_info("pcg")}
        return None

    lrb.run_world(n_cpu, program)
    log(f"[bench c4] done ({time.monotonic() - t0:.1f}s)")
    n, nnz, h, n_buf = rec["plan"]
    peak, peak_kind = measured_peak()
    value = float(np.mean(rec["value_ms"]))
    achieved = float(np.mean([a / (ms * 1e-3) / 1e9 for a, ms in zip(rec["alg"], rec["value_ms"])]))
    desc = WORKLOADS["c4"][3].format(N=N, cells=f"{N ** 3 / 1e6:.3g}M", n_cpu=n_cpu, n_gpu=args.gpus,
                                      alpha=alpha)
    return {
        "metric": METRIC, "value": round(value, 4), "unit": "ms/timestep", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value, 4),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference cavity generator; momentum LDU per SURVEY §8d)",
        "config": {"workload": desc, "n_cells": N ** 3, "n_cpu": n_cpu, "alpha": alpha, "mode": "direct",
                   "tol": TOL, "timesteps": f"{2 + args.warmup}..{1 + args.warmup + args.steps}",
                   "l2": "inputs larger than L2 (no flush needed)"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None, "peak_kind": peak_kind,
                     "kernel": "whole timestep: 2 scatters + 3 team_bicgstab_stream_kernel + "
                               "team_cg_stream_kernel<JAC=true>",
                     "kernel_geometry": rec.get("kinfo"),
                     "alg_bytes_per_launch": int(np.mean(rec["alg"])),
                     "kernel_ms": round(float(np.mean(rec["kernel_ms"])), 4)},
        "e2e": {"value": round(float(np.mean(rec["e2e_ms"])), 4), "unit": "ms/timestep",
                "timer": "host wall clock around the synchronous API calls of rank 0",
                "h2d_bytes_per_step": int(2 * 8 * n_buf + 8 * n * (MOM_RHS + 1)),
                "d2h_bytes_per_step": int(8 * n * (MOM_RHS + 1))},
        "breakdown": {"iterations_momentum": rec["iters_m"], "iterations_pressure": rec["iters_p"],
                      "create_s": round(rec["create_s"], 2)},
        "gpu_launches": int(rec["launches"]),
        "clocks": sampler.summary(),
    }


# ---------------------------------------------------------------------------
# CPU baseline: the reference algorithm (oracle port) on the host cores
# ---------------------------------------------------------------------------
def cpu_baseline(args, iters_per_step=None, full_warmup=False):
    from oracle import cavity as ocav
    from oracle import krylov
    from oracle.pipeline import OraclePipeline

    N, _, method_default, desc = WORKLOADS[args.workload]
    n_gpu = args.gpus
    n_cpu = args.rpg * n_gpu
    alpha = args.rpg
    t0 = time.monotonic()
    probs = ocav.cavity_problems((N, N, N), n_cpu)
    offsets = np.concatenate(([0], np.cumsum([p.n for p in probs]))).astype(np.int64)
    pipe = OraclePipeline(probs, offsets, alpha)
    t_create = time.monotonic() - t0
    table = iters_per_step or _iteration_table(N, n_cpu, alpha)
    samples = []
    timed = list(range(2 + args.warmup, 2 + args.warmup + args.steps))
    n_warm = args.warmup if full_warmup else 1
    steps = list(range(timed[0] - n_warm, timed[0])) + timed
    k_iter = 3
    for i, step in enumerate(steps):
        ps = [ocav.perturb(p, step) for p in probs]
        ts = time.perf_counter()
        pipe.update(ps)
        t_up = time.perf_counter() - ts
        S = pipe.system
        bs = pipe.rhs_ones()
        ts = time.perf_counter()
        krylov.cg(S, bs, 1e-300, k_iter, jacobi=(method_default == "pcg"))
        t_it = (time.perf_counter() - ts) / k_iter
        ts = time.perf_counter()
        S.spmv(bs)
        t_spmv = time.perf_counter() - ts
        if step in table:
            its = table[step]
            checks = its // 10 + (1 if its % 10 else 0)
            ms = (t_up + its * t_it + checks * t_spmv) * 1e3
        else:   # small case: just run the whole solve
            ts = time.perf_counter()
            krylov.cg(S, bs, TOL, MAX_ITER, jacobi=(method_default == "pcg"))
            ms = (t_up + time.perf_counter() - ts) * 1e3
        if i >= n_warm:
            samples.append(ms)
        if time.monotonic() - t0 > args.cpu_budget_s and len(samples) >= 1:
            break
    return {"value": round(float(np.mean(samples)), 2), "unit": "ms/timestep", "cores": 1,
            "kind": "port",
            "sample": (f"oracle/ numpy port of the reference path, {N}^3 {n_cpu} ranks -> "
                       f"{n_gpu} part(s): full update + {k_iter} timed "
                       f"{'Jacobi-PCG' if method_default == 'pcg' else 'CG'} iterations + 1 SpMV "
                       f"per step, scaled to the step's iteration count; create "
                       f"{t_create:.1f}s excluded; {len(samples)} steps"),
            "create_s": round(t_create, 1)}


def _iteration_table(N, n_cpu, alpha):
    path = os.path.join(ROOT, "tests", "golden", f"iters_{N}_r{n_cpu}_a{alpha}.json")
    if not os.path.exists(path):
        cand = [f for f in os.listdir(os.path.join(ROOT, "tests", "golden"))
                if f.startswith(f"iters_{N}_")]
        if not cand:
            return {}
        path = os.path.join(ROOT, "tests", "golden", cand[0])
    with open(path) as fh:
        return {row["step"]: row["iterations"] for row in json.load(fh)["steps"]}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    args.cpu_budget_s = max(args.cpu_budget_s, 240.0)
    base = cpu_baseline(args, full_warmup=True)
    N, _, method_default, desc = WORKLOADS[args.workload]
    n_cpu = args.rpg * args.gpus
    return {
        "metric": METRIC, "value": base["value"], "unit": "ms/timestep", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": base["value"],
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": desc.format(n_cpu=n_cpu, n_gpu=args.gpus, alpha=args.rpg, N=N,
                                           cells=f"{N ** 3 / 1e6:.3g}M"),
                   "n_cells": N ** 3, "n_cpu": n_cpu, "alpha": args.rpg, "method": method_default,
                   "tol": TOL},
        "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": base["value"], "unit": "ms/timestep", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c3")
    ap.add_argument("--rpg", type=int, default=None, help="CPU ranks per GPU (alpha)")
    ap.add_argument("--n", type=int, default=None, help="cavity edge (c4; default 300)")
    ap.add_argument("--mode", choices=("direct", "staged"), default="direct")
    ap.add_argument("--method", choices=("cg", "pcg", "pcg1"), default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=60.0)
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
        if line is not None and args.workload == "c4":
            line["cpu_baseline"] = None
            line["cpu_baseline_note"] = ("the CPU reference arm is measured on the headline workload (c3); "
                                         "a 300^3 oracle pipeline does not fit the bench's minutes budget")
        elif line is not None and rank == 0 and world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = {k: v for k, v in cpu_baseline(args, {
                2 + args.warmup + i: it for i, it in enumerate(line["breakdown"]["iterations"])
            }).items() if k != "create_s"}
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
