"""Per-phase device time of one solve (globaltimer at every team-barrier
release, lrb_team_profile), for the streaming and the classic solver.

    python tools/phase_profile.py [--n 200] [--ranks 8] [--step 6] [--method pcg]

Prints one JSON line per solver family: phase counts, mean microseconds per
phase kind and the HBM GB/s each phase reaches on its algorithmic bytes
(A = 12nnz+4(n+1)+16n (+16n p_old/z on the fly), B = 48n (+16n
PCG), C = 12nnz+4(n+1)+16n).
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import MAX_ITER, TOL, Problem  # noqa: E402


def phase_kinds(hist, iterations, tol):
    kinds = ["init"]
    for it in range(1, iterations + 1):
        kinds += ["A", "B"]
        rec = hist[it - 1] if it - 1 < len(hist) else 0.0
        if rec <= tol or it % 10 == 0:
            kinds.append("C")
    return kinds


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200)
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--step", type=int, default=6)
    ap.add_argument("--method", default="pcg")
    ap.add_argument("--repeat", type=int, default=3)
    ap.add_argument("--alpha", type=int, default=None, help="ranks per GPU part (default: all -> 1 part)")
    args = ap.parse_args()
    import paper_2510_08536_b200 as lrb
    from paper_2510_08536_b200.device import Team
    prob = Problem(args.n, args.ranks, range(args.ranks))
    pm = lrb.make_partition_map(prob.cells, args.alpha or args.ranks)
    holder = {"keep": []}

    def program(ctx):
        s = lrb.repartition(*prob.base[ctx.rank], pm, ctx)
        lrb.update(s, *prob.produce(ctx.rank, args.step), "direct")
        if s.is_owner:
            s.part.sync()
            parts = s.comm.allgather(s.part)   # every owner part on this one GPU
            holder["keep"].append(s)
            if s.comm.group_rank == 0:
                holder["parts"] = parts
                holder["plan"] = parts[0].plan
        return None

    lrb.run_world(args.ranks, program)
    parts = holder["parts"]
    plan = holder["plan"]
    n, nnz, h = plan.n, plan.nnz_local + plan.nnz_nonlocal, plan.n_halo
    bytes_of = {"init": 32 * n, "A": 12 * nnz + 4 * (n + 1) + 32 * n + 8 * h,
                "B": 48 * n + (16 * n if args.method == "pcg" else 0),
                "C": 12 * nnz + 4 * (n + 1) + 16 * n + 8 * h}
    for family in ("stream", "classic"):
        if family == "classic":
            os.environ["LRB_SOLVER"] = "classic"
        else:
            os.environ.pop("LRB_SOLVER", None)
        team = Team(parts)
        team.profile(4 * MAX_ITER)
        bs = [np.ones(p.n) for p in parts]
        per = {}
        total = []
        for _ in range(args.repeat):
            _, rep, hist = team.solve(args.method, bs, TOL, MAX_ITER, want_x=False, hist_cap=MAX_ITER)
            ts = team.phase_times_ns().reshape(-1, 2)   # (last arrival, release) per phase
            kinds = phase_kinds(hist, rep.iterations, TOL)
            kinds += ["X"] * (len(ts) - len(kinds))   # the lazy-x final update phase
            for q in range(1, len(ts)):
                k = kinds[q]
                per.setdefault(k, []).append((ts[q, 1] - ts[q - 1, 1]) / 1e3)
                per.setdefault(k + "_sync", []).append((ts[q, 1] - ts[q, 0]) / 1e3)
            total.append(rep.device_ms)
        out = {"family": family, "iterations": rep.iterations, "device_ms": round(float(np.mean(total)), 4),
               "info": team.kernel_info(args.method)}
        cnt = team.wait_counters(args.method)
        if cnt.size:
            # mean over CTAs, in us at the sampled SM clock, per phase kind
            mhz = float(os.environ.get("LRB_SM_MHZ", "1965"))
            names = ("data_wait", "end_bar", "stage_wait", "team_bar", "body", "reduce", "slot_wait",
                     "issue")
            out["waits_us"] = {kind: {nm: round(float(cnt[:, ki, wi].mean()) / mhz, 1)
                                      for wi, nm in enumerate(names)}
                               for ki, kind in enumerate(("init", "A", "B", "C"))}
            tl = team.last_timeline_ns.astype(np.float64)
            t0 = tl[:, 0].min()
            rel = (tl - t0) / 1e3
            names_tl = ("entry", "issuer_fenced", "issuer_hdr", "issuer_issued", "first_data",
                        "consumers_done", "reducer_done", "barrier_out")
            out["last_A_timeline_us"] = {}
            for j, nm in enumerate(names_tl):
                ok = tl[:, j] >= tl[:, 0]   # stamps left over from an earlier phase A are stale
                if not ok.any():
                    continue
                col = np.where(ok, rel[:, j], np.nan)
                out["last_A_timeline_us"][nm] = {
                    "min": round(float(np.nanmin(col)), 2), "mean": round(float(np.nanmean(col)), 2),
                    "max": round(float(np.nanmax(col)), 2), "argmax_cta": int(np.nanargmax(col)),
                    "ctas": int(ok.sum())}
            # the slowest CTA per counter (stragglers set the phase time)
            out["waits_us_max"] = {kind: {nm: round(float(cnt[:, ki, wi].max()) / mhz, 1)
                                          for wi, nm in enumerate(names)}
                                   for ki, kind in enumerate(("init", "A", "B", "C"))}
        for k, v in sorted(per.items()):
            us = float(np.mean(v))
            out[k] = {"count": len(v) // args.repeat, "us": round(us, 2)}
            if k in bytes_of:
                out[k]["gbs"] = round(bytes_of[k] / (us * 1e-6) / 1e9, 1)
        print(json.dumps(out), flush=True)
        del team


if __name__ == "__main__":
    main()
