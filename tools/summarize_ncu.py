"""Summarise ncu captures into profiles/ (run in the build container).

    python tools/summarize_ncu.py --tag r1_c3 --full gpurun_out/prof.ncu-rep \
        --step-json gpurun_out/profile_step.json --launches gpurun_out/launches.csv

Writes profiles/<tag>_summary.md and merges the solve kernel's DRAM traffic
per algorithmic byte into profiles/traffic.json (read by bench.py).
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warps_issue_stalled_barrier_per_warp_active.pct"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {"name": vals[hdr.index("Kernel Name")]}
        for h, u, v in zip(hdr, units, vals):
            if h in KEYS:
                try:
                    d[h] = float(v.replace(",", "")) * SCALE.get(u, 1.0)
                except ValueError:
                    d[h] = v
        kernels.append(d)
    return kernels


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: i for i, h in enumerate(hdr)}
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
        v = float(r[ix["Metric Value"]].replace(",", "")) * SCALE.get(r[ix["Metric Unit"]], 1e-9)
        tot[name] += v
        cnt[name] += 1
    return tot, cnt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--step-json")
    ap.add_argument("--launches")
    ap.add_argument("--workload", default="c3")
    args = ap.parse_args()
    lines = [f"# ncu summary `{args.tag}`", ""]
    step = None
    if args.step_json:   # the JSON line among ncu's own stdout lines
        for line in open(args.step_json):
            if line.startswith("{"):
                step = json.loads(line)
    if step:
        lines += [f"Profiled timestep: step {step['step']}, {step['iterations']} PCG iterations, "
                  f"{step['checks']} true-residual checks; n={step['n']}, nnz={step['nnz']}, "
                  f"SELL entries={step['sell_entries']} ({step['uniform_entries']} in pattern "
                  f"slices); algorithmic bytes of the solve launch = {step['alg_bytes']:.4e}, "
                  f"of one full scatter = {step['scatter_alg_bytes']:.4e}.", ""]
    traffic = {}
    for rep in args.full:
        lines.append(f"## `{os.path.basename(rep)}` (ncu --set full --clock-control none)")
        lines.append("")
        for k in raw(rep):
            dram = k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
            t = k.get("gpu__time_duration.sum", 0)
            lines.append(f"- kernel `{k['name']}`: {t * 1e3:.3f} ms, DRAM {dram / 1e9:.3f} GB "
                         f"({dram / t / 1e9 if t else 0:.0f} GB/s), regs "
                         f"{k.get('launch__registers_per_thread')}, grid {k.get('launch__grid_size')}, "
                         f"warps active {k.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.1f}%, "
                         f"L2 hit {k.get('lts__t_sector_hit_rate.pct', 0):.1f}%, L1 hit "
                         f"{k.get('l1tex__t_sector_hit_rate.pct', 0):.1f}%")
            if step and "team_" in k["name"]:
                ratio = dram / step["alg_bytes"]
                lines.append(f"  - DRAM bytes / algorithmic bytes = {ratio:.3f} "
                             f"(SELL pattern slices skip the 4-byte column stream)")
                traffic[args.workload] = {"dram_bytes_per_alg_byte": ratio,
                                          "note": f"ncu {args.tag}: solve launch of step "
                                                  f"{step['step']}, DRAM {dram:.4e} B for "
                                                  f"{step['alg_bytes']:.4e} algorithmic B"}
            if step and "scatter" in k["name"]:
                seg = step["scatter_alg_bytes"] / 8
                lines.append(f"  - one segment of 8: algorithmic {seg:.4e} B, DRAM/alg = "
                             f"{dram / seg:.3f}")
        lines.append("")
    if args.launches:
        tot, cnt = launches(args.launches)
        s = sum(tot.values())
        lines += ["## Launch list (ncu gpu__time_duration, cold-cache, serialised)", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k in sorted(tot, key=tot.get, reverse=True):
            lines.append(f"| `{k}` | {cnt[k]} | {tot[k] * 1e3:.3f} | {tot[k] / s:.1%} |")
        lines.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{args.tag}_summary.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    if traffic:
        path = os.path.join(ROOT, "profiles", "traffic.json")
        cur = json.load(open(path)) if os.path.exists(path) else {}
        cur.update(traffic)
        json.dump(cur, open(path, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
