"""Measured cost-model curves: the C3 ranks-per-GPU sweep on
one B200 written as the reference cost model's CSV (n, t_as, t_ls), so its
`load_curves_csv` / advise path can read our timings.

    python tools/curves.py [--rpg 1 2 4 8 16] [--steps 5] [--out profiles/r2_curves_c3.csv]

n = CPU ranks per GPU (alpha); t_as = update wall time per timestep (the
ranks' coefficient upload + scatter, s); t_ls = solve wall time per timestep
(s).  Each point is one `bench.py --rpg n` run (e2e breakdown); the full
bench lines go to <out>.jsonl."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rpg", type=int, nargs="*", default=[1, 2, 4, 8, 16])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_curves_c3.csv"))
    args = ap.parse_args()
    from paper_2510_08536_b200.verify import write_curves_csv
    rows = []
    for n in args.rpg:
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--rpg", str(n), "--steps",
                              str(args.steps), "--no-cpu-baseline", "--no-pageable"],
                             capture_output=True, text=True, cwd=ROOT, timeout=900)
        line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
        if not line:
            sys.stderr.write(out.stderr[-2000:])
            raise SystemExit(f"bench --rpg {n} failed")
        full = json.loads(line[-1])
        with open(args.out + ".jsonl", "a") as fh:
            fh.write(json.dumps(full) + "\n")
        e2e = full["e2e"]
        rows.append((n, e2e["update_wall_ms"] / 1e3, e2e["solve_wall_ms"] / 1e3))
        print(json.dumps({"n": n, "t_as_s": rows[-1][1], "t_ls_s": rows[-1][2]}), flush=True)
    write_curves_csv(args.out, rows)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
