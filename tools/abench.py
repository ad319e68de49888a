"""Phase-A-only timing with a diagnostics build (-DLRB_ABENCH=K [-DLRB_NOCOMPUTE=1]):
    LRB_LIB=build/lib_abench.so python tools/abench.py
prints the mean release-to-release time of the K back-to-back SpMV phases."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import Problem  # noqa: E402


def main():
    import paper_2510_08536_b200 as lrb
    from paper_2510_08536_b200.device import Team
    prob = Problem(200, 8, range(8))
    pm = lrb.make_partition_map(prob.cells, 8)
    holder = {}

    def program(ctx):
        s = lrb.repartition(*prob.base[ctx.rank], pm, ctx)
        lrb.update(s, *prob.produce(ctx.rank, 6), "direct")
        if s.is_owner:
            s.part.sync()
            holder["parts"] = [s.part]
            holder["keep"] = s
        return None

    lrb.run_world(8, program)
    team = Team(holder["parts"])
    team.profile(400)
    bs = [np.ones(p.n) for p in holder["parts"]]
    for _ in range(3):
        try:
            team.solve("pcg", bs, 1e-6, 2000, want_x=False, hist_cap=2000)
        except Exception as e:   # the diagnostics build skips the convergence logic
            print("solve:", type(e).__name__, str(e)[:80])
        k = int(os.environ.get("STAMPS", "2"))
        ts = team.phase_times_ns().reshape(-1, k)
        d = np.diff(ts[:, -1]) / 1e3
        if k == 3:
            print(f"  arrival->part_value {np.mean(ts[2:, 1] - ts[2:, 0]) / 1e3:.2f} us, "
                  f"part_value->release {np.mean(ts[2:, 2] - ts[2:, 1]) / 1e3:.2f} us")
        print(f"{os.path.basename(os.environ.get('LRB_LIB', 'default'))}: phases {len(d)}, "
              f"A mean {d[1:].mean():.2f} us (min {d[1:].min():.2f}), sync {np.mean(ts[2:, -1] - ts[2:, 0]) / 1e3:.2f} us")


if __name__ == "__main__":
    main()
