"""Wall time of the create path (repartition) by stage, one GPU.

    python tools/create_profile.py [--n 300] [--ranks 16]

Times, on the owner thread: source description (_Source), native plan build
(lrb_plan_build_ldu), part create (arena layout + index uploads), initial
transfer + scatter, halo plan and team create (stage headers, push runs)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=300)
    ap.add_argument("--ranks", type=int, default=16)
    args = ap.parse_args()
    import paper_2510_08536_b200 as lrb
    from paper_2510_08536_b200 import repart
    t0 = time.monotonic()
    parts = lrb.decompose_slab(lrb.StructuredGrid(args.n, args.n, args.n), args.ranks)
    asm = [lrb.assemble_poisson(p) for p in parts]
    pm = lrb.make_partition_map([p.n_cells for p in parts], args.ranks)
    t_gen = time.monotonic() - t0
    times = {}
    orig = {}

    def wrap(mod, name):
        f = getattr(mod, name)
        orig[name] = f

        def g(*a, **k):
            t = time.monotonic()
            try:
                return f(*a, **k)
            finally:
                times[name] = times.get(name, 0.0) + time.monotonic() - t
        setattr(mod, name, g)

    from paper_2510_08536_b200 import device
    wrap(repart, "_owner_plan")
    wrap(repart, "build_halo_plan")
    for cls, meth in ((device.DevicePart, "__init__"), (device.Team, "__init__"),
                      (device.DevicePart, "update_segment"), (device.DevicePart, "join")):
        f = getattr(cls, meth)
        key = f"{cls.__name__}.{meth}"

        def make(f=f, key=key):
            def g(*a, **k):
                t = time.monotonic()
                try:
                    return f(*a, **k)
                finally:
                    times[key] = times.get(key, 0.0) + time.monotonic() - t
            return g
        setattr(cls, meth, make())
    t1 = time.monotonic()
    lrb.run_world(args.ranks, lambda ctx: lrb.repartition(*asm[ctx.rank], pm, ctx) and None)
    total = time.monotonic() - t1
    print(json.dumps({"n": args.n, "ranks": args.ranks, "generator_s": round(t_gen, 2),
                      "repartition_s": round(total, 2),
                      "stages_s (summed over rank threads)": {k: round(v, 3) for k, v in times.items()}}))


if __name__ == "__main__":
    main()
