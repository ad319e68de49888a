"""profiles/r2_sass_summary.md: per-kernel SASS opcode counts of the in-tree
library (cuobjdump -sass, sm_100a).  Run in the build container."""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2510_08536_b200", "libldurepart_b200.so")
COLS = [("UBLKCP (bulk copy)", r"UBLKCP"), ("UBLKPF (L2 prefetch)", r"UBLKPF"), ("SYNCS (mbarrier)", r"SYNCS"),
        ("DFMA", r"DFMA"), ("DMUL", r"DMUL"), ("DADD", r"DADD"), ("LDS", r"LDS"),
        ("local ld/st", r"(LDL|STL)"), ("UTMA*", r"UTMA"), ("UTC* (tcgen05)", r"UTC")]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        if cur and re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
            funcs[cur].append(line.split("*/", 1)[1].split(";")[0].strip())
    names = {}
    for f in funcs:
        d = subprocess.run(["c++filt", f], capture_output=True, text=True).stdout.strip()
        names[f] = d
    rows = []
    for f, ins in funcs.items():
        ops = [i.split()[0] if not i.startswith("@") else i.split()[1] for i in ins if i]
        cnt = [sum(1 for o in ops if re.match(p, o)) for _, p in COLS]
        rows.append((len(ops), names[f], cnt))
    rows.sort(key=lambda r: -r[0])
    out = ["# SASS summary of libldurepart_b200.so (round 2, `cuobjdump -sass`, sm_100a)", "",
           "| kernel | instructions | " + " | ".join(c for c, _ in COLS) + " |",
           "|---|---|" + "---|" * len(COLS)]
    for n, name, cnt in rows:
        out.append(f"| `{name}` | {n} | " + " | ".join(str(c) for c in cnt) + " |")
    path = os.path.join(ROOT, "profiles", "r2_sass_summary.md")
    note = open(path).read().rstrip().split("\n\n")[-1] if os.path.exists(path) else ""   # closing note
    open(path, "w").write("\n".join(out) + "\n\n" + note)
    print("\n".join(out[:8]))


if __name__ == "__main__":
    sys.exit(main())
