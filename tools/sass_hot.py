"""Summarise an ncu report's SASS source page: stall reasons, opcode mix,
hottest instructions.   python tools/sass_hot.py gpurun_out/prof.ncu-rep [N]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
ix = {k: i for i, k in enumerate(h)}
S = 'Warp Stall Sampling (All Samples)'
I = 'Instructions Executed'
stall_cols = [k for k in h if k.startswith('stall_') and 'Not Issued' not in k]
tot = {k: sum(int(r[ix[k]] or 0) for r in data) for k in stall_cols}
T = sum(tot.values()) or 1
print("stalls:", ", ".join(f"{k[6:]} {v / T * 100:.1f}%" for k, v in
                           sorted(tot.items(), key=lambda x: -x[1])[:8]))
c = Counter()
for r in data:
    t = r[1].split()
    op = t[1] if t[0].startswith('@') else t[0]
    c[op.split('.')[0]] += int(r[ix[I]] or 0)
ti = sum(c.values())
print(f"warp instructions {ti:.3e}:", ", ".join(f"{k} {v / ti * 100:.1f}%" for k, v in c.most_common(16)))
ts = sum(int(r[ix[S]] or 0) for r in data) or 1
for r in sorted(data, key=lambda r: -int(r[ix[S]] or 0))[:top_n]:
    s = int(r[ix[S]])
    st = sorted(((int(r[ix[k]] or 0), k[6:]) for k in stall_cols), reverse=True)[:2]
    print(f"{r[0][-5:]} {s / ts * 100:5.1f}% n={int(r[ix[I]]):>10d} {r[1].strip()[:58]:58s} "
          f"{st[0][1]}:{st[0][0]} {st[1][1]}:{st[1][0]}")
