"""Per-CUDA-source-line instruction and stall attribution of an ncu report
(needs -lineinfo and --import-source on):

    python tools/src_hot.py gpurun_out/prof.ncu-rep [N] [kernel-substring]

Prints the N source lines with the most executed warp instructions, with
their share of stall samples and the top stall reasons."""
import csv
import io
import os
import subprocess
import sys

rep = os.path.abspath(sys.argv[1])
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, cwd="/tmp").stdout
rows = list(csv.reader(io.StringIO(out)))
path, hdr, ix, agg = None, None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        ix = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or not r[0]:
        continue   # sass rows carry an empty line number
    try:
        n = int(r[ix["Instructions Executed"]] or 0)
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, KeyError):
        continue
    stalls = []
    for k, i in ix.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                stalls.append((int(r[i] or 0), k[6:]))
            except ValueError:
                pass
    agg.append((n, s, f"{path}:{r[0]}", r[1].strip()[:80], sorted(stalls, reverse=True)[:2]))
tn = sum(a[0] for a in agg) or 1
ts = sum(a[1] for a in agg) or 1
print(f"warp instructions {tn:.3e}, stall samples {ts}")
for n, s, loc, src, st in sorted(agg, key=lambda a: -a[0])[:top_n]:
    extra = " ".join(f"{k}:{v}" for v, k in st if v)
    print(f"{n / tn * 100:5.1f}% ins {s / ts * 100:5.1f}% smp  {loc:18s} {src}  {extra}")
print("--- by stall samples")
for n, s, loc, src, st in sorted(agg, key=lambda a: -a[1])[:top_n // 2]:
    extra = " ".join(f"{k}:{v}" for v, k in st if v)
    print(f"{n / tn * 100:5.1f}% ins {s / ts * 100:5.1f}% smp  {loc:18s} {src}  {extra}")
