"""Warp-stall samples aggregated per CUDA source line (file, line) of one kernel in an ncu report
(measurement tool).  Usage: python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> [file-substr] [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
fsub = sys.argv[3] if len(sys.argv) > 3 else ""
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, line, text = "?", None, ""
agg = defaultdict(lambda: [0, defaultdict(int), ""])
hdr = None
for r in rows:
    if r and r[0] in ("File Name", "File Path"):
        fname = r[1]
        continue
    if "Warp Stall Sampling (All Samples)" in r:
        hdr = r
        iA = hdr.index("Warp Stall Sampling (All Samples)")
        cols = [(i, c[6:]) for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        line, text = int(r[0]), r[1]
        continue
    try:
        n = int(float(r[iA]))
    except ValueError:
        continue
    a = agg[(fname, line)]
    a[0] += n
    a[2] = text
    for i, c in cols:
        try:
            a[1][c] += int(float(r[i]))
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values())
print("samples", tot)
sel = [(k, v) for k, v in agg.items() if fsub in k[0]]
print("samples in", fsub or "all", sum(v[0] for _, v in sel))
for (f, l), v in sorted(sel, key=lambda kv: -kv[1][0])[:top]:
    st = sorted(v[1].items(), key=lambda x: -x[1])[:3]
    print(f"{v[0]:6d} {f.split('/')[-1]}:{l} {v[2].strip()[:64]:64s} {st}")
