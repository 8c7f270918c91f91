"""Top stalled SASS lines of one kernel in an ncu report (measurement tool).
Usage: python tools/ncu_hot.py <report.ncu-rep> <kernel-regex> [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Source" in r and "Warp Stall Sampling (All Samples)" in r)
k = rows.index(hdr)
data = [r for r in rows[k + 1:] if len(r) == len(hdr)]
iS, iA = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
def num(x):
    try:
        return int(float(x))
    except ValueError:
        return 0
tot = sum(num(r[iA]) for r in data)
print("samples", tot)
for r in sorted(data, key=lambda r: -num(r[iA]))[:top]:
    st = sorted(((c[6:], num(r[hdr.index(c)])) for c in cols if num(r[hdr.index(c)]) > 0), key=lambda x: -x[1])[:3]
    print(f"{num(r[iA]):5d} {r[0][-5:]} {r[iS].strip()[:70]:70s} {st}")
