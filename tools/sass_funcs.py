"""SASS size (instructions) of every function body in a cubin (kernel entries and the non-inlined
device functions they call), from nvdisasm.  Measurement tool for instruction-cache budgets.
Usage: python tools/sass_funcs.py <cubin> [name-substr]"""
import re
import subprocess
import sys

out = subprocess.run(["nvdisasm", sys.argv[1]], capture_output=True, text=True).stdout
sub = sys.argv[2] if len(sys.argv) > 2 else ""
cur, n = None, 0
res = []
for ln in out.splitlines():
    m = re.match(r"^(\$?[_A-Za-z][_A-Za-z0-9$.]*):\s*$", ln)
    if m and not m.group(1).startswith(".L"):
        if cur:
            res.append((cur, n))
        cur, n = m.group(1), 0
        continue
    if cur and re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+[A-Z@]", ln):
        n += 1
if cur:
    res.append((cur, n))
for name, c in res:
    if sub in name:
        short = re.sub(r"_ZN\d+_INTERNAL_\w+?asr", "asr", name)
        print(f"{c:7d} instr {c * 16 / 1024:7.1f} KB  {short[-110:]}")
