"""Instruction count of one kernel's SASS attributed to source files / line ranges (code-size audit of
latency-bound paths, where instruction-cache misses dominate).  Measurement tool.
Usage: python tools/sass_lines.py <cubin> <kernel-substr> [file:lo-hi ...]"""
import re
import subprocess
import sys
from collections import Counter

cubin, ksub = sys.argv[1], sys.argv[2]
out = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
cur_fn, cur_loc = None, None
per_file = Counter()
per_line = Counter()
total = 0
for ln in out.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur_fn = m.group(1)
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur_loc = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if cur_fn and ksub in cur_fn and re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
        total += 1
        if cur_loc:
            per_file[cur_loc[0]] += 1
            per_line[cur_loc] += 1
print("instructions", total, "bytes", total * 16)
for f, c in per_file.most_common(8):
    print(f"  {f}: {c}")
for spec in sys.argv[3:]:
    f, r = spec.split(":")
    lo, hi = map(int, r.split("-"))
    c = sum(v for (ff, l), v in per_line.items() if ff == f and lo <= l <= hi)
    print(f"  {spec}: {c} instructions ({c * 16} bytes)")
