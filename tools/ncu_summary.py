"""Summarise ncu outputs into small text files for profiles/ (measurement tool).

  python tools/ncu_summary.py launches <launches.csv>          per-kernel device times of a launch list
  python tools/ncu_summary.py full <report.ncu-rep>             key metrics + top stall sites per kernel
"""
from __future__ import annotations

import csv
import io
import statistics
import subprocess
import sys
from collections import defaultdict


def short(name: str) -> str:
    return name.split("(")[0].split("::")[-1].strip()


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = defaultdict(list)
    order = []
    unit = ""
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        k = short(r[ki])
        if k not in per:
            order.append(k)
        per[k].append(float(r[vi].replace(",", "")))
        unit = r[ui]
    total = sum(statistics.mean(v) for v in per.values())
    out = [f"# launch list: {path}", f"kernel | launches | mean {unit} | min | max | share of step",
           "---|---|---|---|---|---"]
    for k in order:
        v = per[k]
        out.append(f"{k} | {len(v)} | {statistics.mean(v):.0f} | {min(v):.0f} | {max(v):.0f} | "
                   f"{statistics.mean(v) / total:.1%}")
    out.append(f"sum of per-kernel means: {total:.0f} {unit}")
    return "\n".join(out)


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum"]


def full(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = [f"# ncu --set full: {path}"]
    for r in rows[2:]:
        name = short(r[h.index("Kernel Name")])
        out.append(f"\n## {name}")
        for m in METRICS:
            if m in h:
                i = h.index(m)
                out.append(f"- {m}: {r[i]} {units[i]}")
        stalls = []
        for i, m in enumerate(h):
            if m.startswith("smsp__pcsamp_warps_issue_stalled_") and not m.endswith("_not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), m.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        top = ", ".join(f"{n} {v / tot:.0%}" for v, n in sorted(stalls, reverse=True)[:6])
        out.append(f"- warp-state samples: {top}")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else full(path))
