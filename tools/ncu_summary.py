#!/usr/bin/env python
"""Summarise ncu output for profiles/.

    python tools/ncu_summary.py launches <launches.csv>      # per-kernel share of a launch list
    python tools/ncu_summary.py full <report.ncu-rep>        # key metrics + top stall reasons per profiled launch

Reads files written by the gpurun commands in tools/gpu_*.sh (ncu runs on the
GPU box; the report is read back here with `ncu -i`).
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active_lanes/warp_inst"),
    ("sm__inst_executed.avg.per_cycle_active", "ipc"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
]


def launches(path: str) -> None:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    agg = defaultdict(list)
    for r in rows:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        agg[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':26s} {'launches':>8s} {'total_ms':>10s} {'avg_us':>10s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{k:26s} {len(v):8d} {sum(v) / 1e6:10.3f} {sum(v) / len(v) / 1e3:10.1f} {sum(v) / tot:6.3f}")
    print(f"{'TOTAL':26s} {sum(len(v) for v in agg.values()):8d} {tot / 1e6:10.3f}")


def full(path: str) -> None:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, rows = r[0], r[1], r[2:]
    unit = dict(zip(hdr, units))
    for row in rows:
        d = dict(zip(hdr, row))
        print(f"[{d['ID']}] {d['Kernel Name'].split('(')[0]}  grid={d.get('launch__grid_size')} block={d.get('launch__block_size')}")
        for k, name in KEYS:
            if k in d:
                print(f"    {name:24s} {d[k]:>14s} {unit.get(k, '')}")
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v.replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("    stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
