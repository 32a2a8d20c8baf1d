#!/usr/bin/env python
"""Rank CUDA source lines of one kernel by stall samples / executed instructions.
   ncu -i rep --page source --print-source cuda,sass --csv -k regex:K --launch-count 1 > src.csv
   python tools/ncu_lines.py src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
cur = None
out = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit() and len(r) > 8 and r[2] == "-":
        try:
            s = int(r[4]); ie = int(r[7]); te = int(r[8])
        except ValueError:
            continue
        out.append((s, ie, te, cur, r[0], r[1].strip()[:100]))
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
tt = sum(o[2] for o in out) or 1
print(f"samples {ts}  warp-inst {ti}  thread-inst {tt}  avg lanes {tt / ti:.1f}")
for o in sorted(out, reverse=True)[:top]:
    print(f"{o[0] / ts * 100:5.1f}% smp {o[1] / ti * 100:5.1f}% inst lanes={o[2] / max(1, o[1]):5.1f} {o[3]}:{o[4]} {o[5]}")
