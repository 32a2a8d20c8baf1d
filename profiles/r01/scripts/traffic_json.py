#!/usr/bin/env python
"""profiles/traffic.json from full ncu captures: {"<workload>:<kernel>": dram bytes
(read + write) of the captured launch}.  bench.py reports it as roofline.traffic.

    python tools/traffic_json.py [--out traffic.json] gpurun_out/<tag>/full_<wl>_<kernel>.ncu-rep ...
"""
import csv
import io
import json
import re
import subprocess
import sys
from pathlib import Path

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
args = sys.argv[1:]
out_path = Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
if args[:1] == ["--out"]:
    out_path, args = Path(args[1]), args[2:]
data = json.loads(out_path.read_text()) if out_path.exists() else {}
for rep in args:
    m = re.match(r"full_([^_]+)_(.+)\.ncu-rep$", Path(rep).name)
    if not m:
        continue
    wl, kernel = m.group(1), m.group(2)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    hdr, units, rows = r[0], r[1], r[2:]
    u = dict(zip(hdr, units))
    tot = 0.0
    for row in rows:  # every captured launch: the average per launch
        d = dict(zip(hdr, row))
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(d[k].replace(",", "")) * UNIT.get(u[k], 1)
    data[f"{wl}:{kernel}"] = round(tot / max(1, len(rows)))
    print(wl, kernel, f"{tot / 1e6:.1f} MB")
out_path.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
