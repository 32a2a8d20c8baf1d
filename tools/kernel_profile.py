#!/usr/bin/env python
"""profiles/kernel_profile.json from ncu --set full captures of ONE steady-state
frame's launches of a kernel, plus the bench line printed by the same run:

    ncu --set full --metrics <FP64_METRICS> -k regex:'^<kernel>$' -s <warm*L> -c <L> -o rep \\
        python bench.py --workload <wl> --steps 1 --warmup <warm> --no-cpu-baseline > line.json
    python tools/kernel_profile.py --wl <wl> --kernel <kernel> --bench line.json rep.ncu-rep

With --steps 1 the bench's timed frame is the captured frame (frame index
<warm>), so its device work counters (units_per_frame) are the units of the
captured launches.  Stored per "<wl>:<kernel>": DRAM bytes (read + write), FP64
flops (thread-level DADD + DMUL + 2 DFMA) and FP64 instructions, each per unit
of work (bench.KERNEL_BYTES unit) and per launch.  bench.py scales the per-unit
figures by its own units per launch (roofline.traffic, roofline_fp64).
"""
import argparse
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "inst": 1, "Kinst": 1e3,
        "Minst": 1e6, "Ginst": 1e9}
FP64 = {"smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": 1,
        "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": 1,
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": 2}
FP64_METRICS = ",".join(FP64)


def val(d, u, k):
    v = d.get(k, "0").replace(",", "")
    try:
        return float(v) * UNIT.get(u.get(k, ""), 1)
    except ValueError:
        return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "kernel_profile.json"))
    ap.add_argument("--wl", required=True)
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--bench", required=True, help="bench.py JSON line of the same ncu run (--steps 1)")
    ap.add_argument("--tag", default="")
    ap.add_argument("report")
    a = ap.parse_args()
    import bench
    line = json.loads([x for x in Path(a.bench).read_text().splitlines() if x.startswith("{")][-1])
    unit, _ = bench.KERNEL_BYTES[a.kernel]
    units = float(line["units_per_frame"][unit])
    txt = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    hdr, units_row, rows = r[0], r[1], r[2:]
    u = dict(zip(hdr, units_row))
    dram = flops = inst = dur = 0.0
    for row in rows:
        d = dict(zip(hdr, row))
        dram += val(d, u, "dram__bytes_read.sum") + val(d, u, "dram__bytes_write.sum")
        for k, w in FP64.items():
            n = val(d, u, k)
            flops += w * n
            inst += n
        dur += val(d, u, "gpu__time_duration.sum")
    n = max(1, len(rows))
    data = json.loads(Path(a.out).read_text()) if Path(a.out).exists() else {}
    data[f"{a.wl}:{a.kernel}"] = {
        "launches_captured": len(rows), "unit": unit, "units_captured": units,
        "dram_bytes_per_launch": dram / n, "dram_bytes_per_unit": dram / max(1.0, units),
        "fp64_flops_per_launch": flops / n, "fp64_flops_per_unit": flops / max(1.0, units),
        "fp64_inst_per_unit": inst / max(1.0, units),
        "ncu_ms_per_launch": dur / n / 1e6 if u.get("gpu__time_duration.sum") == "nsecond" else None,
        "source": f"ncu --set full of frame {line['warmup']} (the first timed frame, after {line['warmup']} "
                  f"warm-up frames), {len(rows)} launches{(' ' + a.tag) if a.tag else ''}",
    }
    Path(a.out).write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
    print(a.wl, a.kernel, f"{dram / 1e6:.1f} MB DRAM, {flops / 1e9:.3f} GFLOP FP64 over {len(rows)} launches, "
          f"{units:.0f} {unit}s")


if __name__ == "__main__":
    main()
