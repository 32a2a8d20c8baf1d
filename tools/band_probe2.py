"""Per-band frame time of every band of an n-way split (emulated on one GPU),
equal bands vs bands balanced on the first frames' image (parallel.balanced_bands).
    python tools/band_probe2.py <workload> <world>"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2605_11536_b200 import parallel, scenes  # noqa: E402
from paper_2605_11536_b200.api import Renderer  # noqa: E402

wl, n = sys.argv[1], int(sys.argv[2])
scene_name, w, h, cfg, desc = bench.WORKLOADS[wl]
sd = scenes.bundled(scene_name, w, h)
r = Renderer(0)


def run(rows_of):
    out = []
    for g in range(n):
        sess = parallel.BandSession(r, sd, cfg, rank=g, world=n, group=None, emulate=True, rows=rows_of[g])
        for _ in range(3):
            sess.step()
        ms = sess.timed_steps(20, [0.0] * 6) / 20
        out.append(ms)
        sess.sess.close()
    return out


full = parallel.BandSession(r, sd, cfg)
for _ in range(3):
    full.step()
t_full = full.timed_steps(20, [0.0] * 6) / 20
full.sess.row_cost(True)
for _ in range(2):
    full.step()
cost = full.sess.row_cost(False)
weights = parallel.row_weights(full.read_image_host(), cost)
full.sess.close()
eq = run([parallel.band_rows(h, n, g) for g in range(n)])
bal_rows = parallel.balanced_bands(weights, n, parallel.halo_rows(cfg.spatial_radius, cfg.spatial_passes))
bal = run(bal_rows)
print(f"{wl} full {t_full:.3f} ms")
print(f"equal bands: max {max(eq):.3f} ms -> {t_full / max(eq):.2f}x", [round(x, 3) for x in eq])
print(f"balanced:    max {max(bal):.3f} ms -> {t_full / max(bal):.2f}x", [round(x, 3) for x in bal], bal_rows)
