"""Iterated band rebalancing from measured band times, emulated on one GPU:
every band of an n-way split is rendered alone; the split is refined with
parallel.rebalance_bands from the measured times.
    python tools/band_probe3.py <workload> <world> [iterations]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2605_11536_b200 import parallel, scenes  # noqa: E402
from paper_2605_11536_b200.api import Renderer  # noqa: E402

wl, n = sys.argv[1], int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
scene_name, w, h, cfg, desc = bench.WORKLOADS[wl]
sd = scenes.bundled(scene_name, w, h)
r = Renderer(0)
halo = parallel.halo_rows(cfg.spatial_radius, cfg.spatial_passes)


def band_times(bands):
    out = []
    for g in range(n):
        sess = parallel.BandSession(r, sd, cfg, rank=g, world=n, group=None, emulate=True, bands=bands)
        for _ in range(3):
            sess.step()
        out.append(sess.timed_steps(10, [0.0] * 6) / 10)
        sess.sess.close()
    return out


full = parallel.BandSession(r, sd, cfg)
for _ in range(3):
    full.step()
t_full = full.timed_steps(20, [0.0] * 6) / 20
full.sess.close()
bands = [parallel.band_rows(h, n, g) for g in range(n)]
for it in range(iters + 1):
    t = band_times(bands)
    print(f"{wl} n={n} iter {it}: max {max(t):.3f} ms -> {t_full / max(t):.2f}x  times {[round(x, 3) for x in t]} "
          f"bands {bands}", flush=True)
    bands = parallel.rebalance_bands(bands, t, halo)
