"""Occupancy probe of the C4 reservoir configuration (boxes_doppler 1080p,
1024 bins, depth 8, temporal + 1x3 spatial r10): one row band of an n-way
split rendered on one GPU (halo rows arrive empty), printing per frame the
pool rows each sparse grid holds and the frame time.
    python tools/c4_occupancy.py [world] [rank] [frames]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2605_11536_b200 import _ffi as F  # noqa: E402
from paper_2605_11536_b200 import scenes  # noqa: E402
from paper_2605_11536_b200.api import RenderConfig, Renderer  # noqa: E402
from paper_2605_11536_b200.parallel import band_rows, halo_rows  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 16
rank = int(sys.argv[2]) if len(sys.argv) > 2 else world // 2
frames = int(sys.argv[3]) if len(sys.argv) > 3 else 20
cfg = RenderConfig(mode=F.MODE_TRANSIENT, bins=1024, hist_t0=7.0, hist_bin_width=0.01953125, m_init=1,
                   max_depth=8, temporal=True, spatial_passes=1, spatial_neighbors=3, spatial_radius=10,
                   m_cap=20, seed=1)
sd = scenes.bundled("boxes_doppler", 1920, 1080)
y0, y1 = band_rows(1080, world, rank)
halo = halo_rows(cfg.spatial_radius, cfg.spatial_passes)
s = Renderer(0).session(sd, cfg, band=(y0, y1, halo))
s.set_halo_exchange(lambda pass_: None)
items = (y1 - y0) * 1920 * 1024
print(f"band {rank}/{world} rows [{y0},{y1}) items {items}", flush=True)
for f in range(frames):
    t = time.perf_counter()
    st = s.step(stats=True)
    dt = time.perf_counter() - t
    p = s.pool()
    print(f"frame {f} {dt * 1e3:.1f} ms pool {p['rows_used']} cap {p['rows_cap']} "
          f"max frac {max(p['rows_used']) / items:.4f} tjobs {st['temporal']['attempts']} "
          f"sjobs {st['spatial']['attempts']}", flush=True)
