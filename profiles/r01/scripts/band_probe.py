"""Strong-scaling probe on one GPU: frames/s of one emulated row band of an
n-way split (halo rows arrive empty, no transfer) against the full frame.
    python tools/band_probe.py <workload> [worlds...]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2605_11536_b200 import parallel, scenes  # noqa: E402
from paper_2605_11536_b200.api import Renderer  # noqa: E402

wl = sys.argv[1]
worlds = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
scene_name, w, h, cfg, desc = bench.WORKLOADS[wl]
sd = scenes.bundled(scene_name, w, h)
r = Renderer(0)
base = None
for n in worlds:
    rank = n // 2
    sess = parallel.BandSession(r, sd, cfg, rank=rank if n > 1 else 0, world=n, group=None, emulate=n > 1)
    for _ in range(3):
        sess.step()
    st = [0.0] * 6
    ms = sess.timed_steps(30, st)
    fps = 30 / (ms * 1e-3)
    base = base or fps
    print(f"{wl} world {n} rank {rank}: {fps:.1f} frames/s per band ({fps / base:.2f}x the full frame), "
          f"stages {[round(x / 30, 3) for x in st]}", flush=True)
    sess.sess.close()
