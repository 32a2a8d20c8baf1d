"""Host-side timing of the e2e loop pieces for one workload:
    python tools/e2e_probe.py <workload> [frames]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_11536_b200 import parallel, scenes  # noqa: E402
from paper_2605_11536_b200.api import Renderer  # noqa: E402

wl = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 20
scene_name, w, h, cfg, desc = bench.WORKLOADS[wl]
sess = parallel.BandSession(Renderer(0), scenes.bundled(scene_name, w, h), cfg, plain=wl in bench.PLAIN)
for _ in range(3):
    sess.step()
sess.sync()
t = {"step": 0.0, "read_async": 0.0, "wait": 0.0}
bufs = [torch.empty((h, w, 3), dtype=torch.float64, pin_memory=True).numpy() for _ in range(2)]
t0 = time.perf_counter()
for f in range(k):
    a = time.perf_counter()
    sess.sess.step(stats=False)
    b = time.perf_counter()
    if f >= 2:
        sess.sess.wait_read(f & 1)
    c = time.perf_counter()
    sess.sess.read_image_async(bufs[f & 1], f & 1)
    d = time.perf_counter()
    t["step"] += b - a
    t["wait"] += c - b
    t["read_async"] += d - c
sess.sync()
tot = time.perf_counter() - t0
print(wl, f"e2e {k / tot:.1f} fps", {n: round(v / k * 1e3, 3) for n, v in t.items()}, "ms/frame")
t0 = time.perf_counter()
hs = 0.0
for f in range(k):
    a = time.perf_counter()
    sess.sess.step(stats=False)
    hs += time.perf_counter() - a
sess.sync()
tot = time.perf_counter() - t0
print(wl, f"steps only {k / tot:.1f} fps, host step {hs / k * 1e3:.3f} ms/frame")
# pure host enqueue cost: the GPU is idle when each step starts
hs = []
for f in range(k):
    sess.sync()
    a = time.perf_counter()
    sess.sess.step(stats=False)
    hs.append(time.perf_counter() - a)
sess.sync()
print(wl, f"host enqueue per step (idle GPU): median {np.median(hs) * 1e3:.3f} ms, max {max(hs) * 1e3:.3f} ms")
