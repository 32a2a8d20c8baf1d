"""Latency floor of k_shift_solve: per-job cycles (refill -> finish), trial
rounds, Newton iterations and re-projection rays, from a TOFR_SOLVE_PROFILE
build of the library (build it here: python tools/solve_profile.py --build).

    TOFR_B200_LIB=paper_2605_11536_b200/_native/variants/libtofr_b200_sprof.so \\
        python tools/solve_profile.py <workload> [world rank]
"""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

if sys.argv[1:2] == ["--build"]:
    from paper_2605_11536_b200 import build as B
    print(B.build_variants({"sprof": ["-DTOFR_SOLVE_PROFILE=1"]}))
    sys.exit(0)

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2605_11536_b200 import _ffi as F  # noqa: E402
from paper_2605_11536_b200 import parallel, scenes  # noqa: E402
from paper_2605_11536_b200.api import Renderer  # noqa: E402

wl = sys.argv[1]
world, rank = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (1, 0)
scene_name, w, h, cfg, desc = bench.WORKLOADS[wl]
sd = scenes.bundled(scene_name, w, h)
r = Renderer(0)
lib = r._lib
cap = 1 << 22
buf = (C.c_uint64 * (cap * 3))()
n = C.c_uint64()


def grab():
    rc = lib.tofr_gpu_debug_solve_profile(buf, cap, C.byref(n))
    if rc != 0:
        raise SystemExit("library built without TOFR_SOLVE_PROFILE (set TOFR_B200_LIB to the sprof variant)")
    a = np.frombuffer(buf, dtype=np.uint64, count=int(n.value) * 3).reshape(-1, 3).copy()
    return a


sess = parallel.BandSession(r, sd, cfg, rank=rank, world=world, group=None, emulate=world > 1)
for _ in range(cfg.m_cap + 5):
    sess.step()
sess.sync()
grab()
sess.step(stats=True)
a = grab()
cyc = a[:, 0].astype(np.float64)
rounds = (a[:, 1] & 0xffffffff).astype(np.int64)
iters = ((a[:, 1] >> 32) & 0xff).astype(np.int64)
rays = (a[:, 1] >> 40).astype(np.int64)
mhz = 1965.0
print(f"{wl} world {world} rank {rank}: {len(a)} solved jobs in one frame")
for q in (50, 90, 99, 99.9, 100):
    v = np.percentile(cyc, q)
    print(f"  p{q:<5} {v:12.0f} cycles = {v / mhz:8.1f} us")
slow = np.argsort(cyc)[-10:]
print("  slowest: us, rounds, iterations, rays")
for i in slow[::-1]:
    print(f"   {cyc[i] / mhz:8.1f} {rounds[i]:6d} {iters[i]:4d} {rays[i]:5d}")
for k in (0, 1, 2, 3, 4, 5):
    m = iters == k
    if m.any():
        print(f"  iter {k}: {m.sum():7d} jobs, mean {cyc[m].mean() / mhz:7.1f} us, max {cyc[m].max() / mhz:7.1f} us, "
              f"mean rounds {rounds[m].mean():5.1f}, mean rays {rays[m].mean():5.1f}")
# timeline: the frame's solve launches, split at gaps of > 15 us between job
# finishes (each launch is followed by its finish and merge kernels); per
# launch the time by which 50 / 90 / 99 / 100% of its jobs had finished
t = np.sort(a[:, 2].astype(np.float64)) / 1e3
cut = np.flatnonzero(np.diff(t) > 15.0) + 1
print("  launch timeline (us from the launch's first finish): jobs, t50, t90, t99, t100")
for seg in np.split(t, cut):
    s = seg - seg[0]
    print(f"   {len(seg):8d} {np.percentile(s, 50):8.1f} {np.percentile(s, 90):8.1f} {np.percentile(s, 99):8.1f} "
          f"{s[-1]:8.1f}")
r_us = cyc / np.maximum(rounds, 1) / mhz
print(f"  us per trial round: p50 {np.percentile(r_us, 50):.2f} p90 {np.percentile(r_us, 90):.2f} "
      f"p99 {np.percentile(r_us, 99):.2f}")
