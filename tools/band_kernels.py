"""Per-kernel times (CUDA events per launch) of one emulated band vs the full frame.
    python tools/band_kernels.py <workload> <world> <rank>"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2605_11536_b200 import _ffi as F  # noqa: E402
from paper_2605_11536_b200 import parallel, scenes  # noqa: E402
from paper_2605_11536_b200.api import Renderer  # noqa: E402

wl, n, g = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
scene_name, w, h, cfg, desc = bench.WORKLOADS[wl]
sd = scenes.bundled(scene_name, w, h)
r = Renderer(0)
for world, rank in ((1, 0), (n, g)):
    sess = parallel.BandSession(r, sd, cfg, rank=rank, world=world, group=None, emulate=world > 1)
    for _ in range(3):
        sess.step()
    sess.sync()
    F.kernel_times(reset=True)
    F.kernel_timing(True)
    st = [0.0] * 6
    ms = sess.timed_steps(20, st)
    F.kernel_timing(False)
    kt = F.kernel_times(reset=True)
    print(f"world {world} rank {rank} rows {sess.y0}-{sess.y1}: {ms / 20:.3f} ms/frame, stages",
          [round(x / 20, 3) for x in st])
    for k, (t, c) in sorted(kt.items(), key=lambda kv: -kv[1][0])[:8]:
        print(f"   {k:24s} {t / 20:8.3f} ms/frame  {c // 20:4d} launches/frame  {t / c * 1e3:8.1f} us/launch")
    st1 = sess.step(stats=True)
    print("   shift attempts", st1["temporal"]["attempts"], st1["spatial"]["attempts"])
    sess.sess.close()
