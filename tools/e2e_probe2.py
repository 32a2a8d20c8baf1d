"""Where the e2e frames/s go, on the same animation frames (fresh session
each, W warm-up frames, then K timed): device-timed steps, host-timed steps
without read-back, and the e2e loop with read-back.
    python tools/e2e_probe2.py <workload> [K] [W]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2605_11536_b200 import parallel, scenes  # noqa: E402
from paper_2605_11536_b200.api import Renderer  # noqa: E402

wl = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = int(sys.argv[3]) if len(sys.argv) > 3 else 25
scene_name, W, H, cfg, desc = bench.WORKLOADS[wl]
r = Renderer(0)
sd = scenes.bundled(scene_name, W, H)


def fresh():
    s = parallel.BandSession(r, sd, cfg, plain=wl in bench.PLAIN)
    for _ in range(w):
        s.step()
    s.sync()
    return s


s = fresh()
ms = s.timed_steps(k, [0.0] * 6)
print(f"{wl} device-timed steps: {k / ms * 1e3:.1f} fps")
s.sess.close()
s = fresh()
t0 = time.perf_counter()
for _ in range(k):
    s.sess.step(stats=False)
s.sync()
print(f"{wl} host-timed steps, no read-back (fill + drain included): {k / (time.perf_counter() - t0):.1f} fps")
s.sess.close()
s = fresh()
print(f"{wl} e2e loop with read-back: {k / s.run_e2e(k, warm=0):.1f} fps")
s.sess.close()
