"""Per-window device time and SM clock over a long run of one workload: do
frames slow down as the GPU stays loaded (power / thermal clocks)?
    python tools/drift_probe.py <workload> [windows] [frames per window]"""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2605_11536_b200 import parallel, scenes  # noqa: E402
from paper_2605_11536_b200.api import Renderer  # noqa: E402

wl = sys.argv[1]
nw = int(sys.argv[2]) if len(sys.argv) > 2 else 30
k = int(sys.argv[3]) if len(sys.argv) > 3 else 20
scene_name, w, h, cfg, desc = bench.WORKLOADS[wl]
sess = parallel.BandSession(Renderer(0), scenes.bundled(scene_name, w, h), cfg, plain=wl in bench.PLAIN)
for _ in range(25):
    sess.step()
sess.sync()


def clock():
    out = subprocess.run(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw,temperature.gpu",
                          "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
    return out


for i in range(nw):
    ms = sess.timed_steps(k, [0.0] * 6)
    print(f"window {i:3d}: {ms / k:.3f} ms/frame ({k / ms * 1e3:.1f} fps)  clock/power/temp {clock()}", flush=True)
