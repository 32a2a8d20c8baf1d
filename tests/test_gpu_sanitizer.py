"""compute-sanitizer over the device pipeline (race / failure
detection): memcheck (out-of-bounds and misaligned global / shared / local
accesses), racecheck (shared-memory hazards: the staged
frame, the counter reductions) and synccheck (barriers under divergence) on
small renders that reach every kernel family -- gated ReSTIR (wavefront shift
engine, merges), mirror replay (k > 2), transient reservoirs on the sparse
pool with bin reuse and spatial passes, plain deposits (L2 reductions), the
brute-force reference, and the opt-in release/acquire solve -> finish overlap
(TOFR_OVERLAP=1).  Each case runs in a child process under the tool; any
reported error fails the test."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

_CHILD = r"""
import sys
sys.path.insert(0, sys.argv[1])
from paper_2605_11536_b200 import _ffi as F, scenes
from paper_2605_11536_b200.api import GateSpec, RenderConfig, Renderer
case = sys.argv[2]
r = Renderer(0)
g = lambda c, w: GateSpec(F.GATE_LENGTH, c, w, 1.0)
if case == "gated":
    out = r.render_gated(scenes.bundled("boxes_doppler", 24), RenderConfig(gate=g(12.0, 0.3), m_init=2, temporal=True,
                         spatial_passes=1, spatial_neighbors=3, spatial_radius=4, frames=2))
elif case == "mirror":
    sd = scenes.cornell_box(collimated=False, resolution=16, tall_box_material=3, tall_box_kind=F.MAT_MIRROR)
    out = r.render_gated(sd, RenderConfig(gate=g(6.0, 0.4), m_init=2, temporal=True, spatial_passes=1,
                                          spatial_neighbors=3, spatial_radius=3, frames=2, max_depth=8))
elif case == "transient":
    out = r.render_transient(scenes.bundled("cornell", 16), RenderConfig(mode=F.MODE_TRANSIENT, bins=24, hist_t0=8.0,
                             hist_bin_width=0.5, m_init=2, temporal=True, bin_reuse=True, spatial_passes=1,
                             spatial_neighbors=2, spatial_radius=3, frames=2))
elif case == "plain":
    out = r.render_transient_plain(scenes.bundled("boxes_doppler", 16), RenderConfig(mode=F.MODE_TRANSIENT, bins=64,
                                   hist_t0=7.0, hist_bin_width=0.3, m_init=2, max_depth=8, frames=2))
elif case == "ellipsoidal":
    out = r.render_gated(scenes.bundled("cornell_wide", 12), RenderConfig(gate=g(6.0, 0.1), m_init=1,
                         init=F.INIT_ELLIPSOIDAL, temporal=True, spatial_passes=1, spatial_neighbors=2,
                         spatial_radius=2, frames=2))
elif case == "bvh":  # the device BVH build: wide (multi-CTA), per-CTA and per-warp levels, side stream
    r.dump_bvh_device(scenes.bundled("mesh_anim", 16), 7.5)
    out = None
elif case == "reference":
    r.reference_render(scenes.bundled("cornell", 12), 0.0, g(10.0, 0.5), 4, 3, 6)
    out = None
if out is not None:
    assert out.image.max() > 0
    import hashlib
    print("image sha1", hashlib.sha1(out.image.tobytes()).hexdigest())
print("child ok")
"""

CASES = {
    "gated": {},
    "mirror": {},
    "transient": {},
    "plain": {},
    "ellipsoidal": {},
    "reference": {},
    "bvh": {},
    "gated_overlap": {"TOFR_OVERLAP": "1"},
}
TOOLS = ["memcheck", "racecheck", "synccheck"]


@pytest.mark.parametrize("tool", TOOLS)
@pytest.mark.parametrize("name", sorted(CASES))
def test_sanitizer_clean(tmp_path, tool, name):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not Path(cs).exists():
        pytest.skip("compute-sanitizer not found")
    case = name.replace("_overlap", "")
    env = {**os.environ, **CASES[name], "TOFR_PIPELINE": os.environ.get("TOFR_PIPELINE", "1")}
    cmd = [cs, f"--tool={tool}", "--error-exitcode=99", "--print-limit=20"]
    cmd += [sys.executable, "-c", _CHILD, str(ROOT), case]
    p = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=1200)
    log = p.stdout + p.stderr
    (tmp_path / "sanitizer.log").write_text(log)
    if "child ok" not in log and "compute-sanitizer is closed" in log:
        # some GPU pools disable the tool (runs under it left GPUs needing a
        # reset); the recorded clean runs are profiles/r02/pytest_bands_sanitizer.log
        pytest.skip(log.strip().splitlines()[0][:200])
    assert "child ok" in log, log[-3000:]
    assert p.returncode == 0, log[-3000:]
    clean = "ERROR SUMMARY: 0 errors" in log or "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in log
    assert clean, log[-3000:]
