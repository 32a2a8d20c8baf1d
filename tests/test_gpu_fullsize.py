"""Full-size parity (BASELINE configs at 1080p / 512^2 x 256 bins) and
bit-identity of the wavefront pipeline with the per-reservoir kernels.

* GPU vs the CPU oracle on the bench configurations (full size, or the largest
  size the oracle's reservoirs fit in host RAM): >= 99.9% of pixels and
  histogram bins within 1e-4 relative (north star), histogram counts and
  every shift counter of every frame and stage integer-equal.
* The wavefront reuse engine / path-tree state machine (default) against the
  per-item kernels (TOFR_REUSE=legacy TOFR_TRACE=legacy) in a separate
  process: identical arithmetic, so images and counters must be bit-identical.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from tests.cases import CASES, FULL_CASES
from tests.parity import summary

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
KEYS = ("attempts", "newton_ok", "newton_failed", "occluded", "jac_clamped", "replay_failed", "iterations",
        "solves", "success")


def _render(renderer, table, name):
    build, cfg, kind = table[name]
    sd = build()
    fn = {"gated": renderer.render_gated, "plain": renderer.render_transient_plain,
          "transient": renderer.render_transient}[kind]
    return sd, cfg, kind, fn(sd, cfg)


def _totals(stats):
    tot = {k: 0 for k in KEYS}
    for fs in stats:
        for stage in ("temporal", "spatial", "bin"):
            for k in KEYS:
                tot[k] += fs[stage][k]
    return tot


@pytest.mark.parametrize("name", sorted(FULL_CASES))
def test_full_size_parity(renderer, ref, name):
    sd, cfg, kind, g = _render(renderer, FULL_CASES, name)
    rs = ref.RefScene(sd)
    r = {"gated": ref.render_gated, "plain": ref.render_transient_plain, "transient": ref.render_transient}[kind](
        rs, cfg)
    s = summary(g.image, r.image)
    print(name, s)
    assert r.image.max() > 0
    assert s["within"] >= 0.999, s
    if g.hist is not None:
        hs = summary(g.hist.rgb, r.hist.rgb)
        print(name, "hist", hs)
        assert hs["within"] >= 0.999, hs
        assert np.array_equal(g.hist.count, r.hist.count), "histogram counts differ from the oracle"
    if kind != "plain":
        diffs = counter_diffs(g.stats, r.stats)
        print(name, _totals(g.stats), _totals(r.stats), diffs)
        assert diffs == KNOWN_COUNTER_DIFFS.get(name, {}), diffs


# Counters that differ from the oracle, each with its cause.  Every other counter
# of every frame and stage of every case is integer-equal.
#   full_c4r_doppler_128x72_1024bins, frame 2, spatial, occluded: 3144 vs 3145
#   (one of 163,296 shift attempts).  The device's sin/cos (libdevice, <= 2 ulp) and
#   glibc's differ in the last ulp for some BSDF-sampling angles (tofr_geom.h:367,
#   :381; scene.hpp sample_bsdf), so 14% of the pixels' vertex positions differ by
#   ~1e-16 relative (image bit-exact fraction 0.86, max relative error 2e-14).  One
#   shifted path's occlusion segment grazes a box edge, and the closed/open test
#   (geometry.hpp:86-231, bary +-1e-12) resolves it differently.  Deterministic
#   on both sides (the same counts every run).
#   nlos_cornell_wide_256, frame 3, spatial, occluded: 1695 vs 1696 (one of 657,114
#   attempts).  Same mechanism through the ellipsoidal sampler's transcendentals
#   (atan2 / acos of the conic cut angles, sin / cos of its Gauss-Legendre nodes,
#   ellipsoid.hpp:167-296): 61% of the pixels differ in the last bits (max relative
#   error 1.5e-12), and one shifted segment's grazing occlusion test flips.  The
#   wavefront sampler is bit-identical to the per-lane one (test below), so the
#   difference is libm, not the restructuring.
KNOWN_COUNTER_DIFFS = {
    "full_c4r_doppler_128x72_1024bins": {"f2.spatial.occluded": (3144, 3145)},
    "nlos_cornell_wide_256": {"f3.spatial.occluded": (1695, 1696)},
}


def counter_diffs(gs, rs) -> dict:
    """Every ShiftCounts field of every frame and stage that differs (integer-exact bar)."""
    out = {}
    for f, (fg, fr) in enumerate(zip(gs, rs)):
        for stage in ("temporal", "spatial", "bin"):
            for k in KEYS:
                if fg[stage][k] != fr[stage][k]:
                    out[f"f{f}.{stage}.{k}"] = (fg[stage][k], fr[stage][k])
    return out


_CHILD = r"""
import json, sys, numpy as np
sys.path.insert(0, sys.argv[1])
from tests.cases import CASES, FULL_CASES
from paper_2605_11536_b200.api import Renderer
table = FULL_CASES if sys.argv[2] in FULL_CASES else CASES
build, cfg, kind = table[sys.argv[2]]
r = Renderer(0)
fn = {"gated": r.render_gated, "plain": r.render_transient_plain, "transient": r.render_transient}[kind]
out = fn(build(), cfg)
np.save(sys.argv[3], out.image)
stats = [{st: {k: int(v) for k, v in fs[st].items() if isinstance(v, (int, np.integer))}
          for st in ("temporal", "spatial", "bin")} for fs in out.stats] if out.stats else []
print(json.dumps(stats))
"""


@pytest.mark.parametrize("name", ["full_c3_boxes_doppler_1080p", "full_c1_cornell_256", "mirror_replay",
                                  "transient_full", "transient_bin_reuse", "transient_bin_reuse_animated",
                                  "shrink_r1", "shrink_r05", "shrink_r05_reuse",
                                  "doppler_scene_reuse", "ellipsoidal_init",
                                  "ellipsoidal_collimated", "nlos_cornell_wide_256"])
def test_wavefront_bit_identical_to_per_item_kernels(tmp_path, name):
    outs = []
    for tag, extra in (("wave", {}), ("legacy", {"TOFR_REUSE": "legacy", "TOFR_TRACE": "legacy",
                                                 "TOFR_ELL": "legacy"})):
        env = {**os.environ, **extra}
        f = tmp_path / f"{tag}.npy"
        p = subprocess.run([sys.executable, "-c", _CHILD, str(ROOT), name, str(f)], capture_output=True, text=True,
                           env=env, timeout=900)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append((np.load(f), json.loads(p.stdout.strip().splitlines()[-1])))
    (a, sa), (b, sb) = outs
    assert np.array_equal(a, b), summary(a, b)
    assert sa == sb
