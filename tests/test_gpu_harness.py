"""GPU side of the harness / CLI.

* Converged-error parity (north star, parity level 3): the error of the GPU
  ReSTIR render against the GPU brute-force reference equals the CPU
  oracle's error against its own reference (compute_metrics, same seeds).
* Equal-time harness: stepped seeds, averaged repetitions.
* CLI render / reference / compare end to end (files, manifest hashes).
"""
from __future__ import annotations

import json

import numpy as np
import pytest

from paper_2605_11536_b200 import _ffi as F
from paper_2605_11536_b200 import harness as Hn
from paper_2605_11536_b200 import scenes
from paper_2605_11536_b200.api import GateSpec, RenderConfig

pytestmark = pytest.mark.gpu


def test_converged_error_matches_oracle(renderer, ref):
    sd = scenes.bundled("cornell_wide", 48)
    gate = GateSpec(F.GATE_LENGTH, 6.0, 0.3, 1.0)
    cfg = RenderConfig(gate=gate, m_init=2, temporal=True, spatial_passes=1, spatial_neighbors=3, spatial_radius=6,
                       frames=4, accumulate=True, seed=3)
    gm, _ = renderer.reference_render(sd, 0.0, gate, 512, 17, 6)
    rs = ref.RefScene(sd)
    rm, _ = ref.reference_render(rs, 0.0, gate, 512, 17, 6)
    g = renderer.render_gated(sd, cfg).image
    r = ref.render_gated(rs, cfg).image
    mg, mr = Hn.compute_metrics(g, gm), Hn.compute_metrics(r, rm)
    print("gpu", mg, "cpu", mr)
    assert mr.mape > 0
    assert abs(mg.mape - mr.mape) <= 1e-6 * mr.mape
    assert abs(mg.relmse - mr.relmse) <= 1e-6 * mr.relmse


def test_transient_converged_error_matches_oracle(renderer, ref):
    """Parity level 3 for the transient output (pipeline.hpp:396-528, :588-607):
    the relMSE / MAPE of the ReSTIR histogram (temporal reuse, bins as pixels)
    against a high-sample plain-deposit histogram (render_transient_plain, an
    unbiased per-bin estimate) equal the CPU oracle's own errors against its
    own plain reference, to 1e-6 relative."""
    sd = scenes.bundled("cornell", 32)
    base = dict(mode=F.MODE_TRANSIENT, bins=16, hist_t0=8.0, hist_bin_width=0.75, max_depth=6)
    restir = RenderConfig(**base, m_init=2, temporal=True, m_cap=20, frames=4, seed=3)
    plain = RenderConfig(**base, m_init=64, frames=2, seed=17)
    rs = ref.RefScene(sd)
    g_ref, r_ref = renderer.render_transient_plain(sd, plain), ref.render_transient_plain(rs, plain)
    g, r = renderer.render_transient(sd, restir), ref.render_transient(rs, restir)
    mg = Hn.compute_metrics(g.hist.rgb, g_ref.hist.rgb)
    mr = Hn.compute_metrics(r.hist.rgb, r_ref.hist.rgb)
    print("gpu", mg, "cpu", mr)
    assert r_ref.hist.rgb.max() > 0 and mr.relmse > 0
    assert abs(mg.mape - mr.mape) <= 1e-6 * mr.mape
    assert abs(mg.relmse - mr.relmse) <= 1e-6 * mr.relmse
    # and the images (sum over bins) the same way
    mgi, mri = Hn.compute_metrics(g.image, g_ref.image), Hn.compute_metrics(r.image, r_ref.image)
    assert abs(mgi.relmse - mri.relmse) <= 1e-6 * mri.relmse


def test_render_equal_time_reps(renderer):
    sd = scenes.bundled("cornell", 24)
    cfg = RenderConfig(gate=GateSpec(F.GATE_LENGTH, 10.0, 0.3, 1.0), m_init=2, spatial_passes=1,
                       spatial_neighbors=3, spatial_radius=4, seed=5)
    res = Hn.render_equal_time(renderer, sd, cfg, 0.0, min_reps=3, max_reps=3)
    assert res.repetitions == 3 and res.spatial["attempts"] > 0
    acc = np.zeros_like(res.image)
    for rep in range(3):
        c = RenderConfig(**{**cfg.__dict__, "seed": cfg.seed + rep * 0x9E3779B9})
        acc += renderer.render_gated(sd, c).image
    assert np.array_equal(res.image, acc * (1.0 / 3))  # image += r.image; image *= 1/reps


def test_cli_render_reference_compare(tmp_path):
    from paper_2605_11536_b200 import cli
    scn = tmp_path / "cornell.scn"
    scn.write_text(scenes.to_scn(scenes.bundled("cornell", 32)))
    out = str(tmp_path / "r")
    assert cli.main(["render", "--scene", str(scn), "--tau", "10", "--dtau", "0.3", "--candidates", "2",
                     "--spatial", "1", "--neighbors", "3", "--radius", "5", "--temporal", "--frames", "2",
                     "--out", out]) == 0
    man = json.loads((tmp_path / "r_manifest.json").read_text())
    assert man["config"]["gate"]["center"] == 10.0 and len(man["outputs"]) == 3
    for o in man["outputs"]:
        assert o["fnv64"] == Hn.hash_file(o["path"])
    assert (tmp_path / "r_stats.txt").read_text().startswith("frame=0 stage=init")
    assert cli.main(["reference", "--scene", str(scn), "--tau", "10", "--dtau", "0.3", "--spp", "16",
                     "--out", str(tmp_path / "ref")]) == 0
    assert cli.main(["compare", "--est", out + ".pfm", "--ref", str(tmp_path / "ref.pfm")]) == 0
    assert cli.main(["render", "--scene", str(scn), "--mode", "transient", "--tau", "10", "--dtau", "1.0",
                     "--bins", "4", "--candidates", "1", "--out", str(tmp_path / "t")]) == 0
    assert (tmp_path / "t_hist.csv").read_text().startswith("pixel_x,pixel_y,bin,r,g,b,count\n")
