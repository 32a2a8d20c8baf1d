"""Interactive sessions (the frame loop one call at a time, reservoirs resident
on the device) against the one-shot drivers that mirror the reference
(render_gated / render_transient / render_transient_plain,
pipeline.hpp:323-571): same frames, same outputs, bit for bit."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2605_11536_b200 import _ffi as F
from paper_2605_11536_b200 import scenes
from paper_2605_11536_b200.api import GateSpec, RenderConfig, Renderer

pytestmark = pytest.mark.gpu


def _transient_cfg(**kw):
    base = dict(mode=F.MODE_TRANSIENT, bins=32, hist_t0=8.0, hist_bin_width=0.375, m_init=2, frames=3)
    base.update(kw)
    return RenderConfig(**base)


def test_plain_session_equals_render_transient_plain():
    sd = scenes.bundled("cornell", 40)
    cfg = _transient_cfg()
    r = Renderer(0)
    ref = r.render_transient_plain(sd, cfg)
    s = r.session(sd, cfg, plain=True)
    for _ in range(cfg.frames):
        s.step(stats=False)
    rgb, cnt = s.read_histogram()
    assert np.array_equal(cnt, ref.hist.count)
    assert np.array_equal(rgb, ref.hist.rgb)
    img = s.read_image()
    assert np.allclose(img, ref.image, rtol=1e-12, atol=0)


def test_transient_session_equals_render_transient():
    sd = scenes.bundled("cornell_wide", 32)
    cfg = _transient_cfg(hist_t0=3.0, hist_bin_width=0.25, temporal=True, frames=3)
    r = Renderer(0)
    ref = r.render_transient(sd, cfg)
    s = r.session(sd, cfg)
    for _ in range(cfg.frames):
        s.step(stats=False)
    rgb, _ = s.read_histogram()
    assert ref.hist.rgb.max() > 0
    assert np.array_equal(rgb, ref.hist.rgb)


def test_async_read_equals_sync_read():
    import torch
    sd = scenes.bundled("boxes_doppler", 48)
    cfg = RenderConfig(gate=GateSpec(F.GATE_LENGTH, 12.0, 0.3, 1.0), m_init=1, temporal=True, spatial_passes=1,
                       spatial_neighbors=3, spatial_radius=5, frames=4)
    s = Renderer(0).session(sd, cfg)
    bufs = [torch.empty((48, 48, 3), dtype=torch.float64, pin_memory=True).numpy() for _ in range(2)]
    for f in range(cfg.frames):
        s.step(stats=False)
        s.read_image_async(bufs[f & 1], f & 1)
    s.wait_read((cfg.frames - 1) & 1)
    assert np.array_equal(bufs[(cfg.frames - 1) & 1], s.read_image())
    assert bufs[(cfg.frames - 1) & 1].max() > 0


def test_gated_session_equals_render_gated():
    sd = scenes.bundled("cornell", 48)
    cfg = RenderConfig(gate=GateSpec(F.GATE_LENGTH, 10.0, 0.3, 1.0), m_init=2, temporal=True, spatial_passes=2,
                       spatial_neighbors=3, spatial_radius=5, frames=3)
    r = Renderer(0)
    ref = r.render_gated(sd, cfg)
    s = r.session(sd, cfg)
    stats = [s.step(stats=True) for _ in range(cfg.frames)]
    assert np.array_equal(s.read_image(), ref.image)
    for a, b in zip(stats, ref.stats):
        assert a["spatial"]["attempts"] == b["spatial"]["attempts"]
        assert a["temporal"]["success"] == b["temporal"]["success"]


@pytest.mark.parametrize("mode", ["gated", "transient", "doppler"])
@pytest.mark.parametrize("variant", ["radius0", "neighbors0"])
def test_spatial_radius_zero_is_a_no_op(mode, variant):
    """test_pipeline.cpp:132-145: a spatial pass of radius 0 only meets the
    pixel itself (skipped), and one with no neighbours merges nothing
    (pipeline.hpp:246), so it leaves every reservoir as it was -- including
    the velocity chunks of a Doppler reservoir."""
    sd = scenes.bundled("boxes_doppler" if mode == "doppler" else "cornell", 32)
    base = dict(m_init=2, temporal=True, frames=3, seed=5)
    if mode == "gated":
        base["gate"] = GateSpec(F.GATE_LENGTH, 10.0, 0.4, 1.0)
    elif mode == "doppler":
        base.update(gate=GateSpec(F.GATE_VELOCITY, -0.09, 0.06, 1.0), frame0=2)
    else:
        base.update(mode=F.MODE_TRANSIENT, bins=24, hist_t0=8.0, hist_bin_width=0.5)
    r = Renderer(0)
    render = {"gated": r.render_gated, "transient": r.render_transient, "doppler": r.render_doppler}[mode]
    off = render(sd, RenderConfig(**base, spatial_passes=0))
    sp = dict(spatial_neighbors=3, spatial_radius=0.0) if variant == "radius0" else \
        dict(spatial_neighbors=0, spatial_radius=5.0)
    zero = render(sd, RenderConfig(**base, spatial_passes=2, **sp))
    assert off.image.max() > 0
    assert np.array_equal(zero.image, off.image)


@pytest.mark.parametrize("name", ["gated", "gated_depth2", "gated_temporal_only", "transient",
                                  "transient_temporal_only"])
def test_pipelined_frames_equal_serial(name, monkeypatch):
    """Pipelined sessions (the default) run the camera and initial sampling of
    frame f on a side stream while frame f-1 (gated: also frame f-2, a fourth
    grid and a third frame slot; TOFR_PIPE_DEPTH=2: two frames) finishes: the
    frames must equal those of one stream (TOFR_PIPELINE=0).  Seven frames take
    the gated ring of grids and slots around twice."""
    sd = scenes.bundled("boxes_doppler", 40)
    if name == "gated_depth2":
        monkeypatch.setenv("TOFR_PIPE_DEPTH", "2")
    if name.startswith("gated"):
        sp = dict(spatial_passes=0) if name == "gated_temporal_only" else \
            dict(spatial_passes=1, spatial_neighbors=3, spatial_radius=5)
        cfg = RenderConfig(gate=GateSpec(F.GATE_LENGTH, 12.0, 0.3, 1.0), m_init=1, temporal=True, frames=7, **sp)
    elif name == "transient":
        cfg = _transient_cfg(hist_t0=7.0, hist_bin_width=0.5, temporal=True, spatial_passes=1,
                             spatial_neighbors=3, spatial_radius=4, frames=4)
    else:  # sparse grids with three-frame buffers (a fourth grid, a third slot)
        cfg = _transient_cfg(hist_t0=7.0, hist_bin_width=0.5, temporal=True, frames=7)
    render = Renderer(0).render_gated if name.startswith("gated") else Renderer(0).render_transient
    got = render(sd, cfg)
    monkeypatch.setenv("TOFR_PIPELINE", "0")
    ref = render(sd, cfg)
    assert ref.image.max() > 0
    assert np.array_equal(got.image, ref.image)


def test_plain_deposits_are_deterministic():
    """Plain deposits are L2 reductions; a pixel's trees run on one lane, so
    every bin receives its deposits in emission order: two renders are bit
    identical (and the sums are the reference's sequential rgb += v)."""
    sd = scenes.bundled("boxes_doppler", 40)
    cfg = _transient_cfg(bins=200, hist_t0=7.0, hist_bin_width=0.1, m_init=4, max_depth=8, frames=2)
    r = Renderer(0)
    a = r.render_transient_plain(sd, cfg)
    b = r.render_transient_plain(sd, cfg)
    assert a.hist.count.sum() > 0
    assert np.array_equal(a.hist.rgb, b.hist.rgb)
    assert np.array_equal(a.hist.count, b.hist.count)
    assert np.array_equal(a.image, b.image)


@pytest.mark.parametrize("name", ["cornell", "mesh"])
def test_static_scene_snapshot_cache_is_bit_identical(name, monkeypatch):
    """Static scenes upload their frame snapshot once per slot (the host SAH
    build of a 10^5-triangle mesh would run every frame otherwise): the frames
    equal those of per-frame rebuilds (TOFR_STATIC_FRAMES=0)."""
    sd = scenes.mesh_scene(32) if name == "mesh" else scenes.bundled("cornell", 40)
    cfg = RenderConfig(gate=GateSpec(F.GATE_LENGTH, 6.0 if name == "mesh" else 10.0, 0.3, 1.0), m_init=1,
                       temporal=True, spatial_passes=1, spatial_neighbors=3, spatial_radius=4, frames=4)
    got = Renderer(0).render_gated(sd, cfg)
    monkeypatch.setenv("TOFR_STATIC_FRAMES", "0")
    ref = Renderer(0).render_gated(sd, cfg)
    assert ref.image.max() > 0
    assert np.array_equal(got.image, ref.image)


@pytest.mark.parametrize("kind", ["gated", "transient", "plain", "ellipsoidal", "reference"])
def test_walk_cutoff_is_bit_identical(kind, monkeypatch):
    """Path trees end once their length passes the sink's reach (lengths only
    grow along a walk, so no later candidate could be wanted; the next tree has
    its own RNG stream): every output equals the full walks' (TOFR_WALK_CUTOFF=0)."""
    r = Renderer(0)
    sd = scenes.bundled("boxes_doppler" if kind in ("gated", "plain") else "cornell_wide", 40)
    if kind == "gated":
        cfg = RenderConfig(gate=GateSpec(F.GATE_LENGTH, 12.0, 0.2, 1.0), m_init=2, temporal=True, spatial_passes=1,
                           spatial_neighbors=3, spatial_radius=5, frames=3)
        run = lambda: (r.render_gated(sd, cfg).image,)  # noqa: E731
    elif kind == "transient":
        cfg = _transient_cfg(hist_t0=3.0, hist_bin_width=0.25, temporal=True, spatial_passes=1,
                             spatial_neighbors=2, spatial_radius=3, frames=3)
        run = lambda: (r.render_transient(sd, cfg).hist.rgb,)  # noqa: E731
    elif kind == "plain":
        cfg = _transient_cfg(bins=100, hist_t0=7.0, hist_bin_width=0.05, m_init=4, max_depth=8, frames=2)
        run = lambda: (lambda o: (o.hist.rgb, o.hist.count))(r.render_transient_plain(sd, cfg))  # noqa: E731
    elif kind == "ellipsoidal":
        cfg = RenderConfig(gate=GateSpec(F.GATE_LENGTH, 6.0, 0.1, 1.0), m_init=2, init=F.INIT_ELLIPSOIDAL,
                           temporal=True, spatial_passes=1, spatial_neighbors=3, spatial_radius=4, frames=2)
        run = lambda: (r.render_gated(sd, cfg).image,)  # noqa: E731
    else:
        gate = GateSpec(F.GATE_LENGTH, 6.0, 0.3, 1.0)
        run = lambda: r.reference_render(sd, 0.0, gate, 16, 3, 6)  # noqa: E731
    got = run()
    monkeypatch.setenv("TOFR_WALK_CUTOFF", "0")
    full = run()
    assert full[0].max() > 0
    for a, b in zip(got, full):
        assert np.array_equal(a, b)
