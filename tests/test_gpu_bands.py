"""Row-band sessions on one GPU: n band sessions (one context / stream each,
driven from n threads, halo rows moved by device copies inside the library's
exchange callback) must reproduce the full-frame session bit for bit -- the
device analogue of the reference's worker-count determinism test
(test_pipeline.cpp:80-106).  The multi-process NCCL transport is the same
callback with isend/irecv (parallel.HaloExchanger, covered with gloo in
test_multirank.py)."""
from __future__ import annotations

import threading

import numpy as np
import pytest

from paper_2605_11536_b200 import _ffi as F
from paper_2605_11536_b200 import scenes
from paper_2605_11536_b200.api import GateSpec, RenderConfig, Renderer
from paper_2605_11536_b200.parallel import _wrap, band_rows, halo_rows, motion_rows_for

pytestmark = pytest.mark.gpu


def _moving_camera(res):
    sd = scenes.bundled("cornell_wide", res)
    base = sd.camera.base
    sd.camera.track = [(0.0, scenes.CameraPose((0.0, 0.0, 3.0), base.forward, base.up)),
                       (10.0, scenes.CameraPose((0.0, 0.02, 3.0), base.forward, base.up))]
    return sd


CASES = {
    "cornell_c1": (lambda: scenes.bundled("cornell", 48),
                   RenderConfig(gate=GateSpec(F.GATE_LENGTH, 10.0, 0.3, 1.0), m_init=2, temporal=True,
                                spatial_passes=2, spatial_neighbors=3, spatial_radius=5, frames=3)),
    "doppler_animated": (lambda: scenes.bundled("boxes_doppler", 40),
                         RenderConfig(gate=GateSpec(F.GATE_LENGTH, 12.0, 0.3, 1.0), m_init=1, temporal=True,
                                      spatial_passes=1, spatial_neighbors=4, spatial_radius=6, frames=3)),
    "transient_sparse": (lambda: scenes.bundled("cornell", 40),
                         RenderConfig(mode=F.MODE_TRANSIENT, bins=24, hist_t0=8.0, hist_bin_width=0.5, m_init=2,
                                      temporal=True, spatial_passes=2, spatial_neighbors=3, spatial_radius=4,
                                      frames=3)),
    "moving_camera": (lambda: _moving_camera(40),
                      RenderConfig(gate=GateSpec(F.GATE_LENGTH, 6.0, 0.3, 1.0), m_init=1, temporal=True,
                                   spatial_passes=1, spatial_neighbors=3, spatial_radius=4, frames=3)),
    # temporal reuse only: the band keeps a reprojection halo (parallel.MOTION_HALO_ROWS)
    "moving_camera_temporal_only": (lambda: _moving_camera(48),
                                    RenderConfig(gate=GateSpec(F.GATE_LENGTH, 6.0, 0.3, 1.0), m_init=1,
                                                 temporal=True, frames=3)),
}


def _render_bands(sd, cfg, world, bands=None, transport="peer"):
    """transport "peer": the library's native in-process transport (peer copies
    between the band sessions' streams, no host callback); "callback": device
    copies issued from the exchange callback (the host-staged path)."""
    import torch
    H = sd.camera.height
    halo = halo_rows(cfg.spatial_radius, cfg.spatial_passes, motion_rows_for(sd, cfg))
    bands = bands or [band_rows(H, world, g) for g in range(world)]
    rs = [Renderer(0) for _ in range(world)]
    ss = [rs[g].session(sd, cfg, band=(*bands[g], halo)) for g in range(world)]
    if transport == "peer":
        if halo > 0:
            for g in range(world - 1):
                ss[g].link_halo(ss[g + 1])
            assert all(s.halo_transport() == "peer" for s in ss)
        return _run_threads(ss, cfg, None)
    dev = torch.device("cuda", 0)
    bufs = []
    for s in ss:
        hb = s.halo_buffers()
        bufs.append({k: _wrap(hb[k], hb["bytes_lo" if k.endswith("lo") else "bytes_hi"], dev)
                     for k in ("send_lo", "recv_lo", "send_hi", "recv_hi")})
    bar = threading.Barrier(world)

    def make_cb(g):
        def cb(pass_):
            ss[g].sync_stream()
            bar.wait()  # every band has packed its edge rows
            if g > 0 and bufs[g]["recv_lo"] is not None:
                bufs[g]["recv_lo"].copy_(bufs[g - 1]["send_hi"])
            if g < world - 1 and bufs[g]["recv_hi"] is not None:
                bufs[g]["recv_hi"].copy_(bufs[g + 1]["send_lo"])
            torch.cuda.synchronize()
            bar.wait()  # nobody repacks before every copy landed
        return cb

    for g, s in enumerate(ss):
        s.set_halo_exchange(make_cb(g))
    return _run_threads(ss, cfg, bar)


def _run_threads(ss, cfg, bar):
    world = len(ss)
    errs = []

    def run(g):
        try:
            for _ in range(cfg.frames):
                ss[g].step(stats=False)
            ss[g].sync()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)
            if bar is not None:
                bar.abort()

    ts = [threading.Thread(target=run, args=(g,)) for g in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    return np.concatenate([s.read_image() for s in ss])


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("transport", ["peer", "callback"])
def test_bands_equal_full_frame(name, world, transport):
    build, cfg = CASES[name]
    sd = build()
    full = Renderer(0).session(sd, cfg)
    for _ in range(cfg.frames):
        full.step(stats=False)
    ref = full.read_image()
    got = _render_bands(sd, cfg, world, transport=transport)
    assert ref.max() > 0
    assert np.array_equal(got, ref), f"{int((got != ref).sum())} values differ"


def test_sparse_bands_unequal_heights_and_pools(monkeypatch):
    """Sparse transient grids with a memory-limited pool (TOFR_POOL_FRAC < 1)
    and unequal band heights (edge bands keep one halo, middle bands two):
    the compacted halo layout must agree between sender and receiver."""
    sd = scenes.bundled("cornell", 48)
    cfg = RenderConfig(mode=F.MODE_TRANSIENT, bins=256, hist_t0=8.0, hist_bin_width=0.046875, m_init=2,
                       temporal=True, spatial_passes=2, spatial_neighbors=3, spatial_radius=4, frames=3)
    full = Renderer(0).session(sd, cfg)
    for _ in range(cfg.frames):
        full.step(stats=False)
    ref = full.read_image()
    # every band gets the same fixed pool (the full frame's peak occupancy, so no band
    # overflows): each band's pool share (rows / items stored) differs, and a halo
    # capacity derived from it would differ between a sender and its receiver
    rows = int(max(full.pool()["rows_used"]) * 1.05) + 64
    monkeypatch.setenv("TOFR_POOL_ROWS", str(rows))
    # this small frame is densely filled (m_init 2, two spatial passes): a larger
    # compacted-halo capacity than the default half of the halo rows, still < n
    monkeypatch.setenv("TOFR_HALO_FRAC", "0.9")
    got = _render_bands(sd, cfg, 3, bands=[(0, 12), (12, 36), (36, 48)])
    assert ref.max() > 0
    assert np.array_equal(got, ref), f"{int((got != ref).sum())} values differ"


def test_moving_camera_band_without_halo_is_rejected():
    """A sub-band of a moving camera with temporal reuse and no halo would read
    reprojected reservoirs outside its rows: rejected up front."""
    sd = _moving_camera(32)
    cfg = RenderConfig(gate=GateSpec(F.GATE_LENGTH, 6.0, 0.3, 1.0), m_init=1, temporal=True, frames=2)
    with pytest.raises(Exception, match="reprojection halo"):
        Renderer(0).session(sd, cfg, band=(0, 16, 0))


def test_nccl_transport_initialises():
    """The library's own NCCL communicator (libnccl.so.2 loaded at run time)
    comes up on this device and becomes the band's transport.  A second rank
    cannot share one GPU with NCCL, so the send/recv pairs themselves run only
    on multi-GPU nodes (same group calls as the peer path's copies)."""
    r = Renderer(0)
    uid = r.nccl_unique_id()
    if uid is None:
        pytest.skip("libnccl.so.2 not loadable")
    assert len(uid) == 128
    sd = scenes.bundled("cornell", 32)
    cfg = RenderConfig(gate=GateSpec(F.GATE_LENGTH, 10.0, 0.3, 1.0), m_init=1, temporal=True, spatial_passes=1,
                       spatial_neighbors=3, spatial_radius=4, frames=1)
    band = r.session(sd, cfg, band=(0, 16, 4))
    assert band.halo_transport() == "none"
    with pytest.raises(Exception, match="without a neighbour rank"):
        band.halo_nccl(uid, 0, 1)  # its lower halo would have no sender
    s = r.session(sd, cfg)  # world 1: the whole frame, no halo
    s.halo_nccl(uid, 0, 1)
    assert s.halo_transport() == "nccl"
    s.step(stats=False)
    s.sync()
    assert s.read_image().max() > 0
