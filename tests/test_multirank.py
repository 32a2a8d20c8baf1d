"""Row-band sharding (parallel.py) on CPU with the gloo backend, world sizes 2
and 3: band partition, halo sizing against the reference's neighbour offsets
(pipeline.hpp:232-239), the HaloExchanger P2P pattern, and a banded spatial
stencil that must equal the full-frame stencil bit for bit -- the multi-rank
analogue of the reference's worker-count determinism test
(test_pipeline.cpp:80-106)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import restate as RS
from paper_2605_11536_b200.parallel import HaloExchanger, balanced_bands, band_rows, halo_rows, row_weights


def test_band_rows_partition():
    for H in (1, 7, 135, 1080):
        for n in (1, 2, 3, 4, 8):
            if n > H:
                continue
            rows = [band_rows(H, n, g) for g in range(n)]
            assert rows[0][0] == 0 and rows[-1][1] == H
            for a, b in zip(rows, rows[1:]):
                assert a[1] == b[0]
            sizes = [b - a for a, b in rows]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_balanced_bands_partition(world):
    """Cost-balanced bands (bench.py at N > 1): contiguous, covering, at least
    the halo thick, and no band heavier than an equal-row split's heaviest."""
    rng = np.random.default_rng(world)
    H, halo = 1080, 10
    img = np.zeros((H, 64, 3))
    img[300:700, :40] = rng.random((400, 40, 3))  # a lit block in the middle rows
    w = row_weights(img)
    bands = balanced_bands(w, world, halo)
    assert bands[0][0] == 0 and bands[-1][1] == H and len(bands) == world
    for a, b in zip(bands, bands[1:]):
        assert a[1] == b[0]
    assert min(b - a for a, b in bands) >= (halo if world > 1 else 1)
    cost = lambda bs: max(w[a:b].sum() for a, b in bs)  # noqa: E731
    equal = [band_rows(H, world, g) for g in range(world)]
    assert cost(bands) <= cost(equal) + 1e-9
    if world == 8:
        assert cost(bands) < 0.75 * cost(equal)


@pytest.mark.parametrize("radius", [0.5, 1.0, 3.0, 5.5, 10.0])
def test_halo_covers_reference_neighbour_offsets(radius):
    """Every offset neighbor_offset can produce satisfies |dy| <= halo_rows."""
    h = halo_rows(radius)
    worst = 0
    for pix in range(0, 4000, 7):
        for pass_ in range(2):
            rk = RS.spatial_rot_key(pix, pass_, 1, 3)
            for count in (1, 3, 5, 8):
                for j in range(count):
                    dx, dy = RS.neighbor_offset(j, count, radius, rk)
                    worst = max(worst, abs(dy))
    assert worst <= h
    assert halo_rows(radius, passes=0) == 0
    # a moving camera with temporal reuse keeps a reprojection margin even without spatial passes
    assert halo_rows(radius, passes=0, motion_rows=16) == 16
    assert halo_rows(radius, passes=1, motion_rows=16) == h


def test_motion_rows_only_for_animated_cameras_with_temporal_reuse():
    from paper_2605_11536_b200 import scenes
    from paper_2605_11536_b200.api import RenderConfig
    from paper_2605_11536_b200.parallel import MOTION_HALO_ROWS, motion_rows_for
    sd = scenes.bundled("cornell_wide", 16)
    assert motion_rows_for(sd, RenderConfig(temporal=True)) == 0
    base = sd.camera.base
    sd.camera.track = [(0.0, scenes.CameraPose((0.0, 0.0, 3.0), base.forward, base.up)),
                       (10.0, scenes.CameraPose((0.0, 0.02, 3.0), base.forward, base.up))]
    assert motion_rows_for(sd, RenderConfig(temporal=True)) == MOTION_HALO_ROWS
    assert motion_rows_for(sd, RenderConfig(temporal=False)) == 0


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _stencil_offsets(W, H, radius, count, pass_=0, seed=1, frame=2):
    """Per-pixel neighbour lists from the reference formula (global pixel keys)."""
    offs = {}
    for y in range(H):
        for x in range(W):
            pix = y * W + x
            rk = RS.spatial_rot_key(pix, pass_, seed, frame)
            offs[pix] = [RS.neighbor_offset(j, count, radius, rk) for j in range(count)]
    return offs


def _stencil(grid, y0, y1, r0, W, H, offs):
    """out[y] for y in [y0, y1): sequential per-pixel 'merge' of the valid
    neighbours (order matters, like gris_merge's RNG stream)."""
    out = np.zeros((y1 - y0, W), dtype=np.float64)
    for y in range(y0, y1):
        for x in range(W):
            acc = grid[y - r0, x]
            for dx, dy in offs[y * W + x]:
                nx, ny = x + dx, y + dy
                if (nx, ny) == (x, y) or not (0 <= nx < W and 0 <= ny < H):
                    continue
                acc = acc * 0.75 + grid[ny - r0, nx] * 0.5
            out[y - y0, x] = acc
    return out


def _worker(rank, world, port, W, H, radius, count, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        full = rng.random((H, W))  # the pass-input grid every rank would compute
        y0, y1 = band_rows(H, world, rank)
        halo = halo_rows(radius)
        r0, r1 = max(0, y0 - halo), min(H, y1 + halo)
        local = np.full((r1 - r0, W), np.nan)
        local[y0 - r0:y1 - r0] = full[y0:y1]  # owned rows only; halo rows unknown
        lo, hi = y0 - r0, r1 - y1
        to_t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).view(torch.uint8).reshape(-1)
        send_lo = to_t(local[lo:lo + lo]) if lo else None
        send_hi = to_t(local[y1 - r0 - hi:y1 - r0]) if hi else None
        recv_lo = torch.zeros(lo * W * 8, dtype=torch.uint8) if lo else None
        recv_hi = torch.zeros(hi * W * 8, dtype=torch.uint8) if hi else None
        ex = HaloExchanger(rank, world, dist.group.WORLD, send_lo, recv_lo, send_hi, recv_hi)
        ex(0)
        if lo:
            local[:lo] = recv_lo.view(torch.float64).reshape(lo, W).numpy()
        if hi:
            local[y1 - r0:] = recv_hi.view(torch.float64).reshape(hi, W).numpy()
        assert not np.isnan(local).any()
        offs = _stencil_offsets(W, H, radius, count)
        band = _stencil(local, y0, y1, r0, W, H, offs)
        ref = _stencil(full, y0, y1, 0, W, H, offs)
        q.put((rank, bool(np.array_equal(band, ref)), ex.calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_banded_stencil_equals_full_frame(world):
    W, H, radius, count = 24, 33, 5.0, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, W, H, radius, count, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
