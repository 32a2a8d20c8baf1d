"""Sparse transient reservoir grids (tofr_store.cuh): a dense header plane
plus a pool of sample rows that only non-empty reservoirs hold.  The storage
layout must not change a single bit of the output: every transient
configuration (temporal, spatial, bin reuse, row bands with halo exchange,
the per-item legacy kernels) renders identically with TOFR_SPARSE=0 (dense
grids), the pool accounting is exact, and a full pool raises an error instead
of corrupting reservoirs."""
from __future__ import annotations

import os

import numpy as np
import pytest

from paper_2605_11536_b200 import _ffi as F
from paper_2605_11536_b200 import scenes
from paper_2605_11536_b200.api import RenderConfig, Renderer, TofrError

pytestmark = pytest.mark.gpu


def _cfg(**kw):
    base = dict(mode=F.MODE_TRANSIENT, bins=48, hist_t0=8.0, hist_bin_width=0.25, m_init=2, frames=3,
                temporal=True, spatial_passes=1, spatial_neighbors=3, spatial_radius=4.0, seed=3)
    base.update(kw)
    return RenderConfig(**base)


class _env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        for k, v in self.kv.items():
            os.environ[k] = v

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


CASES = {
    # mirror box: records with replay lanes (k > 2), pools keep all 24 chunk planes
    "mirror_lanes": ("mirror", _cfg(hist_t0=3.0, hist_bin_width=0.5, max_depth=8)),
    "temporal_spatial": ("cornell", _cfg()),
    "bin_reuse": ("cornell_wide", _cfg(hist_t0=3.0, bin_reuse=True, spatial_passes=2)),
    "animated": ("boxes_doppler", _cfg(hist_t0=7.0, hist_bin_width=0.5, max_depth=8)),
}


def _scene(name):
    if name == "mirror":
        from tests.cases import mirror_box
        return mirror_box(36)
    return scenes.bundled(name, 36)


def _render(scene, cfg, **env):
    with _env(**env):
        out = Renderer(0).render_transient(_scene(scene), cfg)
    return out


@pytest.mark.parametrize("name", sorted(CASES))
def test_sparse_equals_dense(name):
    scene, cfg = CASES[name]
    dense = _render(scene, cfg, TOFR_SPARSE="0")
    sparse = _render(scene, cfg, TOFR_SPARSE="1")
    assert dense.hist.rgb.max() > 0
    assert np.array_equal(sparse.hist.rgb, dense.hist.rgb)
    assert np.array_equal(sparse.image, dense.image)
    for a, b in zip(sparse.stats, dense.stats):
        for stage in ("temporal", "spatial", "bin"):
            da = {k: v for k, v in a[stage].items() if k != "seconds"}
            db = {k: v for k, v in b[stage].items() if k != "seconds"}
            assert da == db, stage


def test_sparse_equals_dense_legacy_kernels():
    scene, cfg = CASES["bin_reuse"]
    dense = _render(scene, cfg, TOFR_SPARSE="0", TOFR_REUSE="legacy", TOFR_TRACE="legacy")
    sparse = _render(scene, cfg, TOFR_SPARSE="1", TOFR_REUSE="legacy", TOFR_TRACE="legacy")
    assert np.array_equal(sparse.hist.rgb, dense.hist.rgb)


def test_pool_rows_count_nonempty_reservoirs():
    """After a frame the current grid holds exactly one pool row per
    reservoir that was ever non-empty in it: at least the non-empty ones."""
    scene, cfg = "cornell", _cfg(spatial_passes=0)
    with _env(TOFR_SPARSE="1"):
        r = Renderer(0)
        s = r.session(_scene(scene), cfg)
        for _ in range(3):
            s.step(stats=False)
        pool = s.pool()
    assert pool["rows_cap"] > 0
    assert max(pool["rows_used"]) > 0
    assert max(pool["rows_used"]) <= pool["rows_cap"]


def test_pool_overflow_raises():
    scene, cfg = CASES["temporal_spatial"]
    with pytest.raises(TofrError, match="pool"):
        _render(scene, cfg, TOFR_SPARSE="1", TOFR_POOL_ROWS="16")


# ---------------------------------------------------------------------------
# row batches: a reuse stage whose shifts exceed the job queue runs over row
# ranges of the band, one queue fill each (capi.cpp wave_batches).  Items are
# independent within a stage, so batching must not change a bit.

def test_gated_row_batches_equal_one_batch():
    from paper_2605_11536_b200.api import GateSpec
    sd = scenes.bundled("cornell", 48)
    cfg = RenderConfig(gate=GateSpec(F.GATE_LENGTH, 10.0, 0.3, 1.0), m_init=2, temporal=True, spatial_passes=2,
                       spatial_neighbors=3, spatial_radius=5, frames=3, seed=5)
    one = Renderer(0).render_gated(sd, cfg)
    with _env(TOFR_WAVE_CAP="1500"):  # 4 jobs x 2304 items -> 7 batches
        many = Renderer(0).render_gated(sd, cfg)
    assert one.image.max() > 0
    assert np.array_equal(many.image, one.image)
    for a, b in zip(many.stats, one.stats):
        for stage in ("temporal", "spatial"):
            assert {k: v for k, v in a[stage].items() if k != "seconds"} == \
                   {k: v for k, v in b[stage].items() if k != "seconds"}


@pytest.mark.parametrize("adaptive", ["1", "0"])
def test_transient_row_batches_equal_one_batch(adaptive):
    """Row batches cut from the device-counted per-row job bounds (adaptive,
    the default for transient grids) or uniformly from the worst case: the
    same bits as one batch, and the queue never overflows."""
    scene, cfg = CASES["temporal_spatial"]
    cfg = RenderConfig(**{**cfg.__dict__, "frames": 5})
    one = _render(scene, cfg, TOFR_SPARSE="1")
    many = _render(scene, cfg, TOFR_SPARSE="1", TOFR_WAVE_CAP="20000", TOFR_ADAPTIVE_BATCHES=adaptive)
    assert np.array_equal(many.hist.rgb, one.hist.rgb)
    for a, b in zip(many.stats, one.stats):
        for stage in ("temporal", "spatial"):
            assert {k: v for k, v in a[stage].items() if k != "seconds"} == \
                   {k: v for k, v in b[stage].items() if k != "seconds"}


def test_queue_smaller_than_a_row_raises():
    """A shift queue that cannot hold one image row's worst case is refused
    up front (row batches need at least one row)."""
    scene, cfg = CASES["temporal_spatial"]
    with pytest.raises(TofrError, match="smaller than one image row"):
        _render(scene, cfg, TOFR_WAVE_CAP="10")


@pytest.mark.parametrize("name", ["temporal_spatial", "bin_reuse", "animated"])
def test_compact_rows_equal_full_rows(name):
    """Compact pool rows (224 B: the k = 2 prefix cache rebuilt from the
    G-buffer, ResStore::compact) against full 304 B rows (TOFR_COMPACT_ROWS=0):
    bit-identical histograms and shift counters."""
    scene, cfg = CASES[name]
    a = _render(scene, cfg, TOFR_SPARSE="1")
    b = _render(scene, cfg, TOFR_SPARSE="1", TOFR_COMPACT_ROWS="0")
    assert b.hist.rgb.max() > 0
    assert np.array_equal(a.hist.rgb, b.hist.rgb)
    for x, y in zip(a.stats, b.stats):
        for stage in ("temporal", "spatial", "bin"):
            assert {k: v for k, v in x[stage].items() if k != "seconds"} == \
                   {k: v for k, v in y[stage].items() if k != "seconds"}


def test_transient_1080p_bench_config_invariants():
    """The bench's transient workload at its full size (t1080b64: cornell
    1920x1080 x 64 bins, temporal reuse; the oracle cannot hold its 133 M
    reservoirs): compact rows against full rows and many row batches against
    the default batches give the same histogram bits and counters, and every
    frame's shift counters are self-consistent (success <= newton_ok <= solves
    <= attempts)."""
    import bench
    scene_name, w, h, cfg, _ = bench.WORKLOADS["t1080b64"]
    cfg = RenderConfig(**{**cfg.__dict__, "frames": 4})
    sd = scenes.bundled(scene_name, w, h)

    def run(**env):
        with _env(**env):
            out = Renderer(0).render_transient(sd, cfg)
        return out.hist.rgb, out.stats

    a, sa = run()
    assert a.shape[:2] == (h, w) and a.max() > 0
    for fs in sa:
        t = fs["temporal"]
        assert t["success"] <= t["newton_ok"] <= t["solves"] <= t["attempts"]
    for env in ({"TOFR_COMPACT_ROWS": "0"}, {"TOFR_WAVE_CAP": "4000000"}):
        b, sb = run(**env)
        assert np.array_equal(a, b), env
        del b
        for x, y in zip(sa, sb):
            for stage in ("temporal", "spatial", "bin"):
                assert {k: v for k, v in x[stage].items() if k != "seconds"} == \
                       {k: v for k, v in y[stage].items() if k != "seconds"}, env
