"""CPU: the host runtime of libtofr_b200.so (no GPU calls).

* The C-ABI library loads and exports every symbol include/tofr_gpu.h declares.
* The SAH BVH of every frame is the reference's, node for node (bit-equal
  boxes/areas, same children/leaf ranges, same tri_order) -- traversal order,
  tie-breaking and ellipsoid-descent probabilities depend on it.
* The bundled scenes built programmatically equal the reference parser's.
* The threaded (stackless) traversal, run through its host build, returns the
  reference's closest hit (same triangle, bit-equal t) and any-hit answers on
  10^4 random rays (test_geometry.cpp:112-132 pattern).
* .scn parse errors map to TOFR_ERR_PARSE with the reference's line:col.
"""
from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

from paper_2605_11536_b200 import _ffi as F
from paper_2605_11536_b200 import scenes
from paper_2605_11536_b200.api import Scene, TofrError

ROOT = Path(__file__).resolve().parents[1]
REF_SCENES = Path("/root/reference/proj/scenes")


def test_library_exports_every_declared_symbol():
    lib = F.load_library()
    header = (ROOT / "include" / "tofr_gpu.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|void|const char\*|uint64_t)\s+(tofr_\w+)\s*\(", header, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(F.EXPORTED_SYMBOLS), declared ^ set(F.EXPORTED_SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.tofr_gpu_version()


def test_config_defaults_match_reference():
    lib = F.load_library()
    c = F.RenderConfigC()
    lib.tofr_render_config_default(c)
    from paper_2605_11536_b200.api import RenderConfig
    p = RenderConfig().to_c()
    for name, _ in F.RenderConfigC._fields_:
        assert getattr(c, name) == getattr(p, name), name


SCENE_VARIANTS = {
    "cornell": lambda: scenes.bundled("cornell"),
    "cornell_wide": lambda: scenes.bundled("cornell_wide"),
    "boxes_doppler": lambda: scenes.bundled("boxes_doppler"),
    "cornell_box_mirror": lambda: scenes.cornell_box(False, 16, 3, 0.3, F.MAT_MIRROR),
    "flat_wall": lambda: scenes.flat_wall(8),
}


@pytest.mark.parametrize("name", sorted(SCENE_VARIANTS))
def test_bvh_matches_reference(ref, name):
    sd = SCENE_VARIANTS[name]()
    g = Scene.create(sd)
    r = ref.RefScene(sd)
    for frame in (0.0, 1.0, 13.25, 39.0, 41.0):
        a = g.dump_bvh(frame)
        b = ref.dump_bvh(r, frame)
        for x, y in zip(a[:3], b[:3]):
            assert np.array_equal(x, y)
        assert a[3] == b[3]


@pytest.mark.skipif(not REF_SCENES.exists(), reason="reference scenes not present")
@pytest.mark.parametrize("name", ["cornell", "cornell_wide", "boxes_doppler"])
def test_bundled_builders_equal_parsed_scn(ref, name):
    path = REF_SCENES / f"{name}.scn"
    parsed_ref = ref.RefScene(path)
    parsed_ours = Scene.create(path)
    built = Scene.create(scenes.bundled(name))
    for frame in (0.0, 5.0, 20.0):
        b = ref.dump_bvh(parsed_ref, frame)
        for s in (parsed_ours, built):
            a = s.dump_bvh(frame)
            for x, y in zip(a[:3], b[:3]):
                assert np.array_equal(x, y)


def _rays(n, rng, segments=False, box=3.0):
    o = rng.uniform(-box, box, size=(n, 3))
    if segments:
        return np.concatenate([o, rng.uniform(-box, box, size=(n, 3)), np.zeros((n, 2))], axis=1)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.concatenate([o, d, np.full((n, 1), 1e-6), np.full((n, 1), np.inf)], axis=1)


@pytest.mark.parametrize("name,frame", [("cornell_wide", 0.0), ("boxes_doppler", 7.5), ("cornell_box_mirror", 0.0)])
def test_host_traversal_matches_reference(ref, name, frame):
    sd = SCENE_VARIANTS[name]()
    g = Scene.create(sd)
    r = ref.RefScene(sd)
    rng = np.random.default_rng(7)
    rays = _rays(10000, rng)
    # include axis-aligned directions (inf reciprocals, NaN slab products)
    rays[:6, 3:6] = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]])
    t, tri = g.probe_rays_host(frame, rays, 0)
    rt, rtri = ref.probe_rays(r, frame, rays, 0)
    assert np.array_equal(tri, rtri)
    assert np.array_equal(t, rt)
    assert (tri >= 0).mean() > 0.05
    seg = _rays(10000, rng, segments=True)
    _, occ = g.probe_rays_host(frame, seg, 1)
    _, rocc = ref.probe_rays(r, frame, seg, 1)
    assert np.array_equal(occ, rocc)


def test_parse_errors_carry_line_and_column(ref):
    bad = "camera {\n  position 0 0 x\n}\n"
    with pytest.raises(TofrError) as e:
        Scene.parse(bad)
    assert e.value.code == F.TOFR_ERR_PARSE
    assert "2:" in str(e.value) and "expected a number" in str(e.value)
    with pytest.raises(TofrError) as e:
        Scene.parse("light { regime wide }\n")
    assert "no objects" in str(e.value)
    with pytest.raises(TofrError) as e:
        Scene.parse("bogus { }\n")
    assert "unknown section" in str(e.value)


def test_degenerate_and_empty_meshes_raise():
    sd = scenes.flat_wall(4)
    sd.objects[0].tris.append(((0, 0, 0), (1, 0, 0), (2, 0, 0), 0))  # zero area
    with pytest.raises(TofrError) as e:
        Scene.create(sd).info()
    assert "degenerate" in str(e.value)
    sd = scenes.flat_wall(4)
    sd.objects[0].tris = []
    with pytest.raises(TofrError) as e:
        Scene.create(sd).info()
    assert "empty mesh" in str(e.value)


def test_mesh_bvh_matches_reference(ref, tmp_path):
    """A 102,410-triangle scene (displaced torus, 64,875 nodes: far beyond the
    shared-memory staging limit): the host SAH build is node-for-node the
    reference's (geometry.hpp:234-317), and the OBJ path (scene_io.hpp:102-132)
    gives the same tree as the inline triangles.  (The oracle parses the
    inline triangles: its OBJ reader is not used in a process that also holds
    the device library.)"""
    sd = scenes.mesh_scene(32)
    inline = Scene.create(sd)
    obj = Scene.create(scenes.mesh_scene_file(tmp_path, 32, 32))
    assert inline.info()["n_tris"] == 102410
    a = inline.dump_bvh(0.0)
    b = obj.dump_bvh(0.0)
    r = ref.dump_bvh(ref.RefScene(sd), 0.0, 2 * 102410 + 2)
    assert len(a[0]) > 60000
    for x, y, z in zip(a[:3], b[:3], r[:3]):
        assert np.array_equal(x, y)
        assert np.array_equal(x, z)
    assert a[3] == b[3] == r[3]


def test_animated_mesh_bvh_matches_reference(ref):
    """The moving 102,410-triangle torus (a new tree every frame): the host
    build equals the reference's at several frames of its track."""
    sd = scenes.mesh_scene(32, animated=True)
    g, r = Scene.create(sd), ref.RefScene(sd)
    for frame in (0.0, 7.5, 20.0):
        a = g.dump_bvh(frame)
        b = ref.dump_bvh(r, frame, 2 * 102410 + 2)
        for x, y in zip(a[:3], b[:3]):
            assert np.array_equal(x, y)
        assert a[3] == b[3]
