"""oracle/ref.py -- TEST INFRASTRUCTURE ONLY.

ctypes wrapper of oracle/_ref/libtofr_ref.so: the unmodified CPU reference
renderer (/root/reference/proj/include/tofr, built by oracle/Makefile) behind
the same scene/config structs as the GPU library.  Only tests/,
__graft_entry__.smoke() and bench.py (cpu_baseline, --impl reference) use it,
as the checker / baseline; the product path never imports it.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2605_11536_b200 import _ffi as F
from paper_2605_11536_b200.api import GateSpec, RenderConfig, RenderOutput, TransientHistogram, stats_to_dicts
from paper_2605_11536_b200.scenes import SceneDef

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libtofr_ref.so"
REF_INCLUDE = Path("/root/reference/proj/include")

_lib = None


def available() -> bool:
    return LIB.exists()


def build_if_possible() -> bool:
    """Build oracle/_ref when the reference sources are present (this
    container); the GPU box only uses the prebuilt library."""
    import subprocess
    if REF_INCLUDE.exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "all", "shim"], check=True)
    return LIB.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            raise RuntimeError(f"{LIB} missing (build with `make -C oracle`)")
        L = C.CDLL(str(LIB))
        P = C.POINTER
        vp = C.c_void_p
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_set_threads.restype = None
        L.ref_get_threads.restype = C.c_int
        L.ref_scene_load.argtypes = [C.c_char_p, P(vp), C.c_char_p, C.c_size_t]
        L.ref_scene_parse.argtypes = [C.c_char_p, C.c_char_p, P(vp), C.c_char_p, C.c_size_t]
        L.ref_scene_create.argtypes = [P(F.SceneDesc), P(vp), C.c_char_p, C.c_size_t]
        L.ref_scene_destroy.argtypes = [vp]
        L.ref_scene_destroy.restype = None
        L.ref_scene_set_resolution.argtypes = [vp, C.c_int, C.c_int]
        for n in ("ref_render_gated", "ref_render_transient", "ref_render_transient_plain"):
            getattr(L, n).argtypes = [vp, P(F.RenderConfigC), P(F.Output), C.c_char_p, C.c_size_t]
        L.ref_reference.argtypes = [vp, C.c_double, C.c_double, C.c_double, C.c_int, C.c_uint64, C.c_int,
                                    P(C.c_double), P(C.c_double), C.c_char_p, C.c_size_t]
        L.ref_dump_bvh.argtypes = [vp, C.c_double, C.c_int, P(C.c_double), P(C.c_int), P(C.c_int), C.c_int,
                                   P(C.c_int), P(C.c_int), P(C.c_double), C.c_char_p, C.c_size_t]
        L.ref_probe_rays.argtypes = [vp, C.c_double, P(C.c_double), C.c_int, C.c_int, P(C.c_double), P(C.c_int),
                                     C.c_char_p, C.c_size_t]
        L.ref_rng_stream.argtypes = [C.c_uint64] * 5 + [C.c_int, P(C.c_double), P(C.c_uint64)]
        L.ref_rng_stream.restype = None
        L.ref_bin_of.argtypes = [C.c_int, C.c_double, C.c_double, P(C.c_double), C.c_int, P(C.c_int)]
        L.ref_neighbor_offsets.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_double,
                                           P(C.c_int)]
        L.ref_neighbor_offsets.restype = None
        L.ref_initial_sampling.argtypes = [vp, P(F.RenderConfigC), C.c_int] + [P(C.c_double)] * 4 + \
            [P(C.c_int), P(C.c_int), C.c_char_p, C.c_size_t]
        L.ref_compute_metrics.argtypes = [P(C.c_double), P(C.c_double), C.c_int, C.c_int, P(C.c_double),
                                          P(C.c_double)]
        L.ref_compute_metrics.restype = None
        _lib = L
    return _lib


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _iptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


class RefScene:
    def __init__(self, scene):
        L = lib()
        self.h = C.c_void_p()
        err = C.create_string_buffer(512)
        if isinstance(scene, SceneDef):
            desc, keep = scene.to_desc()
            rc = L.ref_scene_create(C.byref(desc), C.byref(self.h), err, 512)
            del keep
            self.width, self.height = scene.camera.width, scene.camera.height
        else:
            rc = L.ref_scene_load(str(scene).encode(), C.byref(self.h), err, 512)
            self.width = self.height = None
        if rc != 0:
            raise RuntimeError(err.value.decode())

    def set_resolution(self, w, h):
        lib().ref_scene_set_resolution(self.h, w, h)
        self.width, self.height = w, h

    def __del__(self):
        try:
            lib().ref_scene_destroy(self.h)
        except Exception:
            pass


def _check(rc, err):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {err.value.decode()}")


def set_threads(n: int) -> None:
    lib().ref_set_threads(n)


def threads() -> int:
    return lib().ref_get_threads()


def _render(fn, scene: RefScene, cfg: RenderConfig, transient: bool) -> RenderOutput:
    W, H = scene.width, scene.height
    B = cfg.bins if transient else 1
    img = np.zeros((H, W, 3))
    out = F.Output()
    out.image = _dptr(img)
    rgb = cnt = None
    if transient:
        rgb = np.zeros((H, W, B, 3))
        cnt = np.zeros((H, W, B), dtype=np.int64)
        out.hist_rgb = _dptr(rgb)
        out.hist_count = cnt.ctypes.data_as(C.POINTER(C.c_int64))
    n = max(0, cfg.frames)
    stats = (F.FrameStats * max(1, n))()
    out.stats = stats
    out.stats_capacity = n
    err = C.create_string_buffer(512)
    c = cfg.to_c()
    _check(getattr(lib(), fn)(scene.h, C.byref(c), C.byref(out), err, 512), err)
    hist = TransientHistogram(W, H, B, cfg.hist_t0, cfg.hist_bin_width, rgb, cnt) if transient else None
    return RenderOutput(img, hist, stats_to_dicts(stats, n))


def render_gated(scene: RefScene, cfg: RenderConfig) -> RenderOutput:
    return _render("ref_render_gated", scene, cfg, False)


def render_transient(scene: RefScene, cfg: RenderConfig) -> RenderOutput:
    return _render("ref_render_transient", scene, cfg, True)


def render_transient_plain(scene: RefScene, cfg: RenderConfig) -> RenderOutput:
    return _render("ref_render_transient_plain", scene, cfg, True)


def reference_render(scene: RefScene, frame: float, gate: GateSpec, spp: int, seed: int, max_depth: int = 6):
    mean = np.zeros((scene.height, scene.width, 3))
    se = np.zeros_like(mean)
    err = C.create_string_buffer(512)
    _check(lib().ref_reference(scene.h, frame, gate.center, gate.width, spp, seed, max_depth, _dptr(mean),
                               _dptr(se), err, 512), err)
    return mean, se


def dump_bvh(scene: RefScene, frame: float = 0.0, cap: int = 1 << 14):
    nodes = np.zeros((cap, 11))
    parent = np.zeros(cap, dtype=np.int32)
    order = np.zeros(cap, dtype=np.int32)
    nn, nt = C.c_int(), C.c_int()
    diag = C.c_double()
    err = C.create_string_buffer(512)
    _check(lib().ref_dump_bvh(scene.h, frame, cap, _dptr(nodes), _iptr(parent), C.byref(nn), cap, _iptr(order),
                              C.byref(nt), C.byref(diag), err, 512), err)
    return nodes[:nn.value].copy(), parent[:nn.value].copy(), order[:nt.value].copy(), diag.value


def probe_rays(scene: RefScene, frame: float, rays: np.ndarray, mode: int):
    rays = np.ascontiguousarray(rays, dtype=np.float64)
    n = rays.shape[0]
    t = np.zeros(n)
    tri = np.zeros(n, dtype=np.int32)
    err = C.create_string_buffer(512)
    _check(lib().ref_probe_rays(scene.h, frame, _dptr(rays), n, mode, _dptr(t), _iptr(tri), err, 512), err)
    return t, tri


def rng_stream(seed, frame, pixel, sample, lane, count):
    out = np.zeros(count)
    u = np.zeros(count, dtype=np.uint64)
    lib().ref_rng_stream(seed, frame, pixel, sample, lane, count, _dptr(out),
                         u.ctypes.data_as(C.POINTER(C.c_uint64)))
    return out, u


def bin_of(bins, t0, bw, lens):
    lens = np.ascontiguousarray(lens, dtype=np.float64)
    out = np.zeros(lens.shape[0], dtype=np.int32)
    lib().ref_bin_of(bins, t0, bw, _dptr(lens), lens.shape[0], _iptr(out))
    return out


def neighbor_offsets(pix, pass_, seed, frame_idx, count, radius):
    out = np.zeros(2 * count, dtype=np.int32)
    lib().ref_neighbor_offsets(pix, pass_, seed, frame_idx, count, radius, _iptr(out))
    return out.reshape(count, 2)


def initial_sampling(scene: RefScene, cfg: RenderConfig, frame_idx: int):
    n = scene.width * scene.height
    W, M, ph, ln = (np.zeros(n) for _ in range(4))
    has = np.zeros(n, dtype=np.int32)
    k = np.zeros(n, dtype=np.int32)
    err = C.create_string_buffer(512)
    c = cfg.to_c()
    _check(lib().ref_initial_sampling(scene.h, C.byref(c), frame_idx, _dptr(W), _dptr(M), _dptr(ph), _dptr(ln),
                                      _iptr(has), _iptr(k), err, 512), err)
    return {"W": W, "M": M, "phat": ph, "len": ln, "has": has, "k": k}


def compute_metrics(est: np.ndarray, refimg: np.ndarray):
    """The reference's compute_metrics (pipeline.hpp:588-607): (mape, relmse)."""
    est = np.ascontiguousarray(est, dtype=np.float64)
    refimg = np.ascontiguousarray(refimg, dtype=np.float64)
    h, w = est.shape[:2]
    mape, relmse = C.c_double(), C.c_double()
    lib().ref_compute_metrics(_dptr(est), _dptr(refimg), w, h, C.byref(mape), C.byref(relmse))
    return mape.value, relmse.value


def _tool(*args, stdin: str | None = None) -> str:
    """oracle/_ref/ref_tool: the reference's stream-based writers in their own
    process (libstdc++ streams inside the ctypes-loaded library are not safe
    next to this interpreter's runtime)."""
    import subprocess
    exe = LIB.parent / "ref_tool"
    if not exe.exists():
        raise RuntimeError(f"{exe} missing (build with `make -C oracle`)")
    r = subprocess.run([str(exe), *map(str, args)], input=stdin, capture_output=True, text=True, check=True)
    return r.stdout


def write_image(img: np.ndarray, pfm_path: str, txt_path: str) -> None:
    """write_pfm + write_text_matrix (image.hpp:41-82) of the reference."""
    import tempfile
    img = np.ascontiguousarray(img, dtype=np.float64)
    with tempfile.NamedTemporaryFile(suffix=".f64") as f:
        f.write(img.tobytes())
        f.flush()
        _tool("write_image", f.name, img.shape[1], img.shape[0], pfm_path, txt_path)


def hash_file(path: str) -> int:
    """hash_file (image.hpp:99-106) of the reference."""
    return int(_tool("hash", path).strip())


def stats_lines(stats: list) -> str:
    """stats_lines (pipeline.hpp:612-633) of the reference for the given
    per-frame counters and timings."""
    keys = ("attempts", "newton_ok", "newton_failed", "occluded", "jac_clamped", "replay_failed", "iterations",
            "solves", "success")
    rows = []
    for fs in stats:
        row = [str(fs["frame"]), repr(float(fs["t_init"])), repr(float(fs["t_shade"]))]
        for st in ("temporal", "spatial", "bin"):
            row += [str(int(fs[st][k])) for k in keys] + [repr(float(fs[st]["seconds"]))]
        rows.append(" ".join(row))
    return _tool("stats_lines", stdin="\n".join(rows) + "\n")

