"""Python mirror of the reference render API (pipeline.hpp / harness.hpp) over
the C ABI of libtofr_b200.so.

    render_gated(scene, cfg)            -> RenderOutput   (pipeline.hpp:323)
    render_transient(scene, cfg)        -> RenderOutput   (pipeline.hpp:396)
    render_transient_plain(scene, cfg)  -> RenderOutput   (pipeline.hpp:531)
    render_doppler(scene, cfg)          -> RenderOutput   (pipeline.hpp:574, velocity gate)
    reference_render(scene, frame, gate, spp, seed, max_depth) -> (mean, se)

`scene` is a SceneDef (scenes.py), a path to a .scn file, or a Scene handle.
Images are float64 arrays [H, W, 3]; histograms [H, W, B, 3] in the
reference's (y*W + x)*B + b order.  Errors raise TofrError with the library
message (the reference throws std::runtime_error / ParseError).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields

import numpy as np

from . import _ffi as F
from .scenes import SceneDef


class TofrError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[tofr error {code}] {msg}")
        self.code = code


@dataclass
class GateSpec:  # transport.hpp:44-59
    kind: int = F.GATE_LENGTH
    center: float = 0.0
    width: float = 1.0
    f0: float = 1.0


@dataclass
class RenderConfig:  # pipeline.hpp:18-61 (same names and defaults)
    mode: int = F.MODE_GATED
    gate: GateSpec = field(default_factory=GateSpec)
    gate_step: float = 0.0
    bins: int = 1
    hist_t0: float = 0.0
    hist_bin_width: float = 0.0
    m_init: int = 8
    init: int = F.INIT_DIRECT
    shrink_k: float = 10.0
    shrink_r: float = 1.0
    spatial_passes: int = 0
    spatial_neighbors: int = 5
    spatial_radius: float = 10.0
    temporal: bool = False
    bin_reuse: bool = False
    m_cap: float = 20.0
    gauge: int = F.GAUGE_AVG
    newton: bool = True
    seed: int = 1
    frames: int = 1
    frame0: float = 0.0
    max_depth: int = 6
    use_rr: bool = True
    accumulate: bool = False
    normalize_gate: bool = False

    def to_c(self) -> F.RenderConfigC:
        c = F.RenderConfigC()
        c.mode = self.mode
        c.gate_kind = self.gate.kind
        c.gate_center = self.gate.center
        c.gate_width = self.gate.width
        c.gate_f0 = self.gate.f0
        c.gate_step = self.gate_step
        c.bins = self.bins
        c.hist_t0 = self.hist_t0
        c.hist_bin_width = self.hist_bin_width
        c.m_init = self.m_init
        c.init_mode = self.init
        c.shrink_k = self.shrink_k
        c.shrink_r = self.shrink_r
        c.spatial_passes = self.spatial_passes
        c.spatial_neighbors = self.spatial_neighbors
        c.spatial_radius = self.spatial_radius
        c.temporal = int(bool(self.temporal))
        c.bin_reuse = int(bool(self.bin_reuse))
        c.m_cap = self.m_cap
        c.gauge = self.gauge
        c.newton = int(bool(self.newton))
        c.seed = self.seed
        c.frames = self.frames
        c.frame0 = self.frame0
        c.max_depth = self.max_depth
        c.use_rr = int(bool(self.use_rr))
        c.accumulate = int(bool(self.accumulate))
        c.normalize_gate = int(bool(self.normalize_gate))
        return c


@dataclass
class TransientHistogram:  # transport.hpp:100-127
    w: int
    h: int
    bins: int
    t0: float
    bin_width: float
    rgb: np.ndarray  # [H, W, B, 3]
    count: np.ndarray  # [H, W, B] int64


@dataclass
class RenderOutput:  # pipeline.hpp:306-310
    image: np.ndarray
    hist: TransientHistogram | None
    stats: list


def stats_to_dicts(arr, n: int) -> list:
    out = []
    for i in range(n):
        s = arr[i]
        out.append({
            "frame": int(s.frame),
            "t_init": float(s.t_init),
            "t_shade": float(s.t_shade),
            "temporal": dict(s.temporal.shift.as_dict(), seconds=float(s.temporal.seconds)),
            "spatial": dict(s.spatial.shift.as_dict(), seconds=float(s.spatial.seconds)),
            "bin": dict(s.binwise.shift.as_dict(), seconds=float(s.binwise.seconds)),
        })
    return out


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Scene:
    """Handle to a host-side scene of libtofr_b200 (tofr_scene)."""

    def __init__(self, lib, handle):
        self._lib = lib
        self.handle = handle

    @classmethod
    def create(cls, scene, lib=None) -> "Scene":
        lib = lib or F.load_library()
        if isinstance(scene, Scene):
            return scene
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        if isinstance(scene, SceneDef):
            desc, keep = scene.to_desc()
            rc = lib.tofr_scene_create(C.byref(desc), C.byref(h), err, 512)
            del keep
        else:
            rc = lib.tofr_scene_load(str(scene).encode(), C.byref(h), err, 512)
        if rc != F.TOFR_OK:
            raise TofrError(rc, err.value.decode())
        return cls(lib, h)

    @classmethod
    def parse(cls, text: str, base_dir: str = ".", lib=None) -> "Scene":
        lib = lib or F.load_library()
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = lib.tofr_scene_parse(text.encode(), base_dir.encode(), C.byref(h), err, 512)
        if rc != F.TOFR_OK:
            raise TofrError(rc, err.value.decode())
        return cls(lib, h)

    def set_resolution(self, w: int, h: int) -> None:
        rc = self._lib.tofr_scene_set_resolution(self.handle, w, h)
        if rc != F.TOFR_OK:
            raise TofrError(rc, "bad resolution")

    def info(self) -> dict:
        w, h, nt, nn = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        diag = C.c_double()
        err = C.create_string_buffer(512)
        rc = self._lib.tofr_scene_info(self.handle, C.byref(w), C.byref(h), C.byref(nt), C.byref(nn),
                                       C.byref(diag), err, 512)
        if rc != F.TOFR_OK:
            raise TofrError(rc, err.value.decode())
        return {"width": w.value, "height": h.value, "n_tris": nt.value, "n_nodes": nn.value, "diag": diag.value}

    def dump_bvh(self, frame: float = 0.0):
        info = self.info()
        cap = max(16384, 2 * info["n_tris"] + 2)  # a binary tree over n leaves' triangles: < 2n nodes
        nodes = np.zeros((cap, 11))
        parent = np.zeros(cap, dtype=np.int32)
        order = np.zeros(cap, dtype=np.int32)
        nn, nt = C.c_int32(), C.c_int32()
        diag = C.c_double()
        err = C.create_string_buffer(512)
        rc = self._lib.tofr_scene_dump_bvh(self.handle, frame, nodes.shape[0], _dptr(nodes),
                                           parent.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(nn),
                                           order.shape[0], order.ctypes.data_as(C.POINTER(C.c_int32)),
                                           C.byref(nt), C.byref(diag), err, 512)
        if rc != F.TOFR_OK:
            raise TofrError(rc, err.value.decode())
        return nodes[:nn.value].copy(), parent[:nn.value].copy(), order[:nt.value].copy(), diag.value

    def probe_rays_host(self, frame: float, rays: np.ndarray, mode: int):
        rays = np.ascontiguousarray(rays, dtype=np.float64)
        n = rays.shape[0]
        t = np.zeros(n)
        tri = np.zeros(n, dtype=np.int32)
        err = C.create_string_buffer(512)
        rc = self._lib.tofr_scene_probe_rays_host(self.handle, frame, _dptr(rays), n, mode, _dptr(t),
                                                  tri.ctypes.data_as(C.POINTER(C.c_int32)), err, 512)
        if rc != F.TOFR_OK:
            raise TofrError(rc, err.value.decode())
        return t, tri

    def __del__(self):
        try:
            if self.handle:
                self._lib.tofr_scene_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


class Renderer:
    """A tofr_gpu context on one CUDA device."""

    def __init__(self, device: int = 0, lib=None):
        self._lib = lib or F.load_library()
        self.handle = C.c_void_p()
        dev = (C.c_int * 1)(device)
        rc = self._lib.tofr_gpu_create(dev, 1, C.byref(self.handle))
        if rc != F.TOFR_OK:
            raise TofrError(rc, f"tofr_gpu_create failed on device {device}")

    def _check(self, rc: int) -> None:
        if rc != F.TOFR_OK:
            raise TofrError(rc, self._lib.tofr_gpu_last_error(self.handle).decode())

    def _scene(self, scene, width=None, height=None) -> Scene:
        s = Scene.create(scene, self._lib)
        return s

    def _render(self, fn_name: str, scene, cfg: RenderConfig, transient: bool) -> RenderOutput:
        s = self._scene(scene)
        info = s.info()
        W, H = info["width"], info["height"]
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
        nfr = max(0, cfg.frames)
        stats = (F.FrameStats * max(1, nfr))()
        out.stats = stats
        out.stats_capacity = nfr
        c = cfg.to_c()
        self._check(getattr(self._lib, fn_name)(self.handle, s.handle, C.byref(c), C.byref(out)))
        hist = None
        if transient:
            hist = TransientHistogram(W, H, B, cfg.hist_t0, cfg.hist_bin_width, rgb, cnt)
        return RenderOutput(img, hist, stats_to_dicts(stats, nfr))

    def render_gated(self, scene, cfg: RenderConfig) -> RenderOutput:
        return self._render("tofr_gpu_render_gated", scene, cfg, False)

    def render_doppler(self, scene, cfg: RenderConfig) -> RenderOutput:
        """render_gated with the gate read as a Doppler (path-velocity) gate:
        centre/width in Hz, carrier cfg.gate.f0 (pipeline.hpp:573-578)."""
        return self._render("tofr_gpu_render_doppler", scene, cfg, False)

    def render_transient(self, scene, cfg: RenderConfig) -> RenderOutput:
        return self._render("tofr_gpu_render_transient", scene, cfg, True)

    def render_transient_plain(self, scene, cfg: RenderConfig) -> RenderOutput:
        return self._render("tofr_gpu_render_transient_plain", scene, cfg, True)

    def reference_render(self, scene, frame: float, gate: GateSpec, spp: int, seed: int, max_depth: int = 6):
        s = self._scene(scene)
        info = s.info()
        mean = np.zeros((info["height"], info["width"], 3))
        se = np.zeros_like(mean)
        self._check(self._lib.tofr_gpu_reference(self.handle, s.handle, frame, gate.center, gate.width, spp, seed,
                                                 max_depth, _dptr(mean), _dptr(se)))
        return mean, se

    def dump_bvh_device(self, scene, frame: float = 0.0):
        """Scene.dump_bvh of the tree built on the device (bvh_build.cu)."""
        s = self._scene(scene)
        cap = max(16384, 2 * s.info()["n_tris"] + 2)
        nodes = np.zeros((cap, 11))
        parent = np.zeros(cap, dtype=np.int32)
        order = np.zeros(cap, dtype=np.int32)
        nn, nt = C.c_int32(), C.c_int32()
        diag = C.c_double()
        self._check(self._lib.tofr_gpu_dump_bvh_device(self.handle, s.handle, frame, cap, _dptr(nodes),
                                                       parent.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(nn),
                                                       cap, order.ctypes.data_as(C.POINTER(C.c_int32)),
                                                       C.byref(nt), C.byref(diag)))
        return nodes[:nn.value].copy(), parent[:nn.value].copy(), order[:nt.value].copy(), diag.value

    def nccl_unique_id(self) -> bytes | None:
        """A fresh 128-byte ncclUniqueId (None when libnccl.so.2 cannot be loaded)."""
        buf = C.create_string_buffer(128)
        rc = self._lib.tofr_gpu_nccl_unique_id(buf)
        if rc == F.TOFR_ERR_UNSUPPORTED:
            return None
        self._check(rc)
        return buf.raw

    def fp64_peak_gflops(self) -> float:
        """Measured FP64 DFMA throughput of this device (GFLOP/s): the FP64 roofline peak."""
        v = C.c_double(0)
        self._check(self._lib.tofr_gpu_fp64_peak(self.handle, C.byref(v)))
        return float(v.value)

    def probe_rays(self, scene, frame: float, rays: np.ndarray, mode: int):
        s = self._scene(scene)
        rays = np.ascontiguousarray(rays, dtype=np.float64)
        n = rays.shape[0]
        t = np.zeros(n)
        tri = np.zeros(n, dtype=np.int32)
        self._check(self._lib.tofr_gpu_probe_rays(self.handle, s.handle, frame, _dptr(rays), n, mode, _dptr(t),
                                                  tri.ctypes.data_as(C.POINTER(C.c_int32))))
        return t, tri

    def session(self, scene, cfg: RenderConfig, band: tuple | None = None, plain: bool = False) -> "Session":
        return Session(self, self._scene(scene), cfg, band, plain)

    def __del__(self):
        try:
            if self.handle:
                self._lib.tofr_gpu_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


class Session:
    """Interactive frame stepping (the body of the render_gated frame loop).

    With `band=(y0, y1, halo)` the session renders image rows [y0, y1) only
    and keeps `halo` rows on each side for spatial reuse (row-band sharding,
    see parallel.py); the default is the whole frame."""

    def __init__(self, r: Renderer, scene: Scene, cfg: RenderConfig, band: tuple | None = None,
                 plain: bool = False):
        self._r = r
        self._scene = scene
        self.cfg = cfg
        self.plain = plain
        self.transient = plain or cfg.mode == F.MODE_TRANSIENT
        self.handle = C.c_void_p()
        c = cfg.to_c()
        y0, y1, halo = band if band is not None else (0, -1, 0)
        if plain:
            r._check(r._lib.tofr_gpu_session_create_plain(r.handle, scene.handle, C.byref(c), y0, y1,
                                                          C.byref(self.handle)))
        else:
            r._check(r._lib.tofr_gpu_session_create_band(r.handle, scene.handle, C.byref(c), y0, y1, halo,
                                                         C.byref(self.handle)))
        info = scene.info()
        self.width, self.height = info["width"], info["height"]
        a, b, c0, c1 = (C.c_int32() for _ in range(4))
        r._check(r._lib.tofr_gpu_session_band(self.handle, C.byref(a), C.byref(b), C.byref(c0), C.byref(c1)))
        self.y0, self.y1, self.r0, self.r1 = a.value, b.value, c0.value, c1.value
        self._xfn = None

    def step(self, stats: bool = True) -> dict | None:
        """One frame.  stats=False leaves the frame in flight (asynchronous)."""
        if not stats:
            self._r._check(self._r._lib.tofr_gpu_session_step(self.handle, None))
            return None
        st = F.FrameStats()
        self._r._check(self._r._lib.tofr_gpu_session_step(self.handle, C.byref(st)))
        return stats_to_dicts([st], 1)[0]

    def read_image(self, out: np.ndarray | None = None) -> np.ndarray:
        """Last frame's image of this session's rows, [y1 - y0, W, 3]."""
        if out is None:
            out = np.zeros((self.y1 - self.y0, self.width, 3))
        self._r._check(self._r._lib.tofr_gpu_session_read_image(self.handle, _dptr(out)))
        return out

    def read_image_async(self, pinned: np.ndarray, slot: int) -> None:
        """Enqueue this frame's image into `pinned` (page-locked, [rows, W, 3]); see wait_read."""
        self._r._check(self._r._lib.tofr_gpu_session_read_image_async(self.handle, _dptr(pinned), slot))

    def wait_read(self, slot: int) -> None:
        self._r._check(self._r._lib.tofr_gpu_session_wait_read(self.handle, slot))

    def read_histogram(self):
        """(rgb [rows, W, B, 3], count [rows, W, B]) accumulated so far / frames."""
        rows, B = self.y1 - self.y0, self.cfg.bins
        rgb = np.zeros((rows, self.width, B, 3))
        cnt = np.zeros((rows, self.width, B), dtype=np.int64)
        self._r._check(self._r._lib.tofr_gpu_session_read_histogram(
            self.handle, _dptr(rgb), cnt.ctypes.data_as(C.POINTER(C.c_int64))))
        return rgb, cnt

    def halo_buffers(self) -> dict:
        p = [C.c_void_p() for _ in range(4)]
        n = [C.c_uint64() for _ in range(2)]
        self._r._check(self._r._lib.tofr_gpu_session_halo_buffers(
            self.handle, C.byref(p[0]), C.byref(p[1]), C.byref(n[0]), C.byref(p[2]), C.byref(p[3]),
            C.byref(n[1])))
        return {"send_lo": int(p[0].value or 0), "recv_lo": int(p[1].value or 0), "bytes_lo": int(n[0].value),
                "send_hi": int(p[2].value or 0), "recv_hi": int(p[3].value or 0), "bytes_hi": int(n[1].value)}

    def halo_nccl(self, unique_id: bytes, rank: int, world: int) -> None:
        """Native NCCL halo transport (one process per GPU; every rank passes the
        same 128-byte id from Renderer.nccl_unique_id, broadcast by the host)."""
        self._r._check(self._r._lib.tofr_gpu_session_halo_nccl(self.handle, bytes(unique_id), int(rank),
                                                               int(world)))

    def link_halo(self, lower: "Session") -> None:
        """Native in-process transport: this band's bottom halo <-> the band
        directly below (peer copies on the session streams; each band is
        stepped from its own host thread)."""
        self._r._check(self._r._lib.tofr_gpu_session_link_halo(self.handle, lower.handle))

    def halo_transport(self) -> str:
        """"nccl", "peer", "callback" or "none"."""
        n = C.c_char_p()
        self._r._check(self._r._lib.tofr_gpu_session_halo_transport(self.handle, C.byref(n)))
        return n.value.decode()

    def set_halo_exchange(self, fn) -> None:
        """fn(pass) -> None: move the packed halo rows (see tofr_gpu.h)."""
        errors = self.halo_errors = []  # no reference back to self (no GC cycle)

        def _cb(user, pass_):
            try:
                fn(int(pass_))
                return 0
            except Exception as e:  # never unwind through the C ABI
                import traceback
                traceback.print_exc()
                errors.append(e)
                return 1
        self._xfn = F.HALO_FN(_cb)
        self._r._check(self._r._lib.tofr_gpu_session_set_halo_exchange(self.handle, self._xfn, None))

    def stage_totals(self, reset: bool = False):
        ms = (C.c_double * 6)()
        fr = C.c_int64()
        hx = C.c_uint64()
        self._r._check(self._r._lib.tofr_gpu_session_stage_totals(self.handle, ms, C.byref(fr), C.byref(hx),
                                                                  int(reset)))
        return list(ms), int(fr.value), int(hx.value)

    def last_ms(self):
        tot = C.c_double()
        st = (C.c_double * 6)()
        self._r._check(self._r._lib.tofr_gpu_session_last_ms(self.handle, C.byref(tot), st))
        return tot.value, list(st)

    def work(self) -> dict:
        """Device work since the session was created (waits for pending frames)."""
        w = (C.c_uint64 * 5)()
        self._r._check(self._r._lib.tofr_gpu_session_work(self.handle, w))
        return {"shift_jobs": int(w[0]), "rays_closest": int(w[1]), "rays_any": int(w[2]),
                "deposits": int(w[3]), "merges": int(w[4])}

    def pool(self) -> dict:
        """Sparse transient grids: pool rows held per grid now and rows per grid
        (cap 0: dense grids).  Waits for pending frames."""
        used = (C.c_uint64 * 3)()
        cap = C.c_uint64()
        self._r._check(self._r._lib.tofr_gpu_session_pool(self.handle, used, C.byref(cap)))
        return {"rows_used": [int(x) for x in used], "rows_cap": int(cap.value)}

    def row_cost(self, enable: bool):
        """Per-image-row shift cost counted since the last enable (numpy u64,
        image height), then counting on (enable) or off."""
        out = np.zeros(self.height, dtype=np.uint64)
        self._r._check(self._r._lib.tofr_gpu_session_row_cost(self.handle, int(enable),
                                                              out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return out

    def io_bytes(self):
        h2d, d2h = C.c_uint64(), C.c_uint64()
        self._r._check(self._r._lib.tofr_gpu_session_io_bytes(self.handle, C.byref(h2d), C.byref(d2h)))
        return int(h2d.value), int(d2h.value)

    def stream_ptr(self) -> int:
        p = C.c_void_p()
        self._r._check(self._r._lib.tofr_gpu_session_stream(self.handle, C.byref(p)))
        return int(p.value or 0)

    def sync(self) -> None:
        self._r._check(self._r._lib.tofr_gpu_session_sync(self.handle))

    def sync_stream(self) -> None:
        """Wait for the work enqueued so far (usable inside a halo callback)."""
        import torch
        torch.cuda.ExternalStream(self.stream_ptr()).synchronize()

    def close(self) -> None:
        """Free the session's device memory now (waits for its frames)."""
        if self.handle:
            self._r._lib.tofr_gpu_session_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default: Renderer | None = None


def default_renderer() -> Renderer:
    global _default
    if _default is None:
        _default = Renderer(0)
    return _default


def render_gated(scene, cfg: RenderConfig) -> RenderOutput:
    return default_renderer().render_gated(scene, cfg)


def render_transient(scene, cfg: RenderConfig) -> RenderOutput:
    return default_renderer().render_transient(scene, cfg)


def render_transient_plain(scene, cfg: RenderConfig) -> RenderOutput:
    return default_renderer().render_transient_plain(scene, cfg)


def render_doppler(scene, cfg: RenderConfig) -> RenderOutput:
    return default_renderer().render_doppler(scene, cfg)


def reference_render(scene, frame: float, gate: GateSpec, spp: int, seed: int, max_depth: int = 6):
    return default_renderer().reference_render(scene, frame, gate, spp, seed, max_depth)


def config_fields() -> list:
    return [f.name for f in fields(RenderConfig)]
