"""ctypes mirror of include/tofr_gpu.h (structs, enums, prototypes).

Shared by the product bindings (api.py -> libtofr_b200.so) and the test
oracle wrapper (oracle/ref.py -> oracle/_ref/libtofr_ref.so), which take the
same plain-C scene and config structs.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

TOFR_OK = 0
TOFR_ERR_INVALID = 1
TOFR_ERR_PARSE = 2
TOFR_ERR_SCENE = 3
TOFR_ERR_CUDA = 4
TOFR_ERR_OOM = 5
TOFR_ERR_UNSUPPORTED = 6

MAT_DIFFUSE, MAT_GLOSSY, MAT_MIRROR = 0, 1, 2
LIGHT_COLLIMATED, LIGHT_WIDE = 0, 1
MODE_GATED, MODE_TRANSIENT, MODE_DOPPLER = 0, 1, 2
INIT_DIRECT, INIT_ELLIPSOIDAL, INIT_SHRINK = 0, 1, 2
GAUGE_FIXED, GAUGE_RAW, GAUGE_AVG = 0, 1, 2
GATE_LENGTH, GATE_VELOCITY = 0, 1

D3 = C.c_double * 3


class Material(C.Structure):
    _fields_ = [("kind", C.c_int32), ("albedo", D3), ("roughness", C.c_double)]


class Light(C.Structure):
    _fields_ = [("regime", C.c_int32), ("position", D3), ("direction", D3),
                ("cone_half_angle", C.c_double), ("intensity", D3)]


class CameraKey(C.Structure):
    _fields_ = [("frame", C.c_double), ("position", D3), ("forward", D3), ("up", D3)]


class PoseKey(C.Structure):
    _fields_ = [("frame", C.c_double), ("q", C.c_double * 4), ("t", D3)]


class ObjectDesc(C.Structure):
    _fields_ = [("name", C.c_char_p), ("n_tris", C.c_int32), ("verts", C.POINTER(C.c_double)),
                ("materials", C.POINTER(C.c_int32)), ("n_keys", C.c_int32), ("keys", C.POINTER(PoseKey))]


class SceneDesc(C.Structure):
    _fields_ = [("cam_position", D3), ("cam_forward", D3), ("cam_up", D3), ("fov_y", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("n_cam_keys", C.c_int32),
                ("cam_keys", C.POINTER(CameraKey)), ("n_materials", C.c_int32),
                ("materials", C.POINTER(Material)), ("light", Light), ("n_objects", C.c_int32),
                ("objects", C.POINTER(ObjectDesc)), ("dt_frame", C.c_double)]


class RenderConfigC(C.Structure):
    _fields_ = [("mode", C.c_int32), ("gate_kind", C.c_int32), ("gate_center", C.c_double),
                ("gate_width", C.c_double), ("gate_f0", C.c_double), ("gate_step", C.c_double),
                ("bins", C.c_int32), ("hist_t0", C.c_double), ("hist_bin_width", C.c_double),
                ("m_init", C.c_int32), ("init_mode", C.c_int32), ("shrink_k", C.c_double),
                ("shrink_r", C.c_double), ("spatial_passes", C.c_int32), ("spatial_neighbors", C.c_int32),
                ("spatial_radius", C.c_double), ("temporal", C.c_int32), ("bin_reuse", C.c_int32),
                ("m_cap", C.c_double), ("gauge", C.c_int32), ("newton", C.c_int32), ("seed", C.c_uint64),
                ("frames", C.c_int32), ("frame0", C.c_double), ("max_depth", C.c_int32),
                ("use_rr", C.c_int32), ("accumulate", C.c_int32), ("normalize_gate", C.c_int32)]


class ShiftCounts(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("attempts", "newton_ok", "newton_failed", "occluded", "jac_clamped",
                                          "replay_failed", "iterations", "solves", "success")]

    def as_dict(self) -> dict:
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class StageStats(C.Structure):
    _fields_ = [("shift", ShiftCounts), ("seconds", C.c_double)]


class FrameStats(C.Structure):
    _fields_ = [("frame", C.c_int32), ("temporal", StageStats), ("spatial", StageStats),
                ("binwise", StageStats), ("t_init", C.c_double), ("t_shade", C.c_double)]


class Output(C.Structure):
    _fields_ = [("image", C.POINTER(C.c_double)), ("hist_rgb", C.POINTER(C.c_double)),
                ("hist_count", C.POINTER(C.c_int64)), ("stats", C.POINTER(FrameStats)),
                ("stats_capacity", C.c_int32)]


# int (*tofr_halo_exchange_fn)(void* user, int32_t pass)
HALO_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32)

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "_native" / "libtofr_b200.so"

_lib = None


def _declare(lib) -> None:
    P = C.POINTER
    vp = C.c_void_p
    lib.tofr_render_config_default.argtypes = [P(RenderConfigC)]
    lib.tofr_render_config_default.restype = None
    lib.tofr_gpu_create.argtypes = [P(C.c_int), C.c_int, P(vp)]
    lib.tofr_gpu_destroy.argtypes = [vp]
    lib.tofr_gpu_destroy.restype = None
    lib.tofr_gpu_last_error.argtypes = [vp]
    lib.tofr_gpu_last_error.restype = C.c_char_p
    lib.tofr_gpu_version.restype = C.c_char_p
    lib.tofr_scene_create.argtypes = [P(SceneDesc), P(vp), C.c_char_p, C.c_size_t]
    lib.tofr_scene_parse.argtypes = [C.c_char_p, C.c_char_p, P(vp), C.c_char_p, C.c_size_t]
    lib.tofr_scene_load.argtypes = [C.c_char_p, P(vp), C.c_char_p, C.c_size_t]
    lib.tofr_scene_destroy.argtypes = [vp]
    lib.tofr_scene_destroy.restype = None
    lib.tofr_scene_set_resolution.argtypes = [vp, C.c_int32, C.c_int32]
    lib.tofr_scene_info.argtypes = [vp, P(C.c_int32), P(C.c_int32), P(C.c_int32), P(C.c_int32), P(C.c_double),
                                    C.c_char_p, C.c_size_t]
    for name in ("tofr_gpu_render_gated", "tofr_gpu_render_doppler", "tofr_gpu_render_transient",
                 "tofr_gpu_render_transient_plain"):
        getattr(lib, name).argtypes = [vp, vp, P(RenderConfigC), P(Output)]
    lib.tofr_gpu_reference.argtypes = [vp, vp, C.c_double, C.c_double, C.c_double, C.c_int32, C.c_uint64,
                                       C.c_int32, P(C.c_double), P(C.c_double)]
    lib.tofr_gpu_session_create.argtypes = [vp, vp, P(RenderConfigC), P(vp)]
    lib.tofr_gpu_session_step.argtypes = [vp, P(FrameStats)]
    lib.tofr_gpu_session_read_image.argtypes = [vp, P(C.c_double)]
    lib.tofr_gpu_session_sync.argtypes = [vp]
    lib.tofr_gpu_session_last_ms.argtypes = [vp, P(C.c_double), P(C.c_double)]
    lib.tofr_gpu_session_stream.argtypes = [vp, P(vp)]
    lib.tofr_gpu_session_create_band.argtypes = [vp, vp, P(RenderConfigC), C.c_int32, C.c_int32, C.c_int32, P(vp)]
    lib.tofr_gpu_session_create_plain.argtypes = [vp, vp, P(RenderConfigC), C.c_int32, C.c_int32, P(vp)]
    lib.tofr_gpu_session_read_histogram.argtypes = [vp, P(C.c_double), P(C.c_int64)]
    lib.tofr_gpu_session_read_image_async.argtypes = [vp, P(C.c_double), C.c_int32]
    lib.tofr_gpu_session_wait_read.argtypes = [vp, C.c_int32]
    lib.tofr_gpu_session_band.argtypes = [vp] + [P(C.c_int32)] * 4
    lib.tofr_gpu_session_set_halo_exchange.argtypes = [vp, HALO_FN, vp]
    lib.tofr_gpu_session_halo_buffers.argtypes = [vp, P(vp), P(vp), P(C.c_uint64), P(vp), P(vp), P(C.c_uint64)]
    lib.tofr_gpu_nccl_unique_id.argtypes = [C.c_char_p]
    lib.tofr_gpu_session_halo_nccl.argtypes = [vp, C.c_char_p, C.c_int32, C.c_int32]
    lib.tofr_gpu_session_link_halo.argtypes = [vp, vp]
    lib.tofr_gpu_session_halo_transport.argtypes = [vp, P(C.c_char_p)]
    lib.tofr_gpu_session_stage_totals.argtypes = [vp, P(C.c_double), P(C.c_int64), P(C.c_uint64), C.c_int32]
    lib.tofr_gpu_session_io_bytes.argtypes = [vp, P(C.c_uint64), P(C.c_uint64)]
    lib.tofr_gpu_session_destroy.argtypes = [vp]
    lib.tofr_gpu_session_destroy.restype = None
    lib.tofr_gpu_session_work.argtypes = [vp, P(C.c_uint64)]
    lib.tofr_gpu_session_pool.argtypes = [vp, P(C.c_uint64), P(C.c_uint64)]
    lib.tofr_gpu_session_row_cost.argtypes = [vp, C.c_int32, P(C.c_uint64)]
    lib.tofr_gpu_kernel_timing.argtypes = [C.c_int32]
    lib.tofr_gpu_kernel_launches.argtypes = []
    lib.tofr_gpu_kernel_launches.restype = C.c_uint64
    lib.tofr_gpu_kernel_times.argtypes = [C.c_char_p, C.c_int32, P(C.c_double), P(C.c_uint64), C.c_int32]
    lib.tofr_gpu_kernel_times_reset.argtypes = []
    lib.tofr_gpu_kernel_times_reset.restype = None
    lib.tofr_fnv1a64.argtypes = [C.c_char_p, C.c_uint64]
    lib.tofr_fnv1a64.restype = C.c_uint64
    lib.tofr_gpu_selftest_div.argtypes = [vp, C.c_uint64, C.c_uint64, P(C.c_uint64)]
    lib.tofr_gpu_fp64_peak.argtypes = [vp, P(C.c_double)]
    lib.tofr_gpu_dump_bvh_device.argtypes = [vp, vp, C.c_double, C.c_int32, P(C.c_double), P(C.c_int32),
                                             P(C.c_int32), C.c_int32, P(C.c_int32), P(C.c_int32), P(C.c_double)]
    lib.tofr_gpu_debug_solve_profile.argtypes = [P(C.c_uint64), C.c_uint64, P(C.c_uint64)]
    lib.tofr_gpu_debug_check_selftest.argtypes = [vp, P(C.c_int32)]
    lib.tofr_gpu_probe_rays.argtypes = [vp, vp, C.c_double, P(C.c_double), C.c_int32, C.c_int32,
                                        P(C.c_double), P(C.c_int32)]
    lib.tofr_scene_probe_rays_host.argtypes = [vp, C.c_double, P(C.c_double), C.c_int32, C.c_int32,
                                               P(C.c_double), P(C.c_int32), C.c_char_p, C.c_size_t]
    lib.tofr_scene_dump_bvh.argtypes = [vp, C.c_double, C.c_int32, P(C.c_double), P(C.c_int32), P(C.c_int32),
                                        C.c_int32, P(C.c_int32), P(C.c_int32), P(C.c_double), C.c_char_p,
                                        C.c_size_t]


EXPORTED_SYMBOLS = (
    "tofr_render_config_default", "tofr_gpu_create", "tofr_gpu_destroy", "tofr_gpu_last_error",
    "tofr_gpu_version", "tofr_scene_create", "tofr_scene_parse", "tofr_scene_load", "tofr_scene_destroy",
    "tofr_scene_set_resolution", "tofr_scene_info", "tofr_gpu_render_gated", "tofr_gpu_render_doppler",
    "tofr_gpu_render_transient", "tofr_gpu_render_transient_plain", "tofr_gpu_reference",
    "tofr_gpu_session_create", "tofr_gpu_session_step", "tofr_gpu_session_read_image", "tofr_gpu_session_sync",
    "tofr_gpu_session_last_ms", "tofr_gpu_session_io_bytes", "tofr_gpu_session_stream",
    "tofr_gpu_session_create_band", "tofr_gpu_session_band", "tofr_gpu_session_set_halo_exchange",
    "tofr_gpu_session_halo_buffers", "tofr_gpu_nccl_unique_id", "tofr_gpu_session_halo_nccl",
    "tofr_gpu_session_link_halo", "tofr_gpu_session_halo_transport", "tofr_gpu_session_stage_totals", "tofr_gpu_session_create_plain",
    "tofr_gpu_session_read_histogram", "tofr_gpu_session_read_image_async", "tofr_gpu_session_wait_read", "tofr_gpu_session_work", "tofr_gpu_session_pool", "tofr_gpu_session_row_cost", "tofr_gpu_session_destroy",
    "tofr_gpu_kernel_timing", "tofr_gpu_kernel_launches", "tofr_gpu_kernel_times", "tofr_gpu_kernel_times_reset",
    "tofr_fnv1a64", "tofr_gpu_selftest_div", "tofr_gpu_fp64_peak", "tofr_gpu_dump_bvh_device", "tofr_gpu_debug_solve_profile", "tofr_gpu_debug_check_selftest", "tofr_gpu_probe_rays", "tofr_scene_probe_rays_host", "tofr_scene_dump_bvh",
)


def load_library(path: Path | None = None):
    """Load libtofr_b200.so.  Raises if the native library is missing: there
    is no CPU fallback for the product path."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    import os
    p = Path(path) if path else Path(os.environ.get("TOFR_B200_LIB", LIB_PATH))
    if not p.exists():
        raise RuntimeError(f"native library {p} is missing; run __graft_entry__.build() "
                           "(the GPU path has no fallback)")
    lib = C.CDLL(str(p))
    _declare(lib)
    if path is None:
        _lib = lib
    return lib


# ---------------------------------------------------------------------------
# launch accounting (tofr_gpu_kernel_*)

def kernel_timing(enable: bool) -> bool:
    return bool(load_library().tofr_gpu_kernel_timing(1 if enable else 0))


def kernel_launches() -> int:
    return int(load_library().tofr_gpu_kernel_launches())


def kernel_times(reset: bool = False) -> dict:
    """{kernel name: (total ms, launches)} of the launches timed so far."""
    lib = load_library()
    cap, nl = 64, 48
    names = C.create_string_buffer(cap * nl)
    ms = (C.c_double * cap)()
    n = (C.c_uint64 * cap)()
    k = lib.tofr_gpu_kernel_times(names, nl, ms, n, cap)
    out = {}
    for i in range(k):
        nm = names.raw[i * nl:(i + 1) * nl].split(b"\0", 1)[0].decode()
        out[nm] = (float(ms[i]), int(n[i]))
    if reset:
        lib.tofr_gpu_kernel_times_reset()
    return out

