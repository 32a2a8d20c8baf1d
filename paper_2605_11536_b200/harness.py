"""Measurement harness and on-disk formats of the reference,
on top of the B200 render API.

    compute_metrics(est, ref)                      pipeline.hpp:580-607 (MAPE, relMSE)
    render_equal_time(renderer, scene, cfg, s)     harness.hpp:40-64
    fit_line(x, y)                                 harness.hpp:66-94
    min_path_length_bound(scene, frame)            harness.hpp:96-111
    write_pfm / read_pfm / write_text_matrix       image.hpp:41-88
    hash_file (FNV-1a 64)                          image.hpp:90-106
    write_histogram_csv                            tools/tofr.cpp:148-161
    stats_lines                                    pipeline.hpp:612-633

Host-side arithmetic follows the reference's summation order (sequential
sums via cumulative sums), so metrics computed here equal the reference's
for the same images.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field, replace

import numpy as np

from . import _ffi as F
from .api import RenderConfig, Renderer, Scene

SHIFT_KEYS = ("attempts", "newton_ok", "newton_failed", "occluded", "jac_clamped", "replay_failed", "iterations",
              "solves", "success")


def _seqsum(a: np.ndarray) -> float:
    """Left-to-right float64 sum (the reference's loop order)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    return float(np.cumsum(a)[-1]) if a.size else 0.0


@dataclass
class Metrics:  # pipeline.hpp:583-586
    mape: float = 0.0
    relmse: float = 0.0


def compute_metrics(est: np.ndarray, ref: np.ndarray) -> Metrics:
    """compute_metrics (pipeline.hpp:588-607): eps = 1% of the reference's
    mean luminance-free average, per-channel MAPE and relative MSE."""
    m = Metrics()
    if est.shape != ref.shape or est.size == 0:
        return m
    r = ref.reshape(-1, 3).astype(np.float64)
    e = est.reshape(-1, 3).astype(np.float64)
    eps = _seqsum(((r[:, 0] + r[:, 1]) + r[:, 2]) / 3.0)
    eps = 1e-2 * (eps / float(r.shape[0]))
    d = e - r
    m.mape = _seqsum(np.abs(d) / (r + eps)) / float(r.size)
    m.relmse = _seqsum(d * d / (r * r + eps)) / float(r.size)
    return m


def image_mean(img: np.ndarray) -> float:
    """Image::mean (image.hpp:33-37)."""
    p = img.reshape(-1, 3)
    return _seqsum(((p[:, 0] + p[:, 1]) + p[:, 2]) / 3.0) / p.shape[0] if p.size else 0.0


@dataclass
class EqualTimeResult:  # harness.hpp:32-37
    image: np.ndarray
    repetitions: int = 0
    seconds: float = 0.0
    spatial: dict = field(default_factory=lambda: {k: 0 for k in SHIFT_KEYS})
    temporal: dict = field(default_factory=lambda: {k: 0 for k in SHIFT_KEYS})
    binwise: dict = field(default_factory=lambda: {k: 0 for k in SHIFT_KEYS})


def render_equal_time(renderer: Renderer, scene, base: RenderConfig, budget_seconds: float, min_reps: int = 1,
                      max_reps: int = 1 << 20) -> EqualTimeResult:
    """render_equal_time (harness.hpp:40-64): independent renders with stepped
    seeds (seed + rep * 0x9e3779b9) until the time budget is spent, averaged."""
    s = renderer._scene(scene)
    info = s.info()
    out = EqualTimeResult(image=np.zeros((info["height"], info["width"], 3)))
    t0 = time.perf_counter()
    for rep in range(max_reps):
        if rep >= min_reps and time.perf_counter() - t0 >= budget_seconds:
            break
        cfg = replace(base, seed=(base.seed + rep * 0x9E3779B9) & 0xFFFFFFFFFFFFFFFF)
        r = (renderer.render_transient(s, cfg) if cfg.mode == F.MODE_TRANSIENT else
             renderer.render_doppler(s, cfg) if cfg.gate.kind == F.GATE_VELOCITY else renderer.render_gated(s, cfg))
        out.image += r.image
        for fs in r.stats:
            for k in SHIFT_KEYS:
                out.spatial[k] += fs["spatial"][k]
                out.temporal[k] += fs["temporal"][k]
                out.binwise[k] += fs["bin"][k]
        out.repetitions += 1
    out.seconds = time.perf_counter() - t0
    if out.repetitions > 0:
        out.image *= 1.0 / out.repetitions
    return out


def actual_sr(c: dict) -> float:  # ShiftCounts::actual_sr (shiftmap.hpp:414)
    return c["success"] / c["attempts"] if c["attempts"] else 0.0


def mean_iterations(c: dict) -> float:
    return c["iterations"] / c["solves"] if c["solves"] else 0.0


def newton_sr(c: dict) -> float:
    return c["newton_ok"] / c["solves"] if c["solves"] else 0.0


@dataclass
class LineFit:
    c0: float = 0.0
    c1: float = 0.0
    r2: float = 0.0


def fit_line(x, y) -> LineFit:
    """Least squares y = c0 + c1 x (harness.hpp:71-94)."""
    f = LineFit()
    n = len(x)
    if n < 2:
        return f
    sx = sy = sxx = sxy = 0.0
    for xi, yi in zip(x, y):
        sx += xi
        sy += yi
        sxx += xi * xi
        sxy += xi * yi
    den = n * sxx - sx * sx
    if den == 0:
        return f
    f.c1 = (n * sxy - sx * sy) / den
    f.c0 = (sy - f.c1 * sx) / n
    my = sy / n
    ss_res = ss_tot = 0.0
    for xi, yi in zip(x, y):
        pred = f.c0 + f.c1 * xi
        ss_res += (yi - pred) * (yi - pred)
        ss_tot += (yi - my) * (yi - my)
    f.r2 = 1.0 - ss_res / ss_tot if ss_tot > 0 else 1.0
    return f


def min_path_length_bound(scene, frame: float, cam_pos, light_pos) -> float:
    """Closest approach of camera and light to the scene bounds (harness.hpp:96-111)."""
    s = scene if isinstance(scene, Scene) else Scene.create(scene)
    nodes, _, _, _ = s.dump_bvh(frame)
    lo, hi = nodes[0, 0:3], nodes[0, 3:6]

    def dist(p):
        d2 = 0.0
        for a in range(3):
            d = max(lo[a] - p[a], p[a] - hi[a], 0.0)
            d2 += d * d
        return float(np.sqrt(d2))

    return dist(cam_pos) + dist(light_pos)


# ---------------------------------------------------------------------------
# file formats (image.hpp, tools/tofr.cpp)

def write_pfm(img: np.ndarray, path: str) -> None:
    """Little-endian RGB PFM, rows bottom-to-top, float32 (image.hpp:41-56)."""
    h, w = img.shape[:2]
    with open(path, "wb") as f:
        f.write(f"PF\n{w} {h}\n-1.0\n".encode())
        f.write(np.ascontiguousarray(img[::-1].astype("<f4")).tobytes())


def read_pfm(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        data = f.read()
    parts = data.split(None, 4)
    if len(parts) < 4 or parts[0] != b"PF":
        raise ValueError(f"{path}: not a color PFM")
    w, h = int(parts[1]), int(parts[2])
    # header: "PF" ws w ws h ws scale + single whitespace
    hdr_end = 0
    fields = 0
    i = 0
    while fields < 4:
        while data[i:i + 1].isspace():
            i += 1
        while i < len(data) and not data[i:i + 1].isspace():
            i += 1
        fields += 1
    hdr_end = i + 1
    raw = np.frombuffer(data, dtype="<f4", count=w * h * 3, offset=hdr_end)
    if raw.size != w * h * 3:
        raise ValueError(f"{path}: truncated PFM")
    return raw.reshape(h, w, 3)[::-1].astype(np.float64)


def _g17(v: float) -> str:
    return format(float(v), ".17g")


def write_text_matrix(img: np.ndarray, path: str) -> None:
    """"H W" header then one "r g b" triple per pixel, row-major, 17 digits (image.hpp:71-82)."""
    h, w = img.shape[:2]
    with open(path, "w") as f:
        f.write(f"{h} {w}\n")
        for p in img.reshape(-1, 3):
            f.write(f"{_g17(p[0])} {_g17(p[1])} {_g17(p[2])}\n")


def fnv1a64(data: bytes, h: int = 0xCBF29CE484222325) -> int:
    for b in data:
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def hash_file(path: str) -> int:
    """hash_file (image.hpp:99-106): FNV-1a 64 of the file bytes (native)."""
    with open(path, "rb") as f:
        data = f.read()
    return int(F.load_library().tofr_fnv1a64(data, len(data)))


def write_histogram_csv(hist, path: str) -> None:
    """pixel_x,pixel_y,bin,r,g,b,count with 10 significant digits (tools/tofr.cpp:148-161)."""
    rgb, cnt = hist.rgb, hist.count
    H, W, B = cnt.shape
    with open(path, "w") as f:
        f.write("pixel_x,pixel_y,bin,r,g,b,count\n")
        for y in range(H):
            for x in range(W):
                for b in range(B):
                    v = rgb[y, x, b]
                    f.write(f"{x},{y},{b},{v[0]:.10g},{v[1]:.10g},{v[2]:.10g},{int(cnt[y, x, b])}\n")


def stats_lines(stats: list) -> str:
    """Line-delimited key=value records (pipeline.hpp:612-633)."""
    out = []
    g = lambda v: format(float(v), ".6g")  # noqa: E731 -- std::ostream default precision
    for fs in stats:
        fr = fs["frame"]
        out.append(f"frame={fr} stage=init seconds={g(fs['t_init'])}")
        for stage in ("temporal", "spatial", "bin"):
            s = fs[stage]
            if s["attempts"] == 0 and s["seconds"] == 0:
                continue
            out.append(f"frame={fr} stage={stage} attempts={s['attempts']} solves={s['solves']} "
                       f"converged={s['newton_ok']} newton_failed={s['newton_failed']} occluded={s['occluded']} "
                       f"jacobian_clamped={s['jac_clamped']} replay_failed={s['replay_failed']} "
                       f"success={s['success']} mean_iterations={g(mean_iterations(s))} "
                       f"newton_sr={g(newton_sr(s))} actual_sr={g(actual_sr(s))} seconds={g(s['seconds'])}")
        out.append(f"frame={fr} stage=shade seconds={g(fs['t_shade'])}")
    return "".join(line + "\n" for line in out)
