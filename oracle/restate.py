"""oracle/restate.py -- TEST INFRASTRUCTURE ONLY.

A CPU restatement (numpy / pure Python) of the integer- and index-level parts
of the reference hot path, each function citing the reference it follows.
The full renderer oracle is the reference itself (oracle/_ref, built from the
unmodified headers); this module pins the parts whose parity bar is
bit-exactness (RNG streams, bin indexing, gate membership, neighbour offsets,
reservoir arithmetic) and is itself pinned by tests/test_oracle.py against
the reference's known-answer tests and against oracle/_ref.
"""
from __future__ import annotations

import math

import numpy as np

U64 = np.uint64
_M = (1 << 64) - 1


def mix64(x):
    """splitmix64 finalizer (rng.hpp:9-15); numpy uint64 arrays or Python ints."""
    if isinstance(x, (int, np.integer)) and not isinstance(x, np.ndarray):
        x = (int(x) + 0x9E3779B97F4A7C15) & _M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M
        return x ^ (x >> 31)
    x = np.asarray(x, dtype=U64)
    with np.errstate(over="ignore"):
        x = x + U64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> U64(30))) * U64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> U64(27))) * U64(0x94D049BB133111EB)
    return x ^ (x >> U64(31))


def rng_key(seed, frame, pixel, sample, lane) -> int:
    """Rng(seed, frame, pixel, sample, lane) key chain (rng.hpp:23-31)."""
    k = mix64((seed ^ 0x5BD1E995) & _M)
    k = mix64(k ^ (frame & _M))
    k = mix64(k ^ ((pixel * 0x9E3779B97F4A7C15) & _M))
    k = mix64(k ^ ((sample * 0xC2B2AE3D27D4EB4F) & _M))
    k = mix64(k ^ ((lane * 0x165667B19E3779F9) & _M))
    return k


def rng_u64(key: int, counter: int) -> int:
    """next_u64 for the draw with post-increment counter value `counter`
    (rng.hpp:36): mix64(key ^ (golden * counter))."""
    return mix64(key ^ ((0x9E3779B97F4A7C15 * counter) & _M))


def rng_stream(seed, frame, pixel, sample, lane, n):
    """First n next() draws of a stream: top 53 bits * 2^-53 (rng.hpp:39)."""
    k = rng_key(seed, frame, pixel, sample, lane)
    u = [rng_u64(k, c) for c in range(1, n + 1)]
    return np.array([float(v >> 11) * 2.0 ** -53 for v in u]), np.array(u, dtype=U64)


def gate_weight(center: float, width: float, length):
    """Inclusive box gate |len - center| <= width/2 (transport.hpp:25-27)."""
    return np.where(np.abs(np.asarray(length) - center) <= width / 2, 1.0, 0.0)


def bin_of(bins: int, t0: float, bw: float, length):
    """TransientHistogram::bin_of (transport.hpp:115-119): reject outside
    [t0, t0 + bins*bw], truncate, closed final bin."""
    L = np.asarray(length, dtype=np.float64)
    out = np.full(L.shape, -1, dtype=np.int64)
    ok = ~((L < t0) | (L > t0 + bins * bw))
    b = np.trunc((L[ok] - t0) / bw).astype(np.int64)
    out[ok] = np.minimum(b, bins - 1)
    return out


def bin_gate(t0: float, bw: float, b: int):
    """bin_gate(b) = {t0 + (b + 0.5) * bw, bw} (transport.hpp:112)."""
    return t0 + (b + 0.5) * bw, bw


def deposit(hist_rgb, hist_count, x, y, bins, t0, bw, length, value):
    """TransientHistogram::deposit (transport.hpp:121-126), one candidate."""
    b = int(bin_of(bins, t0, bw, [length])[0])
    if b < 0:
        return
    hist_rgb[y, x, b] += value
    hist_count[y, x, b] += 1


def spatial_rot_key(pix: int, pass_: int, seed: int, frame_idx: int) -> int:
    """Rotation key of the neighbour spiral (pipeline.hpp:256-258); note the
    32-bit unsigned product `pass * 2654435761u`."""
    a = (pix * 1315423911) & _M
    b = (pass_ * 2654435761) & 0xFFFFFFFF
    return mix64((a + b + seed + frame_idx * 97) & _M)


def neighbor_offset(j: int, count: int, radius: float, rot_key: int):
    """Golden-angle spiral offset (pipeline.hpp:232-239)."""
    rot = float(mix64(rot_key) >> 11) * 2.0 ** -53 * 2.0 * math.pi
    rr = radius * math.sqrt((j + 0.5) / count)
    th = j * 2.39996322972865332 + rot
    return _lround(rr * math.cos(th)), _lround(rr * math.sin(th))


def _lround(v: float) -> int:
    """std::lround: round half away from zero."""
    return int(math.floor(v + 0.5)) if v >= 0 else -int(math.floor(-v + 0.5))


def luminance(c) -> float:
    return 0.2126 * c[0] + 0.7152 * c[1] + 0.0722 * c[2]  # math.hpp:75


class Reservoir:
    """Weighted reservoir (ris.hpp:20-56) over opaque samples."""

    def __init__(self):
        self.y = None
        self.has = False
        self.w_sum = 0.0
        self.W = 0.0
        self.M = 0.0
        self.phat = 0.0
        self.nonfinite_rejected = 0

    def empty(self) -> bool:
        return not self.has or self.W <= 0

    def update(self, cand, w: float, m_c: float, phat: float, draw) -> bool:
        """reservoir_update (ris.hpp:34-50); `draw()` returns the next uniform."""
        self.M += m_c
        if not math.isfinite(w) or w < 0:
            self.nonfinite_rejected += 1
            return False
        if w <= 0:
            return False
        self.w_sum += w
        if draw() * self.w_sum < w:
            self.y = cand
            self.has = True
            self.phat = phat
            return True
        return False

    def finalize(self) -> None:
        """ris_finalize (ris.hpp:53-56)."""
        self.W = self.w_sum / self.phat if (self.has and self.phat > 0) else 0.0


def gris_merge(dst: Reservoir, src: Reservoir, valid: bool, jac: float, phat_src_of_dst: float, mapped,
               phat_mapped: float, m_cap: float, draw) -> Reservoir:
    """gris_merge (ris.hpp:78-104): generalized balance heuristic with the
    defensive confidence weights and the M cap."""
    Mc, Ms = dst.M, src.M
    out = Reservoir()
    if not dst.empty():
        pc = dst.phat
        num = Mc * pc
        den = num + Ms * phat_src_of_dst
        m_c = num / den if den > 0 else 0.0
        out.update(dst.y, m_c * pc * dst.W, 0, pc, draw)
    if not src.empty() and valid and jac > 0:
        py = phat_mapped
        if py > 0:
            num = Ms * src.phat / jac
            den = Mc * py + num
            m_s = num / den if den > 0 else 0.0
            out.update(mapped, m_s * py * src.W * jac, 0, py, draw)
    out.M = m_cap if m_cap < Mc + Ms else Mc + Ms  # std::min(Mc + Ms, m_cap)
    out.nonfinite_rejected = dst.nonfinite_rejected
    out.finalize()
    return out


class Stream:
    """A counter-RNG stream as a draw() callable (rng.hpp:219-247)."""

    def __init__(self, seed, frame, pixel, sample, lane):
        self.key = rng_key(seed, frame, pixel, sample, lane)
        self.counter = 0

    def __call__(self) -> float:
        self.counter += 1
        return float(rng_u64(self.key, self.counter) >> 11) * 2.0 ** -53
