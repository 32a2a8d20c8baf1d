"""Image / histogram comparison helpers for the parity tests."""
from __future__ import annotations

import numpy as np

RTOL = 1e-4  # north star: per-pixel relative error vs the CPU oracle


def pixel_rel_err(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """max_c |a_c - b_c| / max_c |b_c| per pixel (0 where both are 0)."""
    a = a.reshape(-1, 3)
    b = b.reshape(-1, 3)
    num = np.abs(a - b).max(axis=1)
    den = np.maximum(np.abs(a).max(axis=1), np.abs(b).max(axis=1))
    out = np.zeros_like(num)
    nz = den > 0
    out[nz] = num[nz] / den[nz]
    return out


def summary(a: np.ndarray, b: np.ndarray, rtol: float = RTOL) -> dict:
    e = pixel_rel_err(a, b)
    n = e.size
    lit = (np.abs(b.reshape(-1, 3)).max(axis=1) > 0) | (np.abs(a.reshape(-1, 3)).max(axis=1) > 0)
    exact = np.all(a.reshape(-1, 3) == b.reshape(-1, 3), axis=1)
    return {
        "n": int(n),
        "lit": int(lit.sum()),
        "within": float((e <= rtol).mean()),
        "within_lit": float((e[lit] <= rtol).mean()) if lit.any() else 1.0,
        "bit_exact": float(exact.mean()),
        "max_rel": float(e.max()) if n else 0.0,
        "n_bad": int((e > rtol).sum()),
        "mean_a": float(a.mean()),
        "mean_b": float(b.mean()),
    }
