"""CPU: pin the oracle before trusting it.

* The numpy restatement (oracle/restate.py) against the reference's own
  known-answer tests (test_transport.cpp, test_ris.cpp) and against the
  compiled reference (oracle/_ref) on random inputs.
* The committed golden vectors (tests/golden/) against both.
"""
from __future__ import annotations

import json
import math
from pathlib import Path

import numpy as np
import pytest

from oracle import restate as O

GOLD = Path(__file__).resolve().parent / "golden"


def test_bin_boundaries_kat():
    # test_transport.cpp:74-106: bins tile [10, 12] with width 0.5
    b = O.bin_of(4, 10.0, 0.5, [9.99, 10.0, 10.5, 11.0, 12.0, 12.0001])
    assert b.tolist() == [-1, 0, 1, 2, 3, -1]
    for L in (10.0, 10.25, 10.5, 11.3, 11.9999, 12.0):
        bb = int(O.bin_of(4, 10.0, 0.5, [L])[0])
        c, w = O.bin_gate(10.0, 0.5, bb)
        assert O.gate_weight(c, w, L) == 1.0
        assert O.gate_weight(11.0, 2.0, L) == 1.0  # covering gate


def test_gate_inclusive_kat():
    # test_transport.cpp:29-36
    assert O.gate_weight(10, 1, 10.0) == 1.0
    assert O.gate_weight(10, 1, 10.51) == 0.0
    assert O.gate_weight(10, 1, 10.5) == 1.0
    assert O.gate_weight(10, 1, 9.5) == 1.0
    assert O.gate_weight(10, 1, 9.4999) == 0.0


def test_reservoir_kats():
    # test_ris.cpp:22-38 reservoir update basics
    d = O.Stream(1, 0, 0, 0, 0)
    r = O.Reservoir()
    assert r.update("a", 1.5, 1.0, 2.0, d)
    assert r.M == 1.0 and r.w_sum == 1.5
    assert not r.update("b", 0.0, 1.0, 9.0, d)
    assert r.w_sum == 1.5 and r.M == 2.0 and r.y == "a"
    assert not r.update("c", float("nan"), 1.0, 1.0, d)
    assert r.nonfinite_rejected == 1
    # test_ris.cpp:59-75: if the second of phat (2, 6) wins, W = 4/6
    d = O.Stream(7, 0, 4, 0, 0)
    for _ in range(64):
        r = O.Reservoir()
        r.update(2.0, 0.5 * 2.0 * 1.0, 1, 2.0, d)
        r.update(6.0, 0.5 * 6.0 * 1.0, 1, 6.0, d)
        assert r.w_sum == pytest.approx(4.0)
        r.finalize()
        if r.y == 6.0:
            assert r.W == pytest.approx(2.0 / 3.0)
            break
    else:
        pytest.fail("second candidate never won")
    # test_ris.cpp:77-85 uniform targets -> W = 1/p
    d = O.Stream(3, 0, 0, 0, 0)
    r = O.Reservoir()
    for _ in range(10):
        r.update(5.0, (1.0 / 10) * 5.0 / 0.25, 1, 5.0, d)
    r.finalize()
    assert r.W == pytest.approx(4.0)


def test_merge_identity_and_empty():
    d = O.Stream(11, 0, 2, 0, 0)
    a = O.Reservoir()
    a.update("x", 2.0, 1, 2.0, d)
    a.finalize()
    a.M = 1
    e = O.Reservoir()
    e.M = 1
    out = O.gris_merge(a, e, False, 1.0, 0.0, None, 0.0, 20, d)
    assert out.y == "x" and out.M == 2 and out.W == pytest.approx(a.W)
    out2 = O.gris_merge(e, e, False, 1.0, 0.0, None, 0.0, 1.5, d)
    assert out2.empty() and out2.M == 1.5  # M cap


def test_rng_restatement_matches_reference(ref):
    rng = np.random.default_rng(0)
    for _ in range(20):
        seed, frame, pixel, sample, lane = (int(v) for v in rng.integers(0, 2**31, size=5))
        a, au = O.rng_stream(seed, frame, pixel, sample, lane, 16)
        b, bu = ref.rng_stream(seed, frame, pixel, sample, lane, 16)
        assert np.array_equal(au, bu)
        assert np.array_equal(a, b)


def test_bin_of_restatement_matches_reference(ref):
    rng = np.random.default_rng(1)
    for bins, t0, bw in ((256, 8.0, 0.046875), (1024, 7.0, 0.01953125), (17, 9.95, 0.1 / 16), (4, 10.0, 0.5)):
        lens = np.concatenate([rng.uniform(t0 - 1, t0 + bins * bw + 1, 20000),
                               t0 + np.arange(bins + 1) * bw,
                               np.nextafter(t0 + np.arange(bins + 1) * bw, np.inf),
                               np.nextafter(t0 + np.arange(bins + 1) * bw, -np.inf)])
        assert np.array_equal(O.bin_of(bins, t0, bw, lens), ref.bin_of(bins, t0, bw, lens))


def test_golden_vectors_against_restatement():
    g = json.loads((GOLD / "kat_vectors.json").read_text())
    for s in g["rng"]:
        v, u = O.rng_stream(*s["args"], len(s["u64"]))
        assert [int(x) for x in u] == s["u64"]
    for h in g["bins"]:
        assert O.bin_of(h["bins"], h["t0"], h["bw"], h["lens"]).tolist() == h["expect"]
    for n in g["neighbors"]:
        key = O.spatial_rot_key(n["pix"], n["pass"], n["seed"], n["frame"])
        got = [list(O.neighbor_offset(j, n["count"], n["radius"], key)) for j in range(n["count"])]
        assert got == n["offsets"]


def test_neighbor_offsets_finite_and_bounded():
    for pix in range(0, 5000, 37):
        key = O.spatial_rot_key(pix, 0, 1, 3)
        for j in range(5):
            dx, dy = O.neighbor_offset(j, 5, 10.0, key)
            assert math.hypot(dx, dy) <= 10.0 + 1.0
