"""Host side of the CLI / harness (paper_2605_11536_b200/harness.py, cli.py)
against the reference's own implementations (oracle/_ref): compute_metrics
bit-for-bit, PFM / text-matrix files byte-for-byte, FNV-1a hashes, stats-line
format; CLI compare / stats verbs."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2605_11536_b200 import harness as Hn


@pytest.fixture(scope="module")
def ref():
    from oracle import ref as R
    if not R.available():
        R.build_if_possible()
    if not R.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return R


def _images(seed=3, h=17, w=23):
    rng = np.random.default_rng(seed)
    a = rng.gamma(0.5, 0.2, size=(h, w, 3))
    a[rng.random((h, w)) < 0.3] = 0.0
    b = a * rng.uniform(0.8, 1.2, size=a.shape) + rng.normal(0, 1e-3, size=a.shape)
    return np.abs(b), a


def test_compute_metrics_bit_exact(ref):
    est, r = _images()
    m = Hn.compute_metrics(est, r)
    rm, rr = ref.compute_metrics(est, r)
    assert (m.mape, m.relmse) == (rm, rr)


def test_image_files_byte_identical(ref, tmp_path):
    img, _ = _images(5)
    Hn.write_pfm(img, str(tmp_path / "a.pfm"))
    Hn.write_text_matrix(img, str(tmp_path / "a.txt"))
    ref.write_image(img, str(tmp_path / "b.pfm"), str(tmp_path / "b.txt"))
    assert (tmp_path / "a.pfm").read_bytes() == (tmp_path / "b.pfm").read_bytes()
    assert (tmp_path / "a.txt").read_bytes() == (tmp_path / "b.txt").read_bytes()
    assert Hn.hash_file(str(tmp_path / "a.pfm")) == ref.hash_file(str(tmp_path / "b.pfm"))
    back = Hn.read_pfm(str(tmp_path / "a.pfm"))
    assert np.array_equal(back, img.astype(np.float32).astype(np.float64))


def test_stats_lines_format(ref):
    """Byte-identical to stats_lines for the same counters and timings."""
    rng = np.random.default_rng(1)
    keys = ("attempts", "newton_ok", "newton_failed", "occluded", "jac_clamped", "replay_failed", "iterations",
            "solves", "success")
    stats = []
    for f in range(4):
        fs = {"frame": f, "t_init": float(rng.uniform(0, 2)), "t_shade": float(rng.uniform(0, 1e-3))}
        for st in ("temporal", "spatial", "bin"):
            d = {k: int(rng.integers(0, 10 ** int(rng.integers(0, 7)))) for k in keys}
            if st == "bin" or (st == "temporal" and f == 0):
                d = {k: 0 for k in keys}
            d["seconds"] = 0.0 if st == "bin" else float(rng.uniform(0, 3))
            fs[st] = d
        stats.append(fs)
    assert Hn.stats_lines(stats) == ref.stats_lines(stats)


def test_fit_line():
    f = Hn.fit_line([0, 1, 2, 3], [1, 3, 5, 7])
    assert (f.c0, f.c1, f.r2) == (1.0, 2.0, 1.0)


def test_cli_compare_and_stats(tmp_path, capsys):
    from paper_2605_11536_b200 import cli
    est, r = _images(9)
    Hn.write_pfm(est, str(tmp_path / "e.pfm"))
    Hn.write_pfm(r, str(tmp_path / "r.pfm"))
    (tmp_path / "s.txt").write_text("frame=0 stage=spatial attempts=10 success=4 actual_sr=0.4\n"
                                    "frame=1 stage=spatial attempts=20 success=6 actual_sr=0.3\n")
    assert cli.main(["compare", "--est", str(tmp_path / "e.pfm"), "--ref", str(tmp_path / "r.pfm")]) == 0
    m = Hn.compute_metrics(Hn.read_pfm(str(tmp_path / "e.pfm")), Hn.read_pfm(str(tmp_path / "r.pfm")))
    assert f"MAPE={m.mape:.6g}" in capsys.readouterr().out
    assert cli.main(["stats", "--file", str(tmp_path / "s.txt")]) == 0
    out = capsys.readouterr().out
    assert "attempts=30" in out and "actual_sr=0.35" in out
    assert cli.main(["compare", "--est", str(tmp_path / "nope.pfm"), "--ref", str(tmp_path / "r.pfm")]) == 2
