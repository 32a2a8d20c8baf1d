"""Regenerate the committed golden fixtures from the CPU reference
(oracle/_ref, built from /root/reference by `make -C oracle`).

  kat_vectors.json     RNG streams (rng.hpp), bin_of on boundary-heavy length
                       sets (transport.hpp:115-119), neighbour spiral offsets
                       (pipeline.hpp:232-258)
  smoke_cornell32.npz  image of __graft_entry__.smoke()'s render
  render_goldens.npz   images/histograms of a few small parity cases, for GPU
                       boxes where oracle/_ref is unavailable

Run:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from oracle import ref as R  # noqa: E402
from paper_2605_11536_b200 import scenes  # noqa: E402
from paper_2605_11536_b200.api import GateSpec, RenderConfig  # noqa: E402

GOLDEN_CASES = ["c1_cornell", "wide_reuse", "plain_cornell", "transient_temporal", "mirror_replay"]


def main():
    R.build_if_possible()
    rng = np.random.default_rng(2024)
    kat = {"rng": [], "bins": [], "neighbors": []}
    for _ in range(12):
        args = [int(v) for v in rng.integers(0, 2**31, size=5)]
        _, u = R.rng_stream(*args, 12)
        kat["rng"].append({"args": args, "u64": [int(x) for x in u]})
    for bins, t0, bw in ((4, 10.0, 0.5), (256, 8.0, 0.046875), (1024, 7.0, 0.01953125), (17, 9.95, 0.1 / 16)):
        edges = t0 + np.arange(bins + 1) * bw
        lens = np.concatenate([edges, np.nextafter(edges, np.inf), np.nextafter(edges, -np.inf),
                               rng.uniform(t0 - 0.5, t0 + bins * bw + 0.5, 64)])
        kat["bins"].append({"bins": bins, "t0": t0, "bw": bw, "lens": lens.tolist(),
                            "expect": R.bin_of(bins, t0, bw, lens).tolist()})
    for pix, pas, seed, frame in ((0, 0, 1, 0), (12345, 0, 1, 3), (2073599, 1, 7, 119), (999, 2, 99, 5)):
        off = R.neighbor_offsets(pix, pas, seed, frame, 5, 10.0)
        kat["neighbors"].append({"pix": pix, "pass": pas, "seed": seed, "frame": frame, "count": 5,
                                 "radius": 10.0, "offsets": off.tolist()})
    (HERE / "kat_vectors.json").write_text(json.dumps(kat))

    sd = scenes.bundled("cornell", 32)
    cfg = RenderConfig(gate=GateSpec(0, 10.0, 0.3, 1.0), m_init=2, temporal=True, spatial_passes=1,
                       spatial_neighbors=3, spatial_radius=5, frames=2, seed=11)
    img = R.render_gated(R.RefScene(sd), cfg).image
    np.savez_compressed(HERE / "smoke_cornell32.npz", image=img)

    from tests.cases import CASES
    out = {}
    for name in GOLDEN_CASES:
        build, c, kind = CASES[name]
        fn = {"gated": R.render_gated, "plain": R.render_transient_plain, "transient": R.render_transient}[kind]
        r = fn(R.RefScene(build()), c)
        out[name + "/image"] = r.image
        if r.hist is not None:
            out[name + "/hist_rgb"] = r.hist.rgb
            out[name + "/hist_count"] = r.hist.count
    np.savez_compressed(HERE / "render_goldens.npz", **out)
    print("wrote", sorted(p.name for p in HERE.iterdir()))


if __name__ == "__main__":
    main()
