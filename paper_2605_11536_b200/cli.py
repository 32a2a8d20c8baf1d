"""tofr command-line driver on the B200 path (tools/tofr.cpp).

    python -m paper_2605_11536_b200 render    --scene s.scn [--mode gated|transient|doppler] ... --out prefix
    python -m paper_2605_11536_b200 reference --scene s.scn --spp N ...
    python -m paper_2605_11536_b200 compare   --est a.pfm --ref b.pfm [--stats s.txt]
    python -m paper_2605_11536_b200 stats     --file prefix_stats.txt
    python -m paper_2605_11536_b200 sweep     --scene s.scn --type gatewidth|kr|bins --budget S --values ...

Same options, defaults and output files as the reference CLI: <out>.pfm,
<out>.txt, <out>_hist.csv (transient), <out>_stats.txt, <out>_manifest.json
(scene FNV-1a hash, configuration, seconds, output hashes).  Errors map to
exit code 2 (tools/tofr.cpp:460-467).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from dataclasses import replace

import numpy as np

from . import _ffi as F
from . import harness as Hn
from .api import GateSpec, RenderConfig, Renderer, Scene, TofrError


def _add_render_options(p: argparse.ArgumentParser) -> None:  # tools/tofr.cpp:46-86
    p.add_argument("--scene", required=True)
    p.add_argument("--out", default="out")
    p.add_argument("--mode", default="gated", choices=["gated", "transient", "doppler"])
    p.add_argument("--tau", type=float, default=10.0)
    p.add_argument("--dtau", type=float, default=0.1)
    p.add_argument("--dtau-rel", type=float, default=-1)
    p.add_argument("--nu", type=float, default=0.0)
    p.add_argument("--dnu", type=float, default=1.0)
    p.add_argument("--f0", type=float, default=1.0)
    p.add_argument("--bins", type=int, default=16)
    p.add_argument("--hist-t0", type=float, default=-1)
    p.add_argument("--hist-width", type=float, default=-1)
    p.add_argument("--candidates", type=int, default=8)
    p.add_argument("--init", default="direct", choices=["direct", "ellipsoidal", "shrink"])
    p.add_argument("--K", type=float, default=10)
    p.add_argument("--R-frac", type=float, default=1.0)
    p.add_argument("--spatial", type=int, default=0)
    p.add_argument("--neighbors", type=int, default=5)
    p.add_argument("--radius", type=float, default=10)
    p.add_argument("--temporal", action="store_true")
    p.add_argument("--bin-reuse", action="store_true")
    p.add_argument("--mcap", type=float, default=20)
    p.add_argument("--gauge", default="avg", choices=["avg", "fixed", "raw"])
    p.add_argument("--naive", action="store_true")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--frames", type=int, default=1)
    p.add_argument("--frame0", type=float, default=0)
    p.add_argument("--gate-step", type=float, default=0)
    p.add_argument("--max-depth", type=int, default=6)
    p.add_argument("--no-rr", action="store_true")
    p.add_argument("--accumulate", action="store_true")
    p.add_argument("--normalize", action="store_true")
    p.add_argument("--threads", type=int, default=0, help="accepted for compatibility (GPU)")
    p.add_argument("--dump-reservoirs", action="store_true", help="accepted for compatibility (not written)")
    p.add_argument("--device", type=int, default=0, help="CUDA device")


def make_config(a, scene: Scene) -> RenderConfig:  # tools/tofr.cpp:88-135
    mode = {"gated": F.MODE_GATED, "transient": F.MODE_TRANSIENT, "doppler": F.MODE_GATED}[a.mode]
    vel = a.mode == "doppler"
    gate = GateSpec(F.GATE_VELOCITY if vel else F.GATE_LENGTH, a.nu if vel else a.tau, a.dnu if vel else a.dtau,
                    a.f0)
    if a.dtau_rel >= 0 and not vel:
        _, _, _, diag = scene.dump_bvh(a.frame0)
        gate.width = a.dtau_rel / 100.0 * diag
    seed = a.seed
    if os.environ.get("TOF_SEED"):
        seed = int(os.environ["TOF_SEED"])
    return RenderConfig(
        mode=mode, gate=gate, gate_step=a.gate_step, bins=a.bins,
        hist_t0=a.hist_t0 if a.hist_t0 >= 0 else a.tau - gate.width / 2,
        hist_bin_width=a.hist_width if a.hist_width > 0 else gate.width / a.bins,
        m_init=a.candidates,
        init={"direct": F.INIT_DIRECT, "ellipsoidal": F.INIT_ELLIPSOIDAL, "shrink": F.INIT_SHRINK}[a.init],
        shrink_k=a.K, shrink_r=a.R_frac, spatial_passes=a.spatial, spatial_neighbors=a.neighbors,
        spatial_radius=a.radius, temporal=a.temporal, bin_reuse=a.bin_reuse, m_cap=a.mcap,
        gauge={"avg": F.GAUGE_AVG, "fixed": F.GAUGE_FIXED, "raw": F.GAUGE_RAW}[a.gauge], newton=not a.naive,
        seed=seed, frames=a.frames, frame0=a.frame0, max_depth=a.max_depth, use_rr=not a.no_rr,
        accumulate=a.accumulate, normalize_gate=a.normalize)


def config_json(c: RenderConfig, doppler: bool) -> dict:  # tools/tofr.cpp:137-171
    return {
        "mode": "doppler" if doppler else ("transient" if c.mode == F.MODE_TRANSIENT else "gated"),
        "gate": {"kind": "velocity" if c.gate.kind == F.GATE_VELOCITY else "length", "center": c.gate.center,
                 "width": c.gate.width, "f0": c.gate.f0, "step": c.gate_step},
        "bins": c.bins, "hist_t0": c.hist_t0, "hist_bin_width": c.hist_bin_width, "candidates": c.m_init,
        "init": {F.INIT_DIRECT: "direct", F.INIT_ELLIPSOIDAL: "ellipsoidal", F.INIT_SHRINK: "shrink"}[c.init],
        "shrink_k": c.shrink_k, "shrink_r": c.shrink_r, "spatial_passes": c.spatial_passes,
        "spatial_neighbors": c.spatial_neighbors, "spatial_radius": c.spatial_radius, "temporal": c.temporal,
        "bin_reuse": c.bin_reuse, "m_cap": c.m_cap,
        "gauge": {F.GAUGE_AVG: "avg", F.GAUGE_FIXED: "fixed", F.GAUGE_RAW: "raw"}[c.gauge], "newton": c.newton,
        "seed": c.seed, "frames": c.frames, "frame0": c.frame0, "max_depth": c.max_depth, "use_rr": c.use_rr,
        "accumulate": c.accumulate, "normalize_gate": c.normalize_gate, "device": "b200",
    }


def _render(r: Renderer, scene: Scene, cfg: RenderConfig):
    if cfg.mode == F.MODE_TRANSIENT:
        return r.render_transient(scene, cfg)
    if cfg.gate.kind == F.GATE_VELOCITY:
        return r.render_doppler(scene, cfg)
    return r.render_gated(scene, cfg)


def cmd_render(a) -> int:  # tools/tofr.cpp:186-244
    scene = Scene.create(a.scene)
    cfg = make_config(a, scene)
    r = Renderer(a.device)
    t0 = time.perf_counter()
    out = _render(r, scene, cfg)
    seconds = time.perf_counter() - t0
    manifest = {"scene": a.scene, "scene_hash": Hn.hash_file(a.scene), "config": config_json(cfg, a.mode == "doppler"),
                "seconds": seconds, "outputs": []}

    def record(path):
        manifest["outputs"].append({"path": path, "fnv64": Hn.hash_file(path)})

    img_path = a.out + ".pfm"
    Hn.write_pfm(out.image, img_path)
    record(img_path)
    txt_path = a.out + ".txt"
    Hn.write_text_matrix(out.image, txt_path)
    record(txt_path)
    if cfg.mode == F.MODE_TRANSIENT:
        csv = a.out + "_hist.csv"
        Hn.write_histogram_csv(out.hist, csv)
        record(csv)
    stats_path = a.out + "_stats.txt"
    with open(stats_path, "w") as f:
        f.write(Hn.stats_lines(out.stats))
    record(stats_path)
    with open(a.out + "_manifest.json", "w") as f:
        f.write(json.dumps(manifest, indent=2) + "\n")
    print(f"wrote {img_path} (mean {Hn.image_mean(out.image):.6g}, {seconds:.6g} s)")
    return 0


def cmd_reference(a) -> int:  # tools/tofr.cpp:246-276
    scene = Scene.create(a.scene)
    cfg = make_config(a, scene)
    if cfg.gate.kind != F.GATE_LENGTH:
        raise TofrError(F.TOFR_ERR_UNSUPPORTED, "reference: the device reference renders length gates")
    r = Renderer(a.device)
    t0 = time.perf_counter()
    mean, se = r.reference_render(scene, cfg.frame0, cfg.gate, a.spp, cfg.seed, cfg.max_depth)
    seconds = time.perf_counter() - t0
    if cfg.normalize_gate and cfg.gate.width > 0:
        mean = mean * (1.0 / cfg.gate.width)
        se = se * (1.0 / cfg.gate.width)
    Hn.write_pfm(mean, a.out + ".pfm")
    Hn.write_pfm(se, a.out + "_se.pfm")
    Hn.write_text_matrix(mean, a.out + ".txt")
    manifest = {"scene": a.scene, "scene_hash": Hn.hash_file(a.scene), "config": config_json(cfg, False),
                "spp": a.spp, "seconds": seconds,
                "outputs": [{"path": a.out + ".pfm", "fnv64": Hn.hash_file(a.out + ".pfm")}]}
    with open(a.out + "_manifest.json", "w") as f:
        f.write(json.dumps(manifest, indent=2) + "\n")
    print(f"wrote {a.out}.pfm (mean {Hn.image_mean(mean):.6g}, {seconds:.6g} s)")
    return 0


def cmd_compare(a) -> int:  # tools/tofr.cpp:278-300
    est = Hn.read_pfm(a.est)
    ref = Hn.read_pfm(a.ref)
    if est.shape != ref.shape:
        print(f"error: image dimensions differ ({est.shape[1]}x{est.shape[0]} vs {ref.shape[1]}x{ref.shape[0]})",
              file=sys.stderr)
        return 2
    m = Hn.compute_metrics(est, ref)
    print(f"MAPE={m.mape:.6g} relMSE={m.relmse:.6g}")
    if a.stats:
        with open(a.stats) as f:
            sys.stdout.write(f.read())
    return 0


def cmd_stats(a) -> int:  # tools/tofr.cpp:302-337
    agg: dict = {}
    rows: dict = {}
    with open(a.file) as f:
        for line in f:
            stage, kv = None, []
            for tok in line.split():
                if "=" not in tok:
                    continue
                k, v = tok.split("=", 1)
                if k == "stage":
                    stage = v
                else:
                    try:
                        kv.append((k, float(v)))
                    except ValueError:
                        kv.append((k, 0.0))
            if not stage:
                continue
            d = agg.setdefault(stage, {})
            for k, v in kv:
                d[k] = d.get(k, 0.0) + v
            rows[stage] = rows.get(stage, 0) + 1
    for stage in sorted(agg):
        parts = []
        for k in sorted(agg[stage]):
            if k == "frame":
                continue
            v = agg[stage][k]
            if k in ("mean_iterations", "newton_sr", "actual_sr"):
                v /= rows[stage]
            parts.append(f"{k}={v:.6g}")
        print(f"{stage}: " + " ".join(parts))
    return 0


def cmd_sweep(a) -> int:  # tools/tofr.cpp:339-412 (equal-time harness on the device)
    scene = Scene.create(a.scene)
    base = make_config(a, scene)
    r = Renderer(a.device)
    _, _, _, diag = scene.dump_bvh(base.frame0)
    values = a.values or {"gatewidth": [0.5, 2.5, 10, 50], "kr": [1, 10, 100, 500],
                          "bins": [4, 8, 16, 32, 64]}[a.type]
    lines = []
    if a.type == "gatewidth":
        lines.append("dtau_frac,dtau,mape_ours,mape_naive,sr_ours,sr_naive")
        for frac in values:
            cfg = replace(base, gate=replace(base.gate, width=frac / 100.0 * diag))
            ref, _ = r.reference_render(scene, cfg.frame0, cfg.gate, a.ref_spp, base.seed + 17, cfg.max_depth)
            ro = Hn.render_equal_time(r, scene, replace(cfg, newton=True), a.budget)
            rn = Hn.render_equal_time(r, scene, replace(cfg, newton=False), a.budget)
            lines.append(f"{frac:.8g},{cfg.gate.width:.8g},{Hn.compute_metrics(ro.image, ref).mape:.8g},"
                         f"{Hn.compute_metrics(rn.image, ref).mape:.8g},{Hn.actual_sr(ro.spatial):.8g},"
                         f"{Hn.actual_sr(rn.spatial):.8g}")
    elif a.type == "kr":
        lines.append("K,R,mape,mean_ratio")
        ref, _ = r.reference_render(scene, base.frame0, base.gate, a.ref_spp, base.seed + 17, base.max_depth)
        ref_mean = Hn.image_mean(ref)
        for K in values:
            for R in (0.0, 0.5, 1.0):
                cfg = replace(base, init=F.INIT_SHRINK, shrink_k=K, shrink_r=R)
                res = Hn.render_equal_time(r, scene, cfg, a.budget)
                ratio = Hn.image_mean(res.image) / ref_mean if ref_mean > 0 else 0
                lines.append(f"{K:.8g},{R:.8g},{Hn.compute_metrics(res.image, ref).mape:.8g},{ratio:.8g}")
    else:
        lines.append("B,seconds_reuse,seconds_trace")
        for bd in values:
            B = int(bd)
            cfg = replace(base, mode=F.MODE_TRANSIENT, bins=B, temporal=True, bin_reuse=True,
                          frames=max(2, base.frames))
            t0 = time.perf_counter()
            r.render_transient(scene, cfg)
            t_reuse = time.perf_counter() - t0
            t0 = time.perf_counter()
            r.render_transient_plain(scene, cfg)
            t_trace = time.perf_counter() - t0
            lines.append(f"{B},{t_reuse:.8g},{t_trace:.8g}")
    with open(a.out + ".csv", "w") as f:
        f.write("\n".join(lines) + "\n")
    print(f"wrote {a.out}.csv")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="tofr", description="time-gated / transient / Doppler Monte Carlo renderer "
                                                          "with reservoir-based path reuse (B200)")
    sub = ap.add_subparsers(dest="verb", required=True)
    p = sub.add_parser("render", help="render with reservoir path reuse")
    _add_render_options(p)
    p = sub.add_parser("reference", help="brute-force gated reference with a stderr image")
    _add_render_options(p)
    p.add_argument("--spp", type=int, default=1024)
    p = sub.add_parser("compare", help="MAPE/relMSE between two PFM images")
    p.add_argument("--est", required=True)
    p.add_argument("--ref", required=True)
    p.add_argument("--stats", default="")
    p = sub.add_parser("stats", help="aggregate a per-frame stats file")
    p.add_argument("--file", required=True)
    p = sub.add_parser("sweep", help="gate-width / K-R / bin-count sweeps (CSV)")
    _add_render_options(p)
    p.add_argument("--type", default="gatewidth", choices=["gatewidth", "kr", "bins"])
    p.add_argument("--budget", type=float, default=2.0)
    p.add_argument("--values", type=float, nargs="*", default=None)
    p.add_argument("--ref-spp", type=int, default=2048)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    try:
        return {"render": cmd_render, "reference": cmd_reference, "compare": cmd_compare, "stats": cmd_stats,
                "sweep": cmd_sweep}[a.verb](a)
    except TofrError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except (OSError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
