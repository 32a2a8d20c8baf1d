#!/usr/bin/env python
"""bench.py -- frames/s and Mpaths/s of the B200 ToF ReSTIR frame pipeline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c3]

A step is one frame of the interactive pipeline (render_gated's frame loop,
pipeline.hpp:323-392): host build_frame + snapshot upload, G-buffer, initial
RIS, temporal reuse, spatial reuse, final shading.  The default workload is
BASELINE.json configs[2] ("C3"): the largest bundled scene (boxes_doppler,
24 triangles, animated -> BVH rebuilt every frame) at 1920x1080, time-gated
with a narrow gate (tau 12.0, dtau 0.041 = 0.5% of the scene diagonal),
m_init 1, temporal + 1x3 spatial reuse of radius 10.

Our arm prints one JSON line with the device-timed `value` (CUDA events on
the library stream, max over ranks), `e2e` (the same frames through the
public Session API, each step also reading the image back to pinned host
memory), the `roofline` of the dominant kernel, `cpu_baseline` (the reference
CPU renderer, oracle/_ref, timed on this host) and the clocks seen.
`--impl reference` times the unmodified reference CPU renderer (oracle/_ref,
built from /root/reference/proj/include) on the same workload.

Multi-GPU (torchrun): the frame is split into row bands, one per rank, and
the spatial-reuse halo rows are exchanged with NCCL (parallel.py).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_2605_11536_b200 import _ffi as F  # noqa: E402
from paper_2605_11536_b200 import scenes  # noqa: E402
from paper_2605_11536_b200.api import GateSpec, RenderConfig  # noqa: E402

METRIC = "frames/sec and Mpaths/s at 1080p (time-gated & transient), 1/2/4/8 B200"


def _gate(c, w):
    return GateSpec(F.GATE_LENGTH, c, w, 1.0)


# name -> (scene, width, height, RenderConfig(frames ignored), description)
WORKLOADS = {
    "c3": ("boxes_doppler", 1920, 1080,
           RenderConfig(gate=_gate(12.0, 0.041), m_init=1, temporal=True, spatial_passes=1, spatial_neighbors=3,
                        spatial_radius=10, m_cap=20, max_depth=6, seed=1),
           "C3: boxes_doppler 1920x1080 gated tau=12.0 dtau=0.041, m_init 1, temporal + 1x3 spatial r10"),
    "c3d": ("boxes_doppler", 1920, 1080,
            RenderConfig(gate=GateSpec(F.GATE_VELOCITY, -0.09, 0.04, 1.0), m_init=1, temporal=True, spatial_passes=1,
                         spatial_neighbors=3, spatial_radius=10, m_cap=20, max_depth=6, seed=1),
            "C3 Doppler: boxes_doppler 1920x1080 velocity gate -0.09 +- 0.02 Hz (f0 1 Hz: receding box), m_init 1, "
            "temporal + 1x3 spatial r10 (render_doppler)"),
    "c3w": ("cornell_wide", 1920, 1080,
            RenderConfig(gate=_gate(6.0, 0.0173), m_init=1, temporal=True, spatial_passes=1, spatial_neighbors=3,
                         spatial_radius=10, m_cap=20, max_depth=6, seed=1),
            "C3': cornell_wide 1920x1080 gated tau=6.0 dtau=0.0173, m_init 1, temporal + 1x3 spatial r10"),
    # the paper's shrink initialisation (wide-gate RIS, shrink_map to the fine
    # gate) on C3' (per-item init kernel, k_init_gated)
    "c3w_shrink": ("cornell_wide", 1920, 1080,
                   RenderConfig(gate=_gate(6.0, 0.0173), m_init=1, init=F.INIT_SHRINK, shrink_k=10.0, shrink_r=1.0,
                                temporal=True, spatial_passes=1, spatial_neighbors=3, spatial_radius=10, m_cap=20,
                                max_depth=6, seed=1),
                   "C3' with shrink initialisation (K 10, R 1): cornell_wide 1920x1080 gated tau=6.0 dtau=0.0173, "
                   "temporal + 1x3 spatial r10"),
    "c5": ("cornell_wide", 1920, 1080,
           RenderConfig(gate=_gate(6.0, 0.0173), gate_step=0.01, m_init=1, temporal=True, spatial_passes=1,
                        spatial_neighbors=3, spatial_radius=10, m_cap=20, max_depth=6, seed=1),
           "C5: cornell_wide 1920x1080 gate sweep 0.01/frame, temporal + 1x3 spatial r10"),
    "c1": ("cornell", 256, 256,
           RenderConfig(gate=_gate(10.0, 0.0866), m_init=1, temporal=True, spatial_passes=1, spatial_neighbors=3,
                        spatial_radius=10, m_cap=20, max_depth=6, seed=1),
           "C1: cornell 256x256 gated tau=10.0 dtau=0.0866, m_init 1, temporal + 1x3 spatial r10"),
    "c2p": ("cornell", 512, 512,
            RenderConfig(mode=F.MODE_TRANSIENT, bins=256, hist_t0=8.0, hist_bin_width=0.046875, m_init=1,
                         max_depth=6, seed=1),
            "C2(i): cornell 512x512 transient 256 bins [8,20), render_transient_plain (trace + histogram deposits)"),
    "c2r": ("cornell", 512, 512,
            RenderConfig(mode=F.MODE_TRANSIENT, bins=256, hist_t0=8.0, hist_bin_width=0.046875, m_init=1,
                         temporal=True, m_cap=20, max_depth=6, seed=1),
            "C2(ii): cornell 512x512 transient 256 bins [8,20), render_transient reservoirs, temporal reuse"),
    # C2(ii) with the optional +-1 bin reuse stage (pipeline.hpp:273-299; per-item
    # kernel k_binreuse)
    "c2r_bin": ("cornell", 512, 512,
                RenderConfig(mode=F.MODE_TRANSIENT, bins=256, hist_t0=8.0, hist_bin_width=0.046875, m_init=1,
                             temporal=True, bin_reuse=True, m_cap=20, max_depth=6, seed=1),
                "C2(ii) + bin reuse: cornell 512x512 transient 256 bins [8,20), render_transient reservoirs, "
                "temporal reuse then +-1 bin reuse"),
    "c4p": ("boxes_doppler", 1920, 1080,
            RenderConfig(mode=F.MODE_TRANSIENT, bins=1024, hist_t0=7.0, hist_bin_width=0.01953125, m_init=1,
                         max_depth=8, seed=1),
            "C4 (plain): boxes_doppler 1920x1080 transient 1024 bins [7,27), depth 8, trace + histogram deposits"),
    "c4r": ("boxes_doppler", 1920, 1080,
            RenderConfig(mode=F.MODE_TRANSIENT, bins=1024, hist_t0=7.0, hist_bin_width=0.01953125, m_init=1,
                         max_depth=8, temporal=True, spatial_passes=1, spatial_neighbors=3, spatial_radius=10,
                         m_cap=20, seed=1),
            "C4 (reservoirs): boxes_doppler 1920x1080 transient 1024 bins [7,27), depth 8, render_transient "
            "temporal + 1x3 spatial r10 per bin, row bands with reservoir halo exchange"),
    # transient ReSTIR at 1080p on one GPU, the paper's transient setting (temporal
    # reuse only) on the C2 scene and bin range
    "t1080": ("cornell", 1920, 1080,
              RenderConfig(mode=F.MODE_TRANSIENT, bins=256, hist_t0=8.0, hist_bin_width=0.046875, m_init=1,
                           temporal=True, m_cap=20, max_depth=6, seed=1),
              "transient 1080p: cornell 1920x1080, 256 bins [8,20), render_transient reservoirs, temporal reuse "
              "only (the paper's transient setting)"),
    "t1080b64": ("cornell", 1920, 1080,
                 RenderConfig(mode=F.MODE_TRANSIENT, bins=64, hist_t0=8.0, hist_bin_width=0.1875, m_init=1,
                              temporal=True, m_cap=20, max_depth=6, seed=1),
                 "transient 1080p: cornell 1920x1080, 64 bins [8,20), render_transient reservoirs, temporal reuse "
                 "only (the paper's transient setting)"),
    # the paper's gated timing (256x256 NLOS scan, ellipsoidal
    # initial sampling + temporal + spatial reuse, 4 ms/image on an RTX 3090),
    # on the bundled wide-light scene with a narrow gate
    "nlos": ("cornell_wide", 256, 256,
             RenderConfig(gate=_gate(6.0, 0.01), m_init=1, init=F.INIT_ELLIPSOIDAL, temporal=True, spatial_passes=1,
                          spatial_neighbors=3, spatial_radius=10, m_cap=20, max_depth=6, seed=1),
             "NLOS-style gated: cornell_wide 256x256, gate tau=6.0 dtau=0.01, ellipsoidal initial sampling + "
             "temporal + 1x3 spatial r10 (paper: 4 ms/image on an RTX 3090)"),
    # an NLOS scan: SCAN_POINTS independent 256^2 images (gate positions 6.0 + 0.05 k,
    # each its own session and stream) in flight at once; value = images/s
    "nlos_scan": ("cornell_wide", 256, 256,
                  RenderConfig(gate=_gate(6.0, 0.01), m_init=1, init=F.INIT_ELLIPSOIDAL, temporal=True,
                               spatial_passes=1, spatial_neighbors=3, spatial_radius=10, m_cap=20, max_depth=6,
                               seed=1),
                  "NLOS scan: 8 scan points (gates tau = 6.0 + 0.05 k, dtau 0.01) of cornell_wide 256x256 "
                  "rendered concurrently (one session / stream each), ellipsoidal init + temporal + 1x3 spatial "
                  "r10; frames/s = images/s over all scan points"),
    # BVH stress: cornell_wide's box + a 102,410-triangle displaced torus (64,875
    # nodes, traversed from global memory), C3' gate and reuse
    "mesh": ("mesh", 1920, 1080,
             RenderConfig(gate=_gate(6.0, 0.0173), m_init=1, temporal=True, spatial_passes=1, spatial_neighbors=3,
                          spatial_radius=10, m_cap=20, max_depth=6, seed=1),
             "mesh: cornell_wide box + 102,410-triangle torus (BVH in global memory) 1920x1080 gated tau=6.0 "
             "dtau=0.0173, m_init 1, temporal + 1x3 spatial r10"),
    "mesh_anim": ("mesh_anim", 1920, 1080,
                  RenderConfig(gate=_gate(6.0, 0.0173), m_init=1, temporal=True, spatial_passes=1,
                               spatial_neighbors=3, spatial_radius=10, m_cap=20, max_depth=6, seed=1),
                  "mesh (animated): the 102,410-triangle torus turning and drifting -- a new BVH every frame, "
                  "built on the device -- 1920x1080 gated tau=6.0 dtau=0.0173, temporal + 1x3 spatial r10"),
}

PLAIN = {"c2p", "c4p"}
# workloads that do not fit one GPU whole: at N = 1 one GPU renders the band of
# rank EMULATE_RANK of an EMULATE_WORLD-way split (per-GPU share of that job;
# its halo rows arrive empty, no transfer), labelled in `config`
BAND_ONLY = {"c4r": (8, 4)}  # render_transient_plain workloads; the others are ReSTIR sessions

# Algorithmic HBM bytes per unit of work of each kernel (
# R = 224 B compact reservoir).  Units are counted on the device
# (shift jobs, pixels, reservoir items) or known from the launch (pixels).
R_BYTES = 224
GHIT_BYTES = 16
KERNEL_BYTES = {
    # shift jobs: job record (64 B) + the source record's geometry (112 B) + hand-off (48 B)
    "k_shift_solve": ("job", 64 + 112 + 48),
    # job + hand-off (112 B) + source record R + mapped record R (forward shifts; inverse: 16 B)
    "k_shift_finish": ("job", 112 + 2 * R_BYTES),
    "k_shift_replay": ("job", 64 + 16),
    # path trees: G-buffer read + reservoir write
    "k_trace_gated": ("pixel", GHIT_BYTES + R_BYTES),
    "k_init_gated": ("pixel", GHIT_BYTES + R_BYTES),
    # transient RIS: G-buffer read + per-bin (w_sum, M) read-modify-write on deposits (counted as 1 bin/pixel)
    "k_trace_bins": ("pixel", GHIT_BYTES + 32 + R_BYTES),
    # plain deposits: 32 B rgb+count read-modify-write per deposit (deposits/pixel measured)
    "k_hist_plain": ("deposit", 32),
    "k_trace_plain": ("deposit", 32),
    "k_ris_finalize": ("item", 32),
    # merge stages: header reads of both sides + header write per item
    "k_temporal_prep": ("item", 16 + 16 + 16),
    "k_temporal_apply": ("merge", 3 * R_BYTES),
    "k_spatial_prep_fwd": ("item", 16),
    "k_spatial_prep_inv": ("item", 16 + 16),
    "k_spatial_apply": ("merge", 3 * R_BYTES),
    # per-item +-1 bin reuse: the three headers (own, b-1, b+1) + the output record
    "k_binreuse": ("item", 3 * 16 + R_BYTES),
    "k_shade_gated": ("pixel", 24 + 12 + 24),
    "k_shade_transient": ("item", 16 + 24),
    "k_gbuffer": ("pixel", GHIT_BYTES),
}


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured"}
    return {"hbm_gbs": 6650.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        # started before the warm-up (nvidia-smi needs ~0.1-0.3 s to produce its
        # first line); only the samples inside mark()..stop() are kept
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.t0 = None
        q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "20"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def mark(self) -> None:
        """Start of the timed region."""
        self.t0 = time.time()

    def wait_ready(self) -> None:
        """Wait (up to 3 s) for nvidia-smi's first line, so that even a short
        timed region is sampled (call before the ranks' barrier)."""
        t_end = time.time() + 3.0
        while self.p is not None and time.time() < t_end:
            try:
                if os.path.getsize(self.f.name) > 0:
                    break
            except OSError:
                break
            time.sleep(0.02)

    def stop(self) -> dict:
        import datetime
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t1 = time.time()
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            try:
                ts = datetime.datetime.strptime(r[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                if self.t0 is not None and not (self.t0 <= ts <= t1):
                    continue
                sm.append(float(r[1]))
                mx = float(r[2])
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
               "samples": len(sm)}
        if not sm and rows:  # unparsable timestamps: every sample of the run
            self.t0 = None
            raw = [x for x in rows if len(x) > 2]
            vals = [float(x[1]) for x in raw if x[1].strip().replace(".", "", 1).isdigit()]
            out.update({"sm_mhz": statistics.median(vals) if vals else None, "samples": len(vals),
                        "window": "whole run (timestamps unparsable)"})
        return out


def kernel_profile(workload: str, kernel: str | None):
    """profiles/kernel_profile.json entry of (workload, kernel), or None."""
    p = ROOT / "profiles" / "kernel_profile.json"
    if not kernel or not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(f"{workload}:{kernel}")
    except Exception:
        return None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# reference arm / cpu baseline: the unmodified reference CPU renderer


def cpu_reference_sample(wl: str, frames: int = 2) -> dict:
    """The reference's own driver (oracle/_ref) with all host threads on the
    full workload, `frames` frames (gated: frame 0 init + spatial, frame 1 adds
    the temporal stage).  Returns seconds and the thread count."""
    from oracle import ref as R
    scene_name, w, h, cfg, _ = WORKLOADS[wl]
    cores = os.cpu_count() or 1
    R.set_threads(cores)
    sd = scenes.bundled(scene_name, w, h)
    # render_transient's 624 B reservoirs per pixel-bin do not fit host RAM at the
    # workload's size (512^2 x 256 bins: 84 GB per grid pair): time a 128-pixel-wide
    # image of the same aspect and scale by the pixel count (labelled in `sample`)
    scaled = cfg.mode == F.MODE_TRANSIENT and wl not in PLAIN
    sw, sh = (128, max(1, round(128 * h / w))) if scaled else (w, h)
    if scaled:
        sd = scenes.bundled(scene_name, sw, sh)
    rs = R.RefScene(sd)
    c = RenderConfig(**{**cfg.__dict__})
    c.frames = frames
    fn = R.render_transient_plain if wl in PLAIN else (R.render_transient if cfg.mode == F.MODE_TRANSIENT
                                                        else R.render_gated)
    t0 = time.perf_counter()
    fn(rs, c)
    dt = time.perf_counter() - t0
    if scaled:
        dt *= (w * h) / (sw * sh)  # extrapolated to the full image (labelled in the sample text)
    drv = "render_transient_plain" if wl in PLAIN else ("render_transient" if cfg.mode == F.MODE_TRANSIENT
                                                         else "render_gated")
    what = (f"{drv}(frames={frames}) at {sw}x{sh}, time scaled x{(w * h) / (sw * sh):.0f} to {w}x{h}" if scaled
            else f"{drv}(frames={frames}) of the full {w}x{h} workload")
    return {"seconds": dt, "frames": frames, "cores": R.threads(), "pixels": w * h, "what": what}


def run_reference(args) -> None:
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    scene_name, w, h, cfg, desc = WORKLOADS[args.workload]
    if args.workload in BAND_ONLY:
        print(json.dumps({"impl": "reference", "unavailable": "the reference's render_transient needs 1.3 TB of "
                                                               "reservoirs per grid at this size (SURVEY 8d)"}))
        return
    for _ in range(args.warmup):
        cpu_reference_sample(args.workload, 1)
    secs, frames, cores = 0.0, 0, 1
    for _ in range(args.steps):
        r = cpu_reference_sample(args.workload, 2)
        secs += r["seconds"]
        frames += r["frames"]
        cores = r["cores"]
    fps = frames / secs
    sample = f"{args.steps} x {r['what']} (frame 0 has no temporal stage)"
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / frames,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "resolution": f"{w}x{h}", "scene": scene_name},
        "mpaths_per_s": w * h * cfg.m_init * fps / 1e6,
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm


SCAN_POINTS = 8


def run_scan(args) -> None:
    """nlos_scan: SCAN_POINTS independent sessions (scan points) stepped round
    robin, each on its own library context / stream, so one point's serial
    shift tails overlap the others' work (independent units shard trivially,
    SURVEY 8e).  Device time = first start event .. last end event."""
    import torch
    from paper_2605_11536_b200.api import Renderer
    scene_name, w, h, cfg, desc = WORKLOADS[args.workload]
    sd = scenes.bundled(scene_name, w, h)
    rs = [Renderer(0) for _ in range(SCAN_POINTS)]
    cfgs = []
    for k in range(SCAN_POINTS):
        c = RenderConfig(**{**cfg.__dict__})
        c.gate = GateSpec(cfg.gate.kind, cfg.gate.center + 0.05 * k, cfg.gate.width, cfg.gate.f0)
        cfgs.append(c)
    warm = max(args.warmup, cfg.m_cap + 5)

    def sessions():
        return [rs[k].session(sd, cfgs[k]) for k in range(SCAN_POINTS)]

    ss = sessions()
    streams = [torch.cuda.ExternalStream(s.stream_ptr()) for s in ss]
    clk = ClockSampler(0)
    for _ in range(warm):
        for s in ss:
            s.step(stats=False)
    for s in ss:
        s.sync()
    clk.wait_ready()
    clk.mark()
    starts = [torch.cuda.Event(enable_timing=True) for _ in ss]
    ends = [torch.cuda.Event(enable_timing=True) for _ in ss]
    for e, st in zip(starts, streams):
        e.record(st)
    l0 = F.kernel_launches()
    for _ in range(args.steps):
        for s in ss:
            s.step(stats=False)
    for e, st in zip(ends, streams):
        e.record(st)
    for e in ends:
        e.synchronize()
    launches = F.kernel_launches() - l0
    t_ms = max(starts[0].elapsed_time(e) for e in ends)
    t_ms = max(t_ms, max(sa.elapsed_time(e) for sa in starts for e in ends))
    clocks = clk.stop()
    images = args.steps * SCAN_POINTS
    # e2e: fresh sessions, every image read back to pinned host memory
    for s in ss:
        s.close()
    ss = sessions()
    bufs = [[torch.empty((h, w, 3), dtype=torch.float64, pin_memory=True).numpy() for _ in range(2)] for _ in ss]
    for _ in range(warm):
        for s in ss:
            s.step(stats=False)
    for s in ss:
        s.sync()
    t0 = time.perf_counter()
    for f in range(args.steps):
        for k, s in enumerate(ss):
            s.step(stats=False)
            if f >= 2:
                s.wait_read(f & 1)
            s.read_image_async(bufs[k][f & 1], f & 1)
    for k, s in enumerate(ss):
        for f in range(max(0, args.steps - 2), args.steps):
            s.wait_read(f & 1)
    e2e_s = time.perf_counter() - t0
    line = {
        "metric": METRIC, "value": images / (t_ms * 1e-3), "unit": "frames/s", "n_gpus": 1, "steps": args.steps,
        "warmup": warm, "warmup_requested": args.warmup, "ms_per_step": t_ms / args.steps,
        "ms_per_image": t_ms / images, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "scene": scene_name, "resolution": f"{w}x{h}", "scan_points": SCAN_POINTS,
                   "parallelism": "single GPU, one stream per scan point"},
        "e2e": {"value": images / e2e_s, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": SCAN_POINTS * w * h * 24},
        "gpu_launches": launches, "clocks": clocks,
        "note": "a step renders one frame of every scan point; value = images/s; paper: 4 ms/image on an RTX 3090",
    }
    print(json.dumps(line), flush=True)


def run_ours(args) -> None:
    import torch
    ws, rank, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the product path has no CPU fallback)")
    # TOFR_DIST_BACKEND=gloo: host-staged halo transport, several ranks may
    # share one GPU (plumbing test of the N > 1 path on a one-GPU box)
    backend = os.environ.get("TOFR_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    from paper_2605_11536_b200 import parallel
    from paper_2605_11536_b200.api import Renderer

    group = None
    if ws > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD
    scene_name, w, h, cfg, desc = WORKLOADS[args.workload]
    plain = args.workload in PLAIN
    sd = scenes.bundled(scene_name, w, h)
    r = Renderer(local)
    emulated = BAND_ONLY[args.workload] if (ws == 1 and args.workload in BAND_ONLY) else None
    # N > 1: the row split is refined from measured band times (the shift work
    # of a frame is far from even over the rows: C3's bottom eighth holds half
    # of it).  Each refinement renders a few frames on the current split, takes
    # every rank's device time, and re-cuts the rows at equal measured cost
    # (parallel.rebalance_bands; TOFR_BALANCE=0: equal rows).  Emulated on one
    # GPU (tools/band_probe3.py) two steps take C3 at 8 bands from 2.8x to 3.0x
    # of one GPU; what remains is each batch's serial Newton-chain floor.
    bands = None
    if ws > 1 and args.workload not in BAND_ONLY and os.environ.get("TOFR_BALANCE", "1") != "0":
        bands = [parallel.band_rows(h, ws, g) for g in range(ws)]
        halo = (parallel.halo_rows(cfg.spatial_radius, cfg.spatial_passes, parallel.motion_rows_for(sd, cfg))
                if not plain else 0)
        for _ in range(2):
            probe = parallel.BandSession(r, sd, cfg, rank=rank, world=ws, group=group, plain=plain, bands=bands)
            for _ in range(3):
                probe.step()
            probe.sync()
            parallel.barrier(group)
            t_band = probe.timed_steps(5, [0.0] * 6)
            times = parallel.gather_floats_all([t_band], group)
            probe.sess.close()
            del probe
            bands = parallel.rebalance_bands(bands, times, max(1, halo))

    def new_session():
        if emulated:
            return parallel.BandSession(r, sd, cfg, rank=emulated[1], world=emulated[0], group=None, plain=plain,
                                        emulate=True)
        return parallel.BandSession(r, sd, cfg, rank=rank, world=ws, group=group, plain=plain, bands=bands)

    # steady state: a ReSTIR frame's cost depends on the reservoirs' confidence
    # M, which saturates at m_cap after m_cap frames of temporal reuse, so the
    # warm-up runs at least m_cap + 5 frames (frame_ms_curve shows the ramp)
    warm = args.warmup
    if cfg.temporal and not plain:
        warm = max(warm, cfg.m_cap + 5)
    sess = new_session()
    clk = ClockSampler(local) if rank == 0 else None
    for _ in range(warm):
        sess.step()
    sess.sync()
    if clk:
        clk.wait_ready()
    parallel.barrier(group)

    # timed region (value): K frames between CUDA events on the session stream,
    # exact launch count and device work counters around it; no per-kernel
    # instrumentation (its events between launches cost ~10% of a gated frame)
    if clk:
        clk.mark()
    stage_tot = [0.0] * 6
    work0 = sess.work()
    l0 = F.kernel_launches()
    t_ms = sess.timed_steps(args.steps, stage_tot)
    launches = F.kernel_launches() - l0
    work1 = sess.work()
    t_max = parallel.max_over_ranks(t_ms, group)
    frames = args.steps
    fps = frames / (t_max * 1e-3)

    # shift counters of one more (synchronous) frame: the work behind the time
    st = sess.step(stats=True)
    if plain:
        st = {k: {n: 0 for n in ("attempts", "solves", "iterations", "newton_ok", "occluded", "success")}
              for k in ("temporal", "spatial")}
    shift_stats = {k: {n: st[k][n] for n in ("attempts", "solves", "iterations", "newton_ok", "occluded",
                                              "success")} for k in ("temporal", "spatial")}

    # per-frame latency (C5): frames stepped one at a time, device
    # time of each frame from its own events (submit -> last kernel)
    latency = None
    if args.latency_frames > 0:
        lat = []
        for _ in range(args.latency_frames):
            sess.step(stats=True)
            tot, _ = sess.sess.last_ms()
            lat.append(tot)
        lat_all = parallel.gather_floats(lat, group) if ws > 1 else lat
        latency = {"frames": len(lat), "p50_ms": float(np.percentile(lat_all, 50)),
                   "p99_ms": float(np.percentile(lat_all, 99)), "max_ms": float(np.max(lat_all))}

    pool_info = None
    if not plain and cfg.mode == F.MODE_TRANSIENT:
        p = sess.sess.pool()
        pool_info = {"rows_used_max": max(p["rows_used"]), "rows_cap": p["rows_cap"],
                     "rows_per_owned_item": max(p["rows_used"]) / max(1, sess.owned_pixels() * cfg.bins)}
    clocks = clk.stop() if clk else None  # the value frames and the stats / latency frames

    # per-kernel times and the roofline's launch durations / units: the same
    # frames (W warm-up, K timed) on a fresh session with every launch bracketed
    # by CUDA events, and one stream (pipelined frames overlap their kernels, so
    # an event pair would also time the wait for SM slots)
    sess.sess.close()
    pipe_env = os.environ.get("TOFR_PIPELINE")
    os.environ["TOFR_PIPELINE"] = "0"
    try:
        sess = new_session()
    finally:
        if pipe_env is None:
            os.environ.pop("TOFR_PIPELINE", None)
        else:
            os.environ["TOFR_PIPELINE"] = pipe_env
    for _ in range(warm):
        sess.step()
    sess.sync()
    parallel.barrier(group)
    F.kernel_times(reset=True)
    F.kernel_timing(True)
    work0k = sess.work()
    sess.timed_steps(args.steps, [0.0] * 6)
    work1k = sess.work()
    F.kernel_timing(False)
    ktimes = F.kernel_times(reset=True)
    sess.sess.close()

    # stage split and per-frame curve: the same frames on a fresh one-stream
    # session without kernel instrumentation, stepped one at a time, so the
    # stage events are sequential and sum to the frame (the pipelined value
    # frames overlap frame f+1's camera + initial sampling with frame f's reuse)
    os.environ["TOFR_PIPELINE"] = "0"
    try:
        sess = new_session()
    finally:
        if pipe_env is None:
            os.environ.pop("TOFR_PIPELINE", None)
        else:
            os.environ["TOFR_PIPELINE"] = pipe_env
    curve, stage_one = [], [0.0] * 6
    for fr in range(warm + args.steps):
        sess.step(stats=True)
        tot, st6 = sess.sess.last_ms()
        curve.append(round(tot, 4))
        if fr >= warm:
            stage_one = [a + b for a, b in zip(stage_one, st6)]

    # e2e through the public API: step + image read-back to pinned host memory,
    # on a fresh session over the same frames as the device-timed run (W warm-up
    # frames of the same loop, untimed, then K timed): transient reservoir grids
    # fill up frame by frame, so later frames cost more and would not compare
    band_px = sess.owned_pixels()
    sess.sess.close()
    sess = new_session()
    parallel.barrier(group)
    e2e_s = sess.run_e2e(args.steps, warm=warm)
    e2e_s = parallel.max_over_ranks(e2e_s * 1e3, group) * 1e-3
    h2d, d2h = sess.io_bytes()

    # roofline of the dominant kernel: algorithmic bytes per launch / average
    # launch duration (CUDA events on the session stream, timed region above)
    avg = [x / args.steps for x in stage_one]
    names = ["init", "temporal", "bin", "spatial", "shade"]
    items = band_px * (cfg.bins if cfg.mode == F.MODE_TRANSIENT or plain else 1)
    # the dominant compute kernel (halo staging, which waits on the exchange at
    # N > 1, and queue control have no algorithmic-bytes model)
    cand = {k: v for k, v in ktimes.items() if k in KERNEL_BYTES} or ktimes
    dom = max(cand, key=lambda k: cand[k][0]) if cand else None
    work = {k: work1k[k] - work0k[k] for k in work1k} if work1k else {}  # the instrumented frames
    units = {"pixel": band_px, "item": items}
    if dom and KERNEL_BYTES.get(dom, ("", 0))[0] == "job":
        per_launch_jobs = work.get("shift_jobs", 0) / max(1, sum(v[1] for k, v in ktimes.items()
                                                                  if k == "k_shift_finish"))
        units["job"] = per_launch_jobs
    if dom and KERNEL_BYTES.get(dom, ("", 0))[0] == "merge":  # merge-list items per apply launch
        units["merge"] = work.get("merges", 0) / max(1, sum(v[1] for k, v in ktimes.items()
                                                             if k.endswith("_apply")))
    if plain:  # deposits per launch (one deposit launch per frame)
        units["deposit"] = work.get("deposits", 0) / args.steps
    unit, per_unit = KERNEL_BYTES.get(dom, ("pixel", 0))
    dom_ms, dom_n = ktimes[dom] if dom else (0.0, 1)
    dur_s = dom_ms / max(1, dom_n) * 1e-3
    algo = per_unit * units.get(unit, 0)
    pk = peaks()
    achieved = algo / dur_s / 1e9 if dur_s > 0 else 0.0
    # ncu evidence of the same kernel (profiles/kernel_profile.json, written by
    # tools/kernel_profile.py from a --set full capture of one steady-state
    # frame's launches of this workload): DRAM bytes and FP64 flops per unit of
    # work, scaled to this run's units per launch
    prof = kernel_profile(args.workload, dom)
    upl = units.get(unit, 0)
    traffic = round(prof["dram_bytes_per_unit"] * upl) if prof else None
    fp64 = None
    fp64_peak = r.fp64_peak_gflops() if rank == 0 else 0.0
    if prof and dur_s > 0 and fp64_peak > 0:
        fl = prof["fp64_flops_per_unit"] * upl
        inst = prof["fp64_inst_per_unit"] * upl
        fp64 = {"bound": "fp64", "kernel": dom, "achieved": fl / dur_s / 1e9, "peak": fp64_peak,
                "peak_src": "measured (k_fp64_peak: DFMA chains on this device)", "unit": "GFLOP/s",
                "frac": fl / dur_s / 1e9 / fp64_peak,
                # --fmad=false (parity): DADD/DMUL issue like a DFMA but count one flop, so the
                # pipe occupancy is the instruction rate over the DFMA instruction peak
                "inst_frac": inst / dur_s / 1e9 / (fp64_peak / 2),
                "flops_per_launch": fl, "flops_per_unit": prof["fp64_flops_per_unit"], "unit_of_work": unit,
                "units_per_launch": upl, "avg_launch_ms": dur_s * 1e3, "source": prof["source"]}
    kernel_ms = {k: round(v[0] / args.steps, 4) for k, v in sorted(ktimes.items(), key=lambda kv: -kv[1][0])}
    kernel_launches = {k: round(v[1] / args.steps, 2) for k, v in sorted(ktimes.items(), key=lambda kv: -kv[1][0])}
    workv = {k: work1[k] - work0[k] for k in work1} if work1 else {}  # the value frames
    rays = (workv.get("rays_closest", 0) + workv.get("rays_any", 0)) if workv else 0
    t_s = t_max * 1e-3

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and args.workload in BAND_ONLY:
        cpu = {"value": None, "unit": "frames/s", "cores": os.cpu_count(), "kind": "reference",
               "sample": "not run: the reference's render_transient holds 2.12 G reservoirs of 624 B (1.3 TB per "
                         "grid) at this size (SURVEY 8d)"}
    elif rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            c = cpu_reference_sample(args.workload, 2)
            cpu = {"value": c["frames"] / c["seconds"], "unit": "frames/s", "cores": c["cores"],
                   "kind": "reference",
                   "sample": f"one {c['what']} ({c['seconds']:.1f} s)"}
        except Exception as e:  # the oracle is a reported baseline only
            cpu = {"value": None, "unit": "frames/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": ws, "steps": args.steps,
            "warmup": warm, "warmup_requested": args.warmup, "ms_per_step": t_max / frames, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "scene": scene_name, "resolution": f"{w}x{h}",
                       "parallelism": (f"rowband{emulated[0]}: the band of rank {emulated[1]} (rows "
                                       f"{sess.y0}-{sess.y1} + {sess.halo}-row halos) on one GPU, halo rows "
                                       f"not transferred; value = that band's frames/s"
                                       if emulated else (f"rowband{ws}" + (f" (rows rebalanced on measured band "
                                                                           f"times: {bands})" if bands else "")
                                                         if ws > 1 else "single")),
                       "l2": "inputs larger than L2 (reservoir grids 2 x 730 MB)"},
            "mpaths_per_s": (sess.owned_pixels() if emulated else w * h) * cfg.m_init * fps / 1e6,
            "stage_ms": {**{n: round(a, 4) for n, a in zip(names + ["total"], avg)},
                         "note": "one-stream pass over the same frames (stages sum to its frame); the "
                                 "pipelined value frame overlaps camera + init of f+1 with reuse of f"},
            "frame_ms_curve": curve,
            "work_per_frame": {k: v / frames for k, v in workv.items()} if workv else None,
            # units of work of one value frame, per KERNEL_BYTES unit (tools/kernel_profile.py)
            "units_per_frame": {"pixel": band_px, "item": items,
                                "job": workv.get("shift_jobs", 0) / frames if workv else 0,
                                "deposit": workv.get("deposits", 0) / frames if workv else 0,
                                "merge": workv.get("merges", 0) / frames if workv else 0},
            "shift_stats_one_frame": shift_stats,
            "frame_latency": latency,
            "e2e": {"value": frames / e2e_s, "unit": "frames/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": pk["hbm_gbs"],
                         "peak_src": pk["src"], "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
                         "traffic": traffic, "algo_bytes_per_launch": algo, "bytes_per_unit": per_unit,
                         "unit_of_work": unit, "units_per_launch": units.get(unit, 0),
                         "avg_launch_ms": dur_s * 1e3, "launches": dom_n,
                         "note": "FP64 latency/divergence-bound shift and trace kernels: HBM fraction is small "
                                 "by construction (SURVEY 8d); see rays_per_s and kernel_ms"},
            "roofline_fp64": fp64,
            "kernel_ms_per_step": kernel_ms,
            "kernel_launches_per_step": kernel_launches,
            "reservoir_pool": pool_info,
            "rays_per_s": rays / t_s if t_s > 0 else None,
            "shift_jobs_per_s": workv.get("shift_jobs", 0) / t_s if (t_s > 0 and workv) else None,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--latency-frames", type=int, default=-1,
                    help="frames stepped one at a time for p50/p99 frame latency (default: 30 for c5, else 0)")
    args = ap.parse_args()
    if args.latency_frames < 0:
        args.latency_frames = 30 if args.workload == "c5" else 0
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "nlos_scan":
        run_scan(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
