"""Parity cases: (name, scene builder, RenderConfig, driver).  Small enough for
the CPU oracle to finish in seconds; together they exercise every stage of
the hot path (init direct/ellipsoidal/shrink, temporal, spatial, bin reuse,
shade, plain transient deposits, the brute-force reference) on all three
light regimes (collimated beam, wide spot, glossy surfaces, mirrors ->
replayed prefixes with k > 2, animated geometry)."""
from __future__ import annotations

from paper_2605_11536_b200 import _ffi as F
from paper_2605_11536_b200 import scenes
from paper_2605_11536_b200.api import GateSpec, RenderConfig


def gate(c, w):
    return GateSpec(F.GATE_LENGTH, c, w, 1.0)


def mirror_box(res=32):
    return scenes.cornell_box(collimated=False, resolution=res, tall_box_material=3,
                              tall_box_kind=F.MAT_MIRROR)


def glossy_box(res=32, rough=0.1):
    return scenes.cornell_box(collimated=False, resolution=res, tall_box_material=3, tall_box_roughness=rough)


CASES = {
    # gated, init only
    "gated_init_cornell": (lambda: scenes.bundled("cornell", 48), RenderConfig(gate=gate(10.0, 0.35), m_init=4),
                           "gated"),
    "gated_init_wide": (lambda: scenes.bundled("cornell_wide", 48), RenderConfig(gate=gate(6.0, 0.3), m_init=4),
                        "gated"),
    # C1-style: temporal + 1x3 spatial, m_init 1, several frames
    "c1_cornell": (lambda: scenes.bundled("cornell", 64),
                   RenderConfig(gate=gate(10.0, 0.0866), m_init=1, temporal=True, spatial_passes=1,
                                spatial_neighbors=3, spatial_radius=10, frames=3), "gated"),
    "c1_cornell_wide_gate": (lambda: scenes.bundled("cornell", 48),
                             RenderConfig(gate=gate(10.0, 0.5), m_init=2, temporal=True, spatial_passes=2,
                                          spatial_neighbors=3, spatial_radius=6, frames=3, seed=7), "gated"),
    "wide_reuse": (lambda: scenes.bundled("cornell_wide", 48),
                   RenderConfig(gate=gate(6.0, 0.2), m_init=2, temporal=True, spatial_passes=1,
                                spatial_neighbors=3, spatial_radius=8, frames=3, gate_step=0.01), "gated"),
    "doppler_scene_reuse": (lambda: scenes.bundled("boxes_doppler", 48),
                            RenderConfig(gate=gate(12.0, 0.3), m_init=2, temporal=True, spatial_passes=1,
                                         spatial_neighbors=3, spatial_radius=8, frames=3, frame0=2), "gated"),
    "mirror_replay": (lambda: mirror_box(32),
                      RenderConfig(gate=gate(6.0, 0.4), m_init=4, temporal=True, spatial_passes=1,
                                   spatial_neighbors=4, spatial_radius=5, frames=2, max_depth=8), "gated"),
    "glossy_low_rough": (lambda: glossy_box(32, 0.1),
                         RenderConfig(gate=gate(6.0, 0.4), m_init=4, temporal=True, spatial_passes=1,
                                      spatial_neighbors=3, spatial_radius=5, frames=2), "gated"),
    "gauge_fixed": (lambda: scenes.bundled("cornell_wide", 32),
                    RenderConfig(gate=gate(6.0, 0.3), m_init=2, spatial_passes=1, spatial_neighbors=3,
                                 spatial_radius=5, gauge=F.GAUGE_FIXED), "gated"),
    "gauge_raw": (lambda: scenes.bundled("cornell_wide", 32),
                  RenderConfig(gate=gate(6.0, 0.3), m_init=2, spatial_passes=1, spatial_neighbors=3,
                               spatial_radius=5, gauge=F.GAUGE_RAW), "gated"),
    "naive_reuse": (lambda: scenes.bundled("cornell", 32),
                    RenderConfig(gate=gate(10.0, 0.3), m_init=2, temporal=True, spatial_passes=1,
                                 spatial_neighbors=3, spatial_radius=5, frames=2, newton=False), "gated"),
    "accum_normalize": (lambda: scenes.bundled("cornell", 32),
                        RenderConfig(gate=gate(10.0, 0.3), m_init=2, temporal=True, frames=3, accumulate=True,
                                     normalize_gate=True), "gated"),
    "ellipsoidal_init": (lambda: scenes.bundled("cornell_wide", 32),
                         RenderConfig(gate=gate(6.0, 0.1), m_init=2, init=F.INIT_ELLIPSOIDAL), "gated"),
    "ellipsoidal_collimated": (lambda: scenes.bundled("cornell", 24),
                               RenderConfig(gate=gate(10.0, 0.1), m_init=2, init=F.INIT_ELLIPSOIDAL,
                                            spatial_passes=1, spatial_neighbors=3, spatial_radius=4), "gated"),
    "shrink_r1": (lambda: scenes.bundled("cornell_wide", 32),
                  RenderConfig(gate=gate(6.0, 0.05), m_init=4, init=F.INIT_SHRINK, shrink_k=10, shrink_r=1.0),
                  "gated"),
    "shrink_r05": (lambda: scenes.bundled("cornell_wide", 32),
                   RenderConfig(gate=gate(6.0, 0.05), m_init=4, init=F.INIT_SHRINK, shrink_k=10, shrink_r=0.5),
                   "gated"),
    # shrink initialiser under temporal + spatial reuse, on moving boxes, and
    # with every tree on the fine gate (R = 0: the plain RIS)
    "shrink_r05_reuse": (lambda: scenes.bundled("boxes_doppler", 28),
                         RenderConfig(gate=gate(10.0, 0.3), m_init=3, init=F.INIT_SHRINK, shrink_k=4, shrink_r=0.5,
                                      temporal=True, spatial_passes=1, spatial_neighbors=3, spatial_radius=4,
                                      frames=3),
                         "gated"),
    "shrink_r0": (lambda: scenes.bundled("cornell_wide", 24),
                  RenderConfig(gate=gate(6.0, 0.05), m_init=2, init=F.INIT_SHRINK, shrink_k=10, shrink_r=0.0,
                               temporal=True, frames=2),
                  "gated"),
    # transient
    "plain_cornell": (lambda: scenes.bundled("cornell", 32),
                      RenderConfig(mode=F.MODE_TRANSIENT, bins=64, hist_t0=8.0, hist_bin_width=0.1875, m_init=2,
                                   frames=2), "plain"),
    "plain_doppler": (lambda: scenes.bundled("boxes_doppler", 24),
                      RenderConfig(mode=F.MODE_TRANSIENT, bins=100, hist_t0=7.0, hist_bin_width=0.2, m_init=2,
                                   frames=2, max_depth=8), "plain"),
    "transient_temporal": (lambda: scenes.bundled("cornell", 24),
                           RenderConfig(mode=F.MODE_TRANSIENT, bins=32, hist_t0=8.0, hist_bin_width=0.375,
                                        m_init=2, temporal=True, frames=3), "transient"),
    "transient_full": (lambda: scenes.bundled("cornell_wide", 20),
                       RenderConfig(mode=F.MODE_TRANSIENT, bins=16, hist_t0=5.0, hist_bin_width=0.25, m_init=2,
                                    temporal=True, bin_reuse=True, spatial_passes=1, spatial_neighbors=2,
                                    spatial_radius=3, frames=2), "transient"),
    # bin reuse after temporal reuse, no spatial pass (the wavefront bin stage
    # alone), and on moving geometry
    "transient_bin_reuse": (lambda: scenes.bundled("cornell", 24),
                            RenderConfig(mode=F.MODE_TRANSIENT, bins=32, hist_t0=8.0, hist_bin_width=0.375,
                                         m_init=2, temporal=True, bin_reuse=True, frames=3), "transient"),
    "transient_bin_reuse_animated": (lambda: scenes.bundled("boxes_doppler", 20),
                                     RenderConfig(mode=F.MODE_TRANSIENT, bins=24, hist_t0=7.0, hist_bin_width=0.5,
                                                  m_init=2, temporal=True, bin_reuse=True, max_depth=8, frames=3),
                                     "transient"),
    "transient_b1_equals_gated": (lambda: scenes.bundled("cornell", 24),
                                  RenderConfig(mode=F.MODE_TRANSIENT, bins=1, hist_t0=10.0 - 0.25,
                                               hist_bin_width=0.5, m_init=4, spatial_passes=1,
                                               spatial_neighbors=2, spatial_radius=3, seed=7), "transient"),
}

# Doppler (velocity) gates: render_doppler, pipeline.hpp:573-578 -- the gated
# pipeline on the path velocity u (receding big box ~ -0.1, approaching small
# box > 0, static geometry 0 in boxes_doppler, f0 = 1 Hz so shift = u)
def vgate(c, w, f0=1.0):
    return GateSpec(F.GATE_VELOCITY, c, w, f0)


CASES.update({
    "doppler_receding": (lambda: scenes.bundled("boxes_doppler", 48),
                         RenderConfig(gate=vgate(-0.09, 0.04), m_init=2, temporal=True, spatial_passes=1,
                                      spatial_neighbors=3, spatial_radius=8, frames=3, frame0=2), "doppler"),
    "doppler_approaching": (lambda: scenes.bundled("boxes_doppler", 48),
                            RenderConfig(gate=vgate(0.06, 0.06), m_init=2, temporal=True, spatial_passes=1,
                                         spatial_neighbors=3, spatial_radius=8, frames=3, frame0=5), "doppler"),
    "doppler_wide_f0": (lambda: scenes.bundled("boxes_doppler", 40),
                        RenderConfig(gate=vgate(-0.1, 0.4, 2.0), m_init=2, temporal=True, spatial_passes=2,
                                     spatial_neighbors=3, spatial_radius=6, frames=3, gate_step=0.01, frame0=1),
                        "doppler"),
})

# 102,410-triangle scene (a real BVH, traversed from global memory)
CASES["mesh_torus_reuse"] = (lambda: scenes.mesh_scene(48),
                             RenderConfig(gate=gate(6.0, 0.2), m_init=1, temporal=True, spatial_passes=1,
                                          spatial_neighbors=3, spatial_radius=6, frames=2), "gated")

# the same mesh moving (a new BVH every frame: built on the device by default)
CASES["mesh_anim_reuse"] = (lambda: scenes.mesh_scene(40, animated=True),
                            RenderConfig(gate=gate(6.0, 0.2), m_init=1, temporal=True, spatial_passes=1,
                                         spatial_neighbors=3, spatial_radius=6, frames=3, frame0=4), "gated")

REFERENCE_CASES = {
    "ref_cornell_wide": (lambda: scenes.bundled("cornell_wide", 32), 0.0, gate(6.0, 0.5), 16, 3, 6),
    "ref_cornell": (lambda: scenes.bundled("cornell", 32), 0.0, gate(10.0, 0.5), 16, 5, 6),
    "ref_doppler": (lambda: scenes.bundled("boxes_doppler", 24), 4.0, gate(12.0, 0.5), 8, 9, 8),
}

# BASELINE.json configurations at their full sizes, or -- where the
# reference's 624 B reservoirs do not fit the GPU box's host RAM -- at the
# largest size the oracle renders in a few minutes with the config otherwise
# unchanged: C2(ii) at 256^2 x 256 bins (21 GB of oracle grids; 512^2 needs
# 84 GB per pair and ~10 min per frame), C4 reservoirs at 128x72 x 1024 bins
# (18 GB), C5 at 256^2 over 25 frames of the gate sweep.
FULL_CASES = {
    "full_c2r_cornell_256_256bins": (lambda: scenes.bundled("cornell", 256, 256),
                                     RenderConfig(mode=F.MODE_TRANSIENT, bins=256, hist_t0=8.0,
                                                  hist_bin_width=0.046875, m_init=1, temporal=True, m_cap=20,
                                                  max_depth=6, frames=3, seed=1), "transient"),
    "full_c4r_doppler_128x72_1024bins": (lambda: scenes.bundled("boxes_doppler", 128, 72),
                                         RenderConfig(mode=F.MODE_TRANSIENT, bins=1024, hist_t0=7.0,
                                                      hist_bin_width=0.01953125, m_init=1, max_depth=8,
                                                      temporal=True, spatial_passes=1, spatial_neighbors=3,
                                                      spatial_radius=10, m_cap=20, frames=3, seed=1),
                                         "transient"),
    # the paper's gated timing configuration: ellipsoidal initial
    # sampling + temporal + spatial reuse at 256^2 with a narrow gate (bench `nlos`)
    "nlos_cornell_wide_256": (lambda: scenes.bundled("cornell_wide", 256, 256),
                              RenderConfig(gate=gate(6.0, 0.01), m_init=1, init=F.INIT_ELLIPSOIDAL, temporal=True,
                                           spatial_passes=1, spatial_neighbors=3, spatial_radius=10, m_cap=20,
                                           max_depth=6, frames=4, seed=1), "gated"),
    "full_c5_cornell_wide_256_25frames": (lambda: scenes.bundled("cornell_wide", 256, 256),
                                          RenderConfig(gate=gate(6.0, 0.0173), gate_step=0.01, m_init=1,
                                                       temporal=True, spatial_passes=1, spatial_neighbors=3,
                                                       spatial_radius=10, m_cap=20, max_depth=6, frames=25,
                                                       seed=1), "gated"),
    "full_c3_boxes_doppler_1080p": (lambda: scenes.bundled("boxes_doppler", 1920, 1080),
                                    RenderConfig(gate=gate(12.0, 0.041), m_init=1, temporal=True, spatial_passes=1,
                                                 spatial_neighbors=3, spatial_radius=10, m_cap=20, max_depth=6,
                                                 frames=3, seed=1), "gated"),
    "full_c3w_cornell_wide_1080p": (lambda: scenes.bundled("cornell_wide", 1920, 1080),
                                    RenderConfig(gate=gate(6.0, 0.0173), m_init=1, temporal=True, spatial_passes=1,
                                                 spatial_neighbors=3, spatial_radius=10, m_cap=20, max_depth=6,
                                                 frames=2, seed=1), "gated"),
    "full_c1_cornell_256": (lambda: scenes.bundled("cornell", 256, 256),
                            RenderConfig(gate=gate(10.0, 0.0866), m_init=1, temporal=True, spatial_passes=1,
                                         spatial_neighbors=3, spatial_radius=10, m_cap=20, max_depth=6, frames=4,
                                         seed=1), "gated"),
    "full_c2p_cornell_512_256bins": (lambda: scenes.bundled("cornell", 512, 512),
                                     RenderConfig(mode=F.MODE_TRANSIENT, bins=256, hist_t0=8.0,
                                                  hist_bin_width=0.046875, m_init=1, max_depth=6, frames=2, seed=1),
                                     "plain"),
}
