/*
 * tofr_gpu.hpp -- C++ drop-in shim for users of the reference library `tofr`
 * (/root/reference/proj/include/tofr).  Include it after the reference
 * headers; it maps the reference's own types onto the C ABI of
 * libtofr_b200.so (tofr_gpu.h) and rethrows library errors as
 * std::runtime_error, the way the reference reports failures.
 *
 *   tofr::gpu::render_gated(def, cfg)            <- tofr::render_gated            (pipeline.hpp:323)
 *   tofr::gpu::render_transient(def, cfg)        <- tofr::render_transient        (pipeline.hpp:396)
 *   tofr::gpu::render_transient_plain(def, cfg)  <- tofr::render_transient_plain  (pipeline.hpp:531)
 *   tofr::gpu::reference_render(def, frame, gate, spp, seed, max_depth)
 *                                                <- tofr::reference_render        (harness.hpp:16)
 *
 * Same arguments, same RenderOutput / ReferenceImages; a caller switches by
 * namespace (the CLI's `--device gpu`).  One process-wide
 * context on device 0 unless tofr::gpu::set_device() is called first.
 */
#ifndef TOFR_GPU_HPP
#define TOFR_GPU_HPP

#include <tofr/harness.hpp>
#include <tofr/pipeline.hpp>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "tofr_gpu.h"

namespace tofr {
namespace gpu {

namespace detail {

inline int& device_index() {
    static int d = 0;
    return d;
}

struct Ctx {
    tofr_gpu* h = nullptr;
    explicit Ctx(int dev) {
        int rc = tofr_gpu_create(&dev, 1, &h);
        if (rc != TOFR_OK) throw std::runtime_error("tofr_gpu_create failed (code " + std::to_string(rc) + ")");
    }
    ~Ctx() { tofr_gpu_destroy(h); }
};

inline tofr_gpu* ctx() {
    static std::unique_ptr<Ctx> c;
    if (!c) c = std::make_unique<Ctx>(device_index());
    return c->h;
}

inline void check(int rc, const char* what) {
    if (rc != TOFR_OK) throw std::runtime_error(std::string(what) + ": " + tofr_gpu_last_error(ctx()));
}

inline void put3(double* d, const Vec3& v) {
    d[0] = v.x;
    d[1] = v.y;
    d[2] = v.z;
}

// SceneDef (scene.hpp:417-429) -> tofr_scene (host object of the library)
struct SceneHandle {
    tofr_scene* h = nullptr;
    explicit SceneHandle(const SceneDef& def) {
        tofr_scene_desc d{};
        put3(d.cam_position, def.camera.base.position);
        put3(d.cam_forward, def.camera.base.forward);
        put3(d.cam_up, def.camera.base.up);
        d.fov_y = def.camera.fov_y;
        d.width = def.camera.width;
        d.height = def.camera.height;
        std::vector<tofr_camera_key> ck;
        for (const auto& [fr, p] : def.camera.track) {
            tofr_camera_key k{};
            k.frame = fr;
            put3(k.position, p.position);
            put3(k.forward, p.forward);
            put3(k.up, p.up);
            ck.push_back(k);
        }
        d.n_cam_keys = int32_t(ck.size());
        d.cam_keys = ck.data();
        std::vector<tofr_material> mats;
        for (const Material& m : def.materials) {
            tofr_material tm{};
            tm.kind = int32_t(m.kind);  // MatKind order = TOFR_MAT_*
            put3(tm.albedo, m.albedo);
            tm.roughness = m.roughness;
            mats.push_back(tm);
        }
        d.n_materials = int32_t(mats.size());
        d.materials = mats.data();
        d.light.regime = def.light.regime == LightRegime::Collimated ? TOFR_LIGHT_COLLIMATED : TOFR_LIGHT_WIDE;
        put3(d.light.position, def.light.position);
        put3(d.light.direction, def.light.direction);
        d.light.cone_half_angle = def.light.cone_half_angle;
        put3(d.light.intensity, def.light.intensity);
        std::vector<tofr_object_desc> objs;
        std::vector<std::vector<double>> verts(def.objects.size());
        std::vector<std::vector<int32_t>> tmat(def.objects.size());
        std::vector<std::vector<tofr_pose_key>> keys(def.objects.size());
        for (size_t i = 0; i < def.objects.size(); ++i) {
            const ObjectDef& o = def.objects[i];
            for (const Triangle& t : o.local_tris) {
                for (const Vec3* v : {&t.v0, &t.v1, &t.v2}) {
                    verts[i].push_back(v->x);
                    verts[i].push_back(v->y);
                    verts[i].push_back(v->z);
                }
                tmat[i].push_back(t.material);
            }
            for (const PoseKey& k : o.track.keys) {
                tofr_pose_key pk{};
                pk.frame = k.frame;
                pk.q[0] = k.pose.q.w;
                pk.q[1] = k.pose.q.x;
                pk.q[2] = k.pose.q.y;
                pk.q[3] = k.pose.q.z;
                put3(pk.t, k.pose.t);
                keys[i].push_back(pk);
            }
            tofr_object_desc od{};
            od.name = o.name.c_str();
            od.n_tris = int32_t(o.local_tris.size());
            od.verts = verts[i].data();
            od.materials = tmat[i].data();
            od.n_keys = int32_t(keys[i].size());
            od.keys = keys[i].data();
            objs.push_back(od);
        }
        d.n_objects = int32_t(objs.size());
        d.objects = objs.data();
        d.dt_frame = def.dt_frame;
        char err[512] = {0};
        int rc = tofr_scene_create(&d, &h, err, sizeof(err));
        if (rc != TOFR_OK) throw std::runtime_error(err);
    }
    ~SceneHandle() { tofr_scene_destroy(h); }
    SceneHandle(const SceneHandle&) = delete;
    SceneHandle& operator=(const SceneHandle&) = delete;
};

// RenderConfig (pipeline.hpp:18-61) -> tofr_render_config
inline tofr_render_config to_c(const RenderConfig& r) {
    tofr_render_config c;
    tofr_render_config_default(&c);
    c.mode = int32_t(r.mode);
    c.gate_kind = r.gate.kind == GateSpec::Kind::Velocity ? TOFR_GATE_VELOCITY : TOFR_GATE_LENGTH;
    c.gate_center = r.gate.center;
    c.gate_width = r.gate.width;
    c.gate_f0 = r.gate.f0;
    c.gate_step = r.gate_step;
    c.bins = r.bins;
    c.hist_t0 = r.hist_t0;
    c.hist_bin_width = r.hist_bin_width;
    c.m_init = r.m_init;
    c.init_mode = int32_t(r.init);
    c.shrink_k = r.shrink_k;
    c.shrink_r = r.shrink_r;
    c.spatial_passes = r.spatial_passes;
    c.spatial_neighbors = r.spatial_neighbors;
    c.spatial_radius = r.spatial_radius;
    c.temporal = r.temporal;
    c.bin_reuse = r.bin_reuse;
    c.m_cap = r.m_cap;
    c.gauge = int32_t(r.gauge);
    c.newton = r.newton;
    c.seed = r.seed;
    c.frames = r.frames;
    c.frame0 = r.frame0;
    c.max_depth = r.max_depth;
    c.use_rr = r.use_rr;
    c.accumulate = r.accumulate;
    c.normalize_gate = r.normalize_gate;
    return c;
}

inline void counts_from(ShiftCounts& o, const tofr_shift_counts& c) {
    o.attempts = c.attempts;
    o.newton_ok = c.newton_ok;
    o.newton_failed = c.newton_failed;
    o.occluded = c.occluded;
    o.jac_clamped = c.jac_clamped;
    o.replay_failed = c.replay_failed;
    o.iterations = c.iterations;
    o.solves = c.solves;
    o.success = c.success;
}

using Driver = int (*)(tofr_gpu*, const tofr_scene*, const tofr_render_config*, tofr_output*);

inline RenderOutput run(Driver fn, const char* name, const SceneDef& def, const RenderConfig& cfg, bool transient) {
    SceneHandle sc(def);
    tofr_render_config c = to_c(cfg);
    int W = def.camera.width, H = def.camera.height;
    size_t npix = size_t(W) * H;
    std::vector<double> img(npix * 3), rgb;
    std::vector<int64_t> cnt;
    std::vector<tofr_frame_stats> st(size_t(std::max(0, cfg.frames)));
    tofr_output out{};
    out.image = img.data();
    if (transient) {
        rgb.resize(npix * size_t(cfg.bins) * 3);
        cnt.resize(npix * size_t(cfg.bins));
        out.hist_rgb = rgb.data();
        out.hist_count = cnt.data();
    }
    out.stats = st.data();
    out.stats_capacity = int32_t(st.size());
    check(fn(ctx(), sc.h, &c, &out), name);
    RenderOutput r;
    r.image = Image(W, H);
    for (size_t i = 0; i < npix; ++i) r.image.px[i] = Vec3(img[3 * i], img[3 * i + 1], img[3 * i + 2]);
    if (transient) {
        r.hist = TransientHistogram(W, H, cfg.bins, cfg.hist_t0, cfg.hist_bin_width);
        for (size_t i = 0; i < r.hist.rgb.size(); ++i) {
            r.hist.rgb[i] = Vec3(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
            r.hist.count[i] = cnt[i];
        }
    }
    for (const tofr_frame_stats& s : st) {
        FrameStats f;
        f.frame = s.frame;
        counts_from(f.temporal.shift, s.temporal.shift);
        counts_from(f.spatial.shift, s.spatial.shift);
        counts_from(f.binwise.shift, s.binwise.shift);
        f.temporal.seconds = s.temporal.seconds;
        f.spatial.seconds = s.spatial.seconds;
        f.binwise.seconds = s.binwise.seconds;
        f.t_init = s.t_init;
        f.t_shade = s.t_shade;
        r.stats.push_back(f);
    }
    return r;
}

}  // namespace detail

inline void set_device(int device) { detail::device_index() = device; }

inline RenderOutput render_gated(const SceneDef& def, const RenderConfig& cfg) {
    return detail::run(tofr_gpu_render_gated, "render_gated", def, cfg, false);
}

// render_doppler (pipeline.hpp:573-578): the gated pipeline on the path velocity
inline RenderOutput render_doppler(const SceneDef& def, const RenderConfig& cfg) {
    return detail::run(tofr_gpu_render_doppler, "render_doppler", def, cfg, false);
}

inline RenderOutput render_transient(const SceneDef& def, const RenderConfig& cfg) {
    return detail::run(tofr_gpu_render_transient, "render_transient", def, cfg, true);
}

inline RenderOutput render_transient_plain(const SceneDef& def, const RenderConfig& cfg) {
    return detail::run(tofr_gpu_render_transient_plain, "render_transient_plain", def, cfg, true);
}

// reference_render(build_frame(def, frame), gate, spp, seed, max_depth)
inline ReferenceImages reference_render(const SceneDef& def, double frame, const GateSpec& gate, int spp,
                                        uint64_t seed, int max_depth = 6) {
    detail::SceneHandle sc(def);
    int W = def.camera.width, H = def.camera.height;
    size_t npix = size_t(W) * H;
    std::vector<double> m(npix * 3), e(npix * 3);
    detail::check(tofr_gpu_reference(detail::ctx(), sc.h, frame, gate.center, gate.width, spp, seed, max_depth,
                                     m.data(), e.data()),
                  "reference_render");
    ReferenceImages r{Image(W, H), Image(W, H)};
    for (size_t i = 0; i < npix; ++i) {
        r.mean.px[i] = Vec3(m[3 * i], m[3 * i + 1], m[3 * i + 2]);
        r.se.px[i] = Vec3(e[3 * i], e[3 * i + 1], e[3 * i + 2]);
    }
    return r;
}

// Same signature as the reference (harness.hpp:16): the snapshot names its
// scene definition and frame; the library rebuilds that frame itself.
inline ReferenceImages reference_render(const SceneFrame& fr, const GateSpec& gate, int spp, uint64_t seed,
                                        int max_depth = 6) {
    if (!fr.def) throw std::runtime_error("reference_render: SceneFrame without a SceneDef");
    return reference_render(*fr.def, fr.frame, gate, spp, seed, max_depth);
}

}  // namespace gpu
}  // namespace tofr

#endif  // TOFR_GPU_HPP
