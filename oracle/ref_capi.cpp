// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin C ABI over the *unmodified* CPU reference headers
// (/root/reference/proj/include/tofr, compiled where they lie; nothing is
// copied).  It lets the parity tests, smoke() and bench.py's cpu_baseline /
// --impl reference arm run the reference renderer on the same scene and
// RenderConfig as the GPU path.  The product library never links this.
//
// Built by oracle/Makefile into oracle/_ref/libtofr_ref.so with the
// reference's own compiler flags (g++ -O2, x86-64 baseline: no FMA
// contraction), so results are the reference's bit for bit.
#include <tofr/harness.hpp>
#include <tofr/scene_io.hpp>

#include <cstring>
#include <functional>
#include <memory>
#include <string>

#include "../include/tofr_gpu.h"

using namespace tofr;

struct ref_scene {
    SceneDef def;
};

namespace {

void set_err(char* err, size_t n, const std::string& m) {
    if (err && n) std::snprintf(err, n, "%s", m.c_str());
}

int guard(char* err, size_t n, const std::function<void()>& fn) {
    try {
        fn();
        set_err(err, n, "");
        return TOFR_OK;
    } catch (const ParseError& e) {
        set_err(err, n, std::to_string(e.line) + ":" + std::to_string(e.col) + ": " + e.what());
        return TOFR_ERR_PARSE;
    } catch (const std::exception& e) {
        set_err(err, n, e.what());
        return TOFR_ERR_SCENE;
    }
}

Vec3 v3(const double* p) { return {p[0], p[1], p[2]}; }

RenderConfig to_ref(const tofr_render_config& c) {
    RenderConfig r;
    r.mode = c.mode == TOFR_MODE_TRANSIENT ? RenderMode::Transient
             : c.mode == TOFR_MODE_DOPPLER ? RenderMode::Doppler
                                           : RenderMode::Gated;
    r.gate.kind = c.gate_kind == TOFR_GATE_VELOCITY ? GateSpec::Kind::Velocity : GateSpec::Kind::Length;
    r.gate.center = c.gate_center;
    r.gate.width = c.gate_width;
    r.gate.f0 = c.gate_f0;
    r.gate_step = c.gate_step;
    r.bins = c.bins;
    r.hist_t0 = c.hist_t0;
    r.hist_bin_width = c.hist_bin_width;
    r.m_init = c.m_init;
    r.init = c.init_mode == TOFR_INIT_ELLIPSOIDAL ? InitMode::Ellipsoidal
             : c.init_mode == TOFR_INIT_SHRINK    ? InitMode::Shrink
                                                  : InitMode::Direct;
    r.shrink_k = c.shrink_k;
    r.shrink_r = c.shrink_r;
    r.spatial_passes = c.spatial_passes;
    r.spatial_neighbors = c.spatial_neighbors;
    r.spatial_radius = c.spatial_radius;
    r.temporal = c.temporal != 0;
    r.bin_reuse = c.bin_reuse != 0;
    r.m_cap = c.m_cap;
    r.gauge = c.gauge == TOFR_GAUGE_FIXED ? GaugeKind::FixedAxis
              : c.gauge == TOFR_GAUGE_RAW ? GaugeKind::RawGradient
                                          : GaugeKind::AverageGradient;
    r.newton = c.newton != 0;
    r.seed = c.seed;
    r.frames = c.frames;
    r.frame0 = c.frame0;
    r.max_depth = c.max_depth;
    r.use_rr = c.use_rr != 0;
    r.accumulate = c.accumulate != 0;
    r.normalize_gate = c.normalize_gate != 0;
    return r;
}

void copy_counts(tofr_shift_counts& o, const ShiftCounts& s) {
    o.attempts = s.attempts;
    o.newton_ok = s.newton_ok;
    o.newton_failed = s.newton_failed;
    o.occluded = s.occluded;
    o.jac_clamped = s.jac_clamped;
    o.replay_failed = s.replay_failed;
    o.iterations = s.iterations;
    o.solves = s.solves;
    o.success = s.success;
}

void write_output(const RenderOutput& r, tofr_output* out) {
    if (!out) return;
    if (out->image)
        for (size_t i = 0; i < r.image.px.size(); ++i) {
            out->image[3 * i + 0] = r.image.px[i].x;
            out->image[3 * i + 1] = r.image.px[i].y;
            out->image[3 * i + 2] = r.image.px[i].z;
        }
    if (out->hist_rgb)
        for (size_t i = 0; i < r.hist.rgb.size(); ++i) {
            out->hist_rgb[3 * i + 0] = r.hist.rgb[i].x;
            out->hist_rgb[3 * i + 1] = r.hist.rgb[i].y;
            out->hist_rgb[3 * i + 2] = r.hist.rgb[i].z;
        }
    if (out->hist_count)
        for (size_t i = 0; i < r.hist.count.size(); ++i) out->hist_count[i] = r.hist.count[i];
    if (out->stats)
        for (size_t f = 0; f < r.stats.size() && int(f) < out->stats_capacity; ++f) {
            const FrameStats& s = r.stats[f];
            tofr_frame_stats& o = out->stats[f];
            std::memset(&o, 0, sizeof(o));
            o.frame = s.frame;
            copy_counts(o.temporal.shift, s.temporal.shift);
            copy_counts(o.spatial.shift, s.spatial.shift);
            copy_counts(o.binwise.shift, s.binwise.shift);
            o.temporal.seconds = s.temporal.seconds;
            o.spatial.seconds = s.spatial.seconds;
            o.binwise.seconds = s.binwise.seconds;
            o.t_init = s.t_init;
            o.t_shade = s.t_shade;
        }
}

}  // namespace

extern "C" {

void ref_set_threads(int n) { worker_count() = n > 0 ? n : int(std::thread::hardware_concurrency()); }
int ref_get_threads(void) { return worker_count(); }

int ref_scene_load(const char* path, ref_scene** out, char* err, size_t n) {
    *out = nullptr;
    return guard(err, n, [&] {
        auto s = std::make_unique<ref_scene>();
        s->def = load_scene(path);
        *out = s.release();
    });
}

int ref_scene_parse(const char* text, const char* base_dir, ref_scene** out, char* err, size_t n) {
    *out = nullptr;
    return guard(err, n, [&] {
        auto s = std::make_unique<ref_scene>();
        s->def = parse_scene(text, base_dir ? base_dir : ".");
        *out = s.release();
    });
}

// SceneDef from the same plain description the GPU library takes.
int ref_scene_create(const tofr_scene_desc* d, ref_scene** out, char* err, size_t n) {
    *out = nullptr;
    return guard(err, n, [&] {
        auto s = std::make_unique<ref_scene>();
        SceneDef& def = s->def;
        def.camera.base.position = v3(d->cam_position);
        def.camera.base.forward = v3(d->cam_forward);
        def.camera.base.up = v3(d->cam_up);
        def.camera.fov_y = d->fov_y;
        def.camera.width = d->width;
        def.camera.height = d->height;
        for (int i = 0; i < d->n_cam_keys; ++i) {
            CameraPose p;
            p.position = v3(d->cam_keys[i].position);
            p.forward = v3(d->cam_keys[i].forward);
            p.up = v3(d->cam_keys[i].up);
            def.camera.track.emplace_back(d->cam_keys[i].frame, p);
        }
        for (int i = 0; i < d->n_materials; ++i) {
            Material m;
            m.kind = MatKind(d->materials[i].kind);
            m.albedo = v3(d->materials[i].albedo);
            m.roughness = d->materials[i].roughness;
            def.add_material(m);
        }
        if (def.materials.empty()) def.add_material(Material{});
        def.light.regime = d->light.regime == TOFR_LIGHT_WIDE ? LightRegime::Wide : LightRegime::Collimated;
        def.light.position = v3(d->light.position);
        def.light.direction = v3(d->light.direction);
        def.light.cone_half_angle = d->light.cone_half_angle;
        def.light.intensity = v3(d->light.intensity);
        for (int i = 0; i < d->n_objects; ++i) {
            const tofr_object_desc& od = d->objects[i];
            ObjectDef o;
            o.name = od.name ? od.name : "";
            for (int t = 0; t < od.n_tris; ++t) {
                const double* v = od.verts + 9 * size_t(t);
                o.local_tris.push_back(
                    make_triangle(v3(v), v3(v + 3), v3(v + 6), od.materials ? od.materials[t] : 0));
            }
            for (int k = 0; k < od.n_keys; ++k) {
                PoseKey pk;
                pk.frame = od.keys[k].frame;
                pk.pose.q = {od.keys[k].q[0], od.keys[k].q[1], od.keys[k].q[2], od.keys[k].q[3]};
                pk.pose.t = v3(od.keys[k].t);
                o.track.keys.push_back(pk);
            }
            def.objects.push_back(std::move(o));
        }
        def.dt_frame = d->dt_frame;
        *out = s.release();
    });
}

void ref_scene_destroy(ref_scene* s) { delete s; }

int ref_scene_set_resolution(ref_scene* s, int w, int h) {
    s->def.camera.width = w;
    s->def.camera.height = h;
    return 0;
}

int ref_render_gated(ref_scene* s, const tofr_render_config* c, tofr_output* out, char* err, size_t n) {
    return guard(err, n, [&] { write_output(render_gated(s->def, to_ref(*c)), out); });
}

int ref_render_transient(ref_scene* s, const tofr_render_config* c, tofr_output* out, char* err, size_t n) {
    return guard(err, n, [&] {
        RenderConfig r = to_ref(*c);
        r.mode = RenderMode::Transient;
        write_output(render_transient(s->def, r), out);
    });
}

int ref_render_transient_plain(ref_scene* s, const tofr_render_config* c, tofr_output* out, char* err,
                               size_t n) {
    return guard(err, n, [&] { write_output(render_transient_plain(s->def, to_ref(*c)), out); });
}

int ref_reference(ref_scene* s, double frame, double center, double width, int spp, uint64_t seed, int max_depth,
                  double* mean, double* se, char* err, size_t n) {
    return guard(err, n, [&] {
        SceneFrame fr = build_frame(s->def, frame);
        GateSpec g;
        g.kind = GateSpec::Kind::Length;
        g.center = center;
        g.width = width;
        ReferenceImages r = reference_render(fr, g, spp, seed, max_depth);
        for (size_t i = 0; i < r.mean.px.size(); ++i) {
            mean[3 * i] = r.mean.px[i].x;
            mean[3 * i + 1] = r.mean.px[i].y;
            mean[3 * i + 2] = r.mean.px[i].z;
            if (se) {
                se[3 * i] = r.se.px[i].x;
                se[3 * i + 1] = r.se.px[i].y;
                se[3 * i + 2] = r.se.px[i].z;
            }
        }
    });
}

// BVH of build_frame(def, frame): nodes as 11 doubles
// {lo.xyz, hi.xyz, tri_area, left, right, first, count} + parent, tri_order
int ref_dump_bvh(ref_scene* s, double frame, int cap_nodes, double* nodes, int* parent, int* n_nodes, int cap_tris,
                 int* tri_order, int* n_tris, double* diag, char* err, size_t n) {
    return guard(err, n, [&] {
        SceneFrame fr = build_frame(s->def, frame);
        const auto& ns = fr.bvh->nodes();
        *n_nodes = int(ns.size());
        *n_tris = int(fr.bvh->triangles().size());
        *diag = fr.bvh->scene_diag();
        if (int(ns.size()) <= cap_nodes)
            for (size_t i = 0; i < ns.size(); ++i) {
                double* o = nodes + 11 * i;
                o[0] = ns[i].box.lo.x;
                o[1] = ns[i].box.lo.y;
                o[2] = ns[i].box.lo.z;
                o[3] = ns[i].box.hi.x;
                o[4] = ns[i].box.hi.y;
                o[5] = ns[i].box.hi.z;
                o[6] = ns[i].tri_area;
                o[7] = ns[i].left;
                o[8] = ns[i].right;
                o[9] = ns[i].first;
                o[10] = ns[i].count;
                parent[i] = ns[i].parent;
            }
        if (int(fr.bvh->tri_order().size()) <= cap_tris)
            for (size_t i = 0; i < fr.bvh->tri_order().size(); ++i) tri_order[i] = fr.bvh->tri_order()[i];
    });
}

// rays[i] = {o.xyz, d.xyz, tmin, tmax}; mode 0: intersect_min -> (t, tri);
// mode 1: occluded(o, d) -> tri = 0/1
int ref_probe_rays(ref_scene* s, double frame, const double* rays, int count, int mode, double* out_t,
                   int* out_tri, char* err, size_t n) {
    return guard(err, n, [&] {
        SceneFrame fr = build_frame(s->def, frame);
        for (int i = 0; i < count; ++i) {
            const double* r = rays + 8 * size_t(i);
            if (mode == 0) {
                Ray ray{v3(r), v3(r + 3)};
                auto h = fr.bvh->intersect_min(ray, r[6], r[7]);
                out_t[i] = h ? h->t : kInf;
                out_tri[i] = h ? h->tri : -1;
            } else {
                out_tri[i] = fr.bvh->occluded(v3(r), v3(r + 3)) ? 1 : 0;
                out_t[i] = 0;
            }
        }
    });
}

// Counter-RNG draws (rng.hpp:24-44): out[i] = i-th next() of the stream
void ref_rng_stream(uint64_t seed, uint64_t frame, uint64_t pixel, uint64_t sample, uint64_t lane, int count,
                    double* out, uint64_t* out_u64) {
    Rng r(seed, frame, pixel, sample, lane);
    Rng r2 = r;
    for (int i = 0; i < count; ++i) {
        if (out) out[i] = r.next();
        if (out_u64) out_u64[i] = r2.next_u64();
    }
}

// stage::neighbor_offset with the key spatial_reuse builds (pipeline.hpp:255-258)
void ref_neighbor_offsets(uint64_t pix, int pass, uint64_t seed, int frame_idx, int count, double radius,
                          int* out_dx_dy) {
    for (int j = 0; j < count; ++j) {
        auto [dx, dy] = stage::neighbor_offset(
            j, count, radius, mix64(pix * 1315423911u + pass * 2654435761u + uint64_t(seed) + uint64_t(frame_idx) * 97));
        out_dx_dy[2 * j] = dx;
        out_dx_dy[2 * j + 1] = dy;
    }
}

int ref_bin_of(int bins, double t0, double bw, const double* lens, int count, int* out) {
    TransientHistogram h(1, 1, bins, t0, bw);
    for (int i = 0; i < count; ++i) out[i] = h.bin_of(lens[i]);
    return 0;
}

// stage::initial_sampling for every pixel of frame `frame_idx` (gated):
// per pixel {W, M, phat, len, has, k}
int ref_initial_sampling(ref_scene* s, const tofr_render_config* c, int frame_idx, double* W, double* M,
                         double* phat, double* len, int* has, int* k, char* err, size_t n) {
    return guard(err, n, [&] {
        RenderConfig cfg = to_ref(*c);
        SceneFrame fr = build_frame(s->def, cfg.frame0 + frame_idx);
        GateSpec gate = cfg.gate_at(frame_idx);
        int Wd = s->def.camera.width, Hd = s->def.camera.height;
        parallel_for(Hd, [&](int y) {
            for (int x = 0; x < Wd; ++x) {
                Reservoir r = stage::initial_sampling(fr, cfg, gate, x, y, frame_idx);
                size_t i = size_t(y) * Wd + x;
                W[i] = r.W;
                M[i] = r.M;
                phat[i] = r.phat_y;
                len[i] = r.y.len;
                has[i] = r.has ? 1 : 0;
                k[i] = r.y.rec.k;
            }
        });
    });
}

// compute_metrics (pipeline.hpp:588-607) on two W x H x 3 images
void ref_compute_metrics(const double* est, const double* refimg, int w, int h, double* mape, double* relmse) {
    Image a(w, h), b(w, h);
    for (size_t i = 0; i < size_t(w) * h; ++i) {
        a.px[i] = {est[3 * i], est[3 * i + 1], est[3 * i + 2]};
        b.px[i] = {refimg[3 * i], refimg[3 * i + 1], refimg[3 * i + 2]};
    }
    Metrics m = compute_metrics(a, b);
    *mape = m.mape;
    *relmse = m.relmse;
}

}  // extern "C"
