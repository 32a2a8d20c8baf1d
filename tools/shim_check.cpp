// shim_check.cpp -- drop-in check of include/tofr_gpu.hpp.
//
// A C++ program written against the reference library's own types
// (tofr::SceneDef, tofr::RenderConfig, tofr::RenderOutput) that renders the
// same scene twice: with the reference CPU renderer (tofr::render_gated,
// pipeline.hpp:323) and through the GPU shim (tofr::gpu::render_gated ->
// libtofr_b200.so).  It prints one JSON line with the fraction of pixels
// within 1e-4 relative error and exits non-zero below 99.9 %.
//
// Built by `make -C oracle shim` into oracle/_ref/shim_check (compiles the
// unmodified reference headers where they lie; test infrastructure only).
#include <cmath>
#include <cstdio>

#include "../include/tofr_gpu.hpp"

using namespace tofr;

namespace {

void quad(ObjectDef& o, Vec3 a, Vec3 b, Vec3 c, Vec3 d, int m) {
    o.local_tris.push_back(make_triangle(a, b, c, m));
    o.local_tris.push_back(make_triangle(a, c, d, m));
}

// A small open box lit by a wide spot below the ceiling (our own geometry).
SceneDef box_scene(int res) {
    SceneDef d;
    d.camera.base.position = Vec3(0, 0, 3);
    d.camera.base.forward = Vec3(0, 0, -1);
    d.camera.base.up = Vec3(0, 1, 0);
    d.camera.fov_y = 0.6435;
    d.camera.width = d.camera.height = res;
    Material white, red, green, gloss;
    white.albedo = Vec3(0.75, 0.75, 0.75);
    red.albedo = Vec3(0.7, 0.15, 0.12);
    green.albedo = Vec3(0.15, 0.6, 0.15);
    gloss.kind = MatKind::Glossy;
    gloss.albedo = Vec3(0.8, 0.8, 0.8);
    gloss.roughness = 0.3;
    int w = d.add_material(white), r = d.add_material(red), g = d.add_material(green), gl = d.add_material(gloss);
    d.light.position = Vec3(0, 0.9, 0);
    d.light.direction = Vec3(0, -1, 0);
    d.light.cone_half_angle = 2.7;
    d.light.intensity = Vec3(8, 8, 8);
    d.light.regime = LightRegime::Wide;
    ObjectDef shell;
    shell.name = "shell";
    quad(shell, {-1, -1, -1}, {1, -1, -1}, {1, 1, -1}, {-1, 1, -1}, w);   // back
    quad(shell, {-1, -1, -1}, {-1, -1, 1}, {1, -1, 1}, {1, -1, -1}, w);   // floor
    quad(shell, {-1, 1, -1}, {1, 1, -1}, {1, 1, 1}, {-1, 1, 1}, w);       // ceiling
    quad(shell, {-1, -1, -1}, {-1, 1, -1}, {-1, 1, 1}, {-1, -1, 1}, r);   // left
    quad(shell, {1, -1, -1}, {1, -1, 1}, {1, 1, 1}, {1, 1, -1}, g);       // right
    ObjectDef block;
    block.name = "block";
    quad(block, {0.1, -1, -0.5}, {0.6, -1, -0.5}, {0.6, -0.3, -0.5}, {0.1, -0.3, -0.5}, gl);
    quad(block, {0.1, -0.3, -0.5}, {0.6, -0.3, -0.5}, {0.6, -0.3, 0.0}, {0.1, -0.3, 0.0}, gl);
    quad(block, {0.1, -1, 0.0}, {0.1, -0.3, 0.0}, {0.6, -0.3, 0.0}, {0.6, -1, 0.0}, gl);
    d.objects.push_back(shell);
    d.objects.push_back(block);
    return d;
}

double within(const Image& a, const Image& b, double* max_rel) {
    size_t ok = 0;
    *max_rel = 0;
    for (size_t i = 0; i < a.px.size(); ++i) {
        const double av[3] = {a.px[i].x, a.px[i].y, a.px[i].z}, bv[3] = {b.px[i].x, b.px[i].y, b.px[i].z};
        bool good = true;
        for (int c = 0; c < 3; ++c) {
            double den = std::max(std::abs(bv[c]), 1e-12);
            double rel = std::abs(av[c] - bv[c]) / den;
            if (std::abs(av[c] - bv[c]) > 1e-12) {
                *max_rel = std::max(*max_rel, rel);
                if (rel > 1e-4) good = false;
            }
        }
        ok += good;
    }
    return double(ok) / double(a.px.size());
}

}  // namespace

int main() {
    SceneDef def = box_scene(48);
    RenderConfig cfg;
    cfg.gate.center = 6.0;
    cfg.gate.width = 0.3;
    cfg.m_init = 2;
    cfg.temporal = true;
    cfg.spatial_passes = 1;
    cfg.spatial_neighbors = 3;
    cfg.spatial_radius = 6;
    cfg.frames = 3;
    RenderOutput cpu = render_gated(def, cfg);
    RenderOutput gpu = gpu::render_gated(def, cfg);
    double mr = 0;
    double frac = within(gpu.image, cpu.image, &mr);

    RenderConfig tc;
    tc.mode = RenderMode::Transient;
    tc.bins = 64;
    tc.hist_t0 = 3.0;
    tc.hist_bin_width = 0.125;
    tc.m_init = 2;
    tc.frames = 2;
    RenderOutput cpu_t = render_transient_plain(def, tc);
    RenderOutput gpu_t = gpu::render_transient_plain(def, tc);
    size_t cnt_diff = 0;
    for (size_t i = 0; i < cpu_t.hist.count.size(); ++i) cnt_diff += cpu_t.hist.count[i] != gpu_t.hist.count[i];
    double mr_t = 0;
    double frac_t = within(gpu_t.image, cpu_t.image, &mr_t);

    uint64_t att_cpu = 0, att_gpu = 0;
    for (const auto& s : cpu.stats) att_cpu += s.spatial.shift.attempts + s.temporal.shift.attempts;
    for (const auto& s : gpu.stats) att_gpu += s.spatial.shift.attempts + s.temporal.shift.attempts;
    std::printf("{\"gated_within\": %.6f, \"gated_max_rel\": %.3e, \"plain_within\": %.6f, \"plain_count_diff\": %zu,"
                " \"shift_attempts_cpu\": %llu, \"shift_attempts_gpu\": %llu, \"image_mean\": %.6e}\n",
                frac, mr, frac_t, cnt_diff, (unsigned long long)att_cpu, (unsigned long long)att_gpu,
                cpu.image.mean());
    bool ok = frac >= 0.999 && frac_t >= 0.999 && cnt_diff == 0 && att_cpu == att_gpu && cpu.image.mean() > 0;
    return ok ? 0 : 1;
}
