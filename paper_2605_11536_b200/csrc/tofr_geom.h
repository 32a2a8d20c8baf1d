// tofr_geom.h -- device-resident frame layout, BVH traversal, materials,
// lights and camera.  Host (g++) and device (nvcc) share this code so the
// collimated-beam trace done on the host matches the device traversal.
//
// Reference behaviour restated here:
//   geometry.hpp:86-119   ray_box slab test, two-sided Moller-Trumbore
//   geometry.hpp:168-231  closest-hit / any-hit stack traversal (push left,
//                         push right, pop right first; first-found wins ties)
//   scene.hpp:32-155      oriented normals, GGX/Lambert/mirror eval/pdf/sample
//   scene.hpp:178-190     delta light sample (1/d^2 inside the cone)
//   scene.hpp:375-405     pixel-centre primary ray, world->pixel projection
//
// Layout (B200-first): the BVH is a *threaded* tree.  Each node carries the
// index of the next node in the reference's visiting order when the box is
// hit (first child popped = right child) and when it is missed or finished
// (escape link).  This reproduces the reference stack order exactly with no
// per-thread stack, so traversal needs no local memory.  Triangles are stored
// in leaf order (tri_order) as {v0, e1, e2} = 72 B records for the
// intersection loop; the rarely read attributes live in a separate array.
#pragma once

#include "tofr_core.h"

namespace tofr_b200 {

enum : int { MAT_DIFFUSE = 0, MAT_GLOSSY = 1, MAT_MIRROR = 2 };
enum : int { LIGHT_COLLIMATED = 0, LIGHT_WIDE = 1 };

struct GNode {            // 64 B, traversal view
    double lo[3], hi[3];  // AABB
    int hit_next;         // internal: right child; leaf: escape
    int miss_next;        // escape link (-1 ends traversal)
    int first, count;     // leaf range in tri_order (count == 0: internal)
};

struct GNodeAux {  // 32 B, ellipsoid-descent view (ellipsoid.hpp:310-380)
    double tri_area;
    int left, right, parent, first, count, pad;
};

struct GTriIsect {  // 72 B, leaf order
    V3 v0, e1, e2;
};

struct GTriInfo {  // 64 B, indexed by original triangle id
    V3 n;
    int mat, obj;
    double area;
    int leaf;       // leaf_of_tri (geometry.hpp:149-153)
    int leaf_slot;  // position of this triangle in leaf order (tri_isect)
    double pad2;
};

struct GMat {
    int kind;
    int reconnectable;  // scene.hpp:26-28
    V3 albedo;
    double roughness;
    double alpha;  // ggx::alpha_of(roughness), scene.hpp:40
};

struct GCam {
    V3 pos, fwd, right, up;
    double tan_half;
    int w, h;
};

struct GLight {
    V3 pos, dir, intensity;
    double cone_half_angle;
    double cos_cone;  // std::cos(cone_half_angle), evaluated by the host libm
    int regime;
    int pad;
};

struct GLightSub {  // scene.hpp:433-440
    int valid;
    int tri, obj, mat;
    V3 pos, n, wo_light, power;
    double chain_len;
};

// Affine velocity field v(x) = A x + c of one object at one frame
// (VelocityField, scene.hpp:308-335); zero when the object does not move.
struct GVel {
    M3 A;
    V3 c;
    int moving;
    int pad;
};

// One frame snapshot as seen by the kernels (SceneFrame, scene.hpp:443-471).
struct FrameView {
    const GNode* nodes;
    const GNodeAux* aux;
    const GTriIsect* tri_isect;  // leaf order
    const int* tri_id;           // leaf slot -> triangle id (tri_order)
    const GTriInfo* tri;         // by triangle id
    const GMat* mats;
    int n_nodes, n_tris, n_mats;
    int geo_motion;  // any object velocity field "moving" (shiftmap.hpp:675-682)
    GCam cam;
    GLight light;
    GLightSub lsub;
    double eps_ray, diag;
    int frame_id;  // identity of the snapshot (Domain::frame pointer compare)
    int n_obj;
    const GVel* vel;  // per object (n_obj)
    const Frame2* tframe;  // tangent_frame per triangle id
    V3 cam_vel;       // central difference of the camera track (scene.hpp:508-513)
};

// SceneFrame::velocity_at (scene.hpp:457-460): A * world + c, or 0
TOFR_HD V3 velocity_at(const FrameView& f, int obj, const V3& p) {
    if (obj < 0 || obj >= f.n_obj) return splat(0);
    const GVel& v = f.vel[obj];
    if (!v.moving) return splat(0);
    return v.A * p + v.c;
}

// ---------------------------------------------------------------------------
// intersection

struct Hit {
    V3 pos;
    double t;
    int tri;
};

// geometry.hpp:86-96
TOFR_HD bool ray_box(const V3& o, const V3& inv, const GNode& n, double tmin, double tmax) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double oa = comp(o, a), ia = comp(inv, a);
        double t0 = (n.lo[a] - oa) * ia;
        double t1 = (n.hi[a] - oa) * ia;
        if (ia < 0) {
            double s = t0;
            t0 = t1;
            t1 = s;
        }
        tmin = dmax(tmin, t0);
        tmax = dmin(tmax, t1);
        if (tmax < tmin) return false;
    }
    return true;
}

// geometry.hpp:99-119
TOFR_HD bool ray_tri(const V3& o, const V3& d, const GTriIsect& tr, double tmin, double tmax,
                     double& t_out) {
    V3 pv = cross(d, tr.e2);
    double dt = dot(tr.e1, pv);
    if (fabs(dt) < 1e-16) return false;
    double inv_det = 1.0 / dt;
    V3 tv = o - tr.v0;
    double u = dot(tv, pv) * inv_det;
    if (u < -1e-12 || u > 1 + 1e-12) return false;
    V3 qv = cross(tv, tr.e1);
    double v = dot(d, qv) * inv_det;
    if (v < -1e-12 || u + v > 1 + 1e-12) return false;
    double t = dot(tr.e2, qv) * inv_det;
    if (t <= tmin || t >= tmax) return false;
    t_out = t;
    return true;
}

// Closest hit on (tmin, tmax); Bvh::intersect_min (geometry.hpp:168-201).
// The traversal bodies are out-of-line on the device (one copy per kernel,
// arguments in registers) so that the many call sites of the reuse kernels
// do not blow up the instruction footprint.
struct TraceHit {
    double t;
    int slot;
};

TOFR_HD TraceHit trace_closest_impl(const GNode* nodes, const GTriIsect* tris, const V3& o, const V3& d,
                                    double tmin, double tmax) {
    V3 inv = V3{1.0 / d.x, 1.0 / d.y, 1.0 / d.z};
    double best = tmax;
    int best_slot = -1;
    int ni = 0;
    while (ni >= 0) {
        const GNode& n = nodes[ni];
        if (!ray_box(o, inv, n, tmin, best)) {
            ni = n.miss_next;
            continue;
        }
        if (n.count > 0) {
            for (int i = 0; i < n.count; ++i) {
                double t;
                if (ray_tri(o, d, tris[n.first + i], tmin, best, t)) {
                    best = t;
                    best_slot = n.first + i;
                }
            }
        }
        ni = n.hit_next;
    }
    return TraceHit{best, best_slot};
}

TOFR_HD bool trace_any_impl(const GNode* nodes, const GTriIsect* tris, const V3& o, const V3& d, double tmin,
                            double tmax) {
    V3 inv = V3{1.0 / d.x, 1.0 / d.y, 1.0 / d.z};
    int ni = 0;
    while (ni >= 0) {
        const GNode& n = nodes[ni];
        if (!ray_box(o, inv, n, tmin, tmax)) {
            ni = n.miss_next;
            continue;
        }
        for (int i = 0; i < n.count; ++i) {
            double t;
            if (ray_tri(o, d, tris[n.first + i], tmin, tmax, t)) return true;
        }
        ni = n.hit_next;
    }
    return false;
}

// One traversal for both ray kinds: closest hit (any = false) or the first hit
// on the segment (any = true; Bvh::occluded keeps t_max fixed and returns at
// the first hit, which is what the unshrunk `best` gives until that hit).
// Lets a kernel trace shadow and extension rays of different lanes together.
TOFR_HD TraceHit trace_ray_impl(const GNode* nodes, const GTriIsect* tris, const V3& o, const V3& d, double tmin,
                                double tmax, bool any) {
    V3 inv = V3{1.0 / d.x, 1.0 / d.y, 1.0 / d.z};
    double best = tmax;
    int best_slot = -1;
    int ni = 0;
    while (ni >= 0) {
        const GNode& n = nodes[ni];
        if (!ray_box(o, inv, n, tmin, best)) {
            ni = n.miss_next;
            continue;
        }
        for (int i = 0; i < n.count; ++i) {
            double t;
            if (ray_tri(o, d, tris[n.first + i], tmin, best, t)) {
                best = t;
                best_slot = n.first + i;
                if (any) return TraceHit{best, best_slot};
            }
        }
        ni = n.hit_next;
    }
    return TraceHit{best, best_slot};
}

#if defined(__CUDACC__)
static __device__ __noinline__ TraceHit trace_closest_dev(const GNode* nodes, const GTriIsect* tris, V3 o, V3 d,
                                                   double tmin, double tmax) {
    return trace_closest_impl(nodes, tris, o, d, tmin, tmax);
}
static __device__ __noinline__ bool trace_any_dev(const GNode* nodes, const GTriIsect* tris, V3 o, V3 d, double tmin,
                                           double tmax) {
    return trace_any_impl(nodes, tris, o, d, tmin, tmax);
}
#endif

TOFR_HD bool trace_closest(const FrameView& f, const V3& o, const V3& d, double tmin, double tmax,
                           Hit& hit) {
#if defined(__CUDA_ARCH__)
    TraceHit r = trace_closest_dev(f.nodes, f.tri_isect, o, d, tmin, tmax);
#else
    TraceHit r = trace_closest_impl(f.nodes, f.tri_isect, o, d, tmin, tmax);
#endif
    if (r.slot < 0) return false;
    hit.t = r.t;
    hit.tri = f.tri_id[r.slot];
    hit.pos = o + d * r.t;
    return true;
}

TOFR_HD bool trace_any(const FrameView& f, const V3& o, const V3& d, double tmin, double tmax) {
#if defined(__CUDA_ARCH__)
    return trace_any_dev(f.nodes, f.tri_isect, o, d, tmin, tmax);
#else
    return trace_any_impl(f.nodes, f.tri_isect, o, d, tmin, tmax);
#endif
}

// Bvh::intersect: t_min = eps_ray, t_max = inf (geometry.hpp:164-166)
TOFR_HD bool intersect(const FrameView& f, const V3& o, const V3& d, Hit& hit) {
    return trace_closest(f, o, d, f.eps_ray, kInf, hit);
}

// Bvh::occluded: open segment (a,b) shrunk by eps_ray at both ends
// (geometry.hpp:205-231)
TOFR_HD bool occluded(const FrameView& f, const V3& a, const V3& b) {
    V3 dd = b - a;
    double dist = norm(dd);
    if (dist <= 2 * f.eps_ray) return false;
    V3 d = dd / dist;
    return trace_any(f, a, d, f.eps_ray, dist - f.eps_ray);
}

// ---------------------------------------------------------------------------
// materials (scene.hpp:32-155)

TOFR_HD V3 oriented_normal(const V3& n, const V3& toward) { return dot(n, toward) >= 0 ? n : -n; }
TOFR_HD V3 reflect(const V3& w, const V3& n) { return n * (2.0 * dot(n, w)) - w; }

TOFR_HD double ggx_ndf(double cos_h, double alpha) {
    double a2 = alpha * alpha;
    double d = cos_h * cos_h * (a2 - 1.0) + 1.0;
    return a2 / (kPi * d * d);
}
TOFR_HD double ggx_g1(double cos_v, double alpha) {
    double a2 = alpha * alpha;
    return 2.0 * cos_v / (cos_v + sqrt(a2 + (1.0 - a2) * cos_v * cos_v));
}

TOFR_HD V3 eval_bsdf(const GMat& m, const V3& n_geo, const V3& wi, const V3& wo) {
    V3 n = oriented_normal(n_geo, wi);
    double ci = dot(n, wi), co = dot(n, wo);
    if (ci <= 0 || co <= 0) return splat(0);
    if (m.kind == MAT_DIFFUSE) return m.albedo * (1.0 / kPi);
    if (m.kind == MAT_GLOSSY) {
        V3 h = normalize(wi + wo);
        double a = m.alpha;
        double d = ggx_ndf(dot(n, h), a);
        double g = ggx_g1(ci, a) * ggx_g1(co, a);
        return m.albedo * (d * g / (4.0 * ci * co));
    }
    return splat(0);
}

TOFR_HD double pdf_bsdf(const GMat& m, const V3& n_geo, const V3& wi, const V3& wo) {
    V3 n = oriented_normal(n_geo, wi);
    double ci = dot(n, wi), co = dot(n, wo);
    if (ci <= 0 || co <= 0) return 0;
    if (m.kind == MAT_DIFFUSE) return co / kPi;
    if (m.kind == MAT_GLOSSY) {
        V3 h = normalize(wi + wo);
        double a = m.alpha;
        double doth = dot(wi, h);
        if (doth <= 0) return 0;
        return ggx_ndf(dot(n, h), a) * dot(n, h) / (4.0 * doth);
    }
    return 0;
}

struct BsdfSample {
    V3 wo;
    double pdf;
    bool is_delta, valid;
};

// sample_bsdf (scene.hpp:105-155).  The returned weight is not used by the
// transport code, so it is not computed.
TOFR_HD BsdfSample sample_bsdf(const GMat& m, const V3& n_geo, const V3& wi, Rng& rng) {
    BsdfSample s;
    s.pdf = 0;
    s.is_delta = false;
    s.valid = false;
    s.wo = splat(0);
    V3 n = oriented_normal(n_geo, wi);
    if (dot(n, wi) <= 0) return s;
    if (m.kind == MAT_DIFFUSE) {
        double u1 = rng_next(rng), u2 = rng_next(rng);
        double cos_t = sqrt(u1), sin_t = sqrt(dmax(0.0, 1.0 - u1));
        double phi = 2.0 * kPi * u2;
        V3 t, b;
        onb(n, t, b);
        s.wo = t * (sin_t * cos(phi)) + b * (sin_t * sin(phi)) + n * cos_t;
        s.pdf = cos_t / kPi;
        if (s.pdf <= 0) return s;
        s.valid = true;
        return s;
    }
    if (m.kind == MAT_GLOSSY) {
        double a = m.alpha;
        double u1 = rng_next(rng), u2 = rng_next(rng);
        double cos_h = sqrt((1.0 - u1) / (1.0 + (a * a - 1.0) * u1));
        double sin_h = sqrt(dmax(0.0, 1.0 - cos_h * cos_h));
        double phi = 2.0 * kPi * u2;
        V3 t, b;
        onb(n, t, b);
        V3 h = t * (sin_h * cos(phi)) + b * (sin_h * sin(phi)) + n * cos_h;
        V3 wo = reflect(wi, h);
        double co = dot(n, wo);
        if (co <= 0) return s;
        double doth = dot(wi, h);
        if (doth <= 0) return s;
        s.wo = wo;
        s.pdf = ggx_ndf(cos_h, a) * cos_h / (4.0 * doth);
        if (s.pdf <= 0) return s;
        s.valid = true;
        return s;
    }
    // mirror
    s.wo = reflect(wi, n);
    s.pdf = 1.0;
    s.is_delta = true;
    s.valid = true;
    return s;
}

// ---------------------------------------------------------------------------
// lights (scene.hpp:178-190)

struct LightSample {
    V3 dir;  // target -> light
    double dist;
    V3 value;
};

TOFR_HD bool light_sample(const GLight& l, const V3& target, LightSample& s) {
    if (l.regime == LIGHT_COLLIMATED) return false;
    V3 to_target = target - l.pos;
    double d = norm(to_target);
    if (d <= 0) return false;
    V3 w = to_target / d;
    if (dot(w, l.dir) < l.cos_cone) return false;
    s.dir = -w;
    s.dist = d;
    s.value = l.intensity / (d * d);
    return true;
}

// geom_term (transport.hpp:86-93)
TOFR_HD double geom_term(const V3& a, const V3& na, const V3& b, const V3& nb) {
    V3 d = b - a;
    double d2 = norm2(d);
    if (d2 <= 0) return 0;
    double dist = sqrt(d2);
    V3 w = d / dist;
    return fabs(dot(na, w)) * fabs(dot(nb, w)) / d2;
}

// ---------------------------------------------------------------------------
// camera (scene.hpp:386-405)

TOFR_HD V3 primary_dir(const GCam& c, int x, int y) {
    double aspect = double(c.w) / double(c.h);
    double px = (2.0 * (x + 0.5) / c.w - 1.0) * c.tan_half * aspect;
    double py = (1.0 - 2.0 * (y + 0.5) / c.h) * c.tan_half;
    return normalize(c.fwd + c.right * px + c.up * py);
}

TOFR_HD bool project(const GCam& c, const V3& world, int& ox, int& oy) {
    V3 d = world - c.pos;
    double z = dot(d, c.fwd);
    if (z <= 0) return false;
    double aspect = double(c.w) / double(c.h);
    double px = dot(d, c.right) / z / (c.tan_half * aspect);
    double py = dot(d, c.up) / z / c.tan_half;
    double fx = floor((px + 1.0) * 0.5 * c.w);
    double fy = floor((1.0 - py) * 0.5 * c.h);
    // out-of-range conversions are rejected explicitly (the reference relies
    // on x86 cvttsd2si returning INT_MIN)
    if (!(fx >= 0 && fx < c.w && fy >= 0 && fy < c.h)) return false;
    ox = int(fx);
    oy = int(fy);
    return true;
}

// ---------------------------------------------------------------------------
// gates (transport.hpp:17-59, 100-127)

TOFR_HD double gate_w(double center, double width, double len) {
    return fabs(len - center) <= width / 2 ? 1.0 : 0.0;
}

struct HistSpec {
    int bins;
    double t0, bw;
};

TOFR_HD int bin_of(const HistSpec& h, double len) {
    if (len < h.t0 || len > h.t0 + h.bins * h.bw) return -1;
    int b = int((len - h.t0) / h.bw);
    return b < h.bins - 1 ? b : h.bins - 1;  // closed final bin
}
// bin_gate(b) = {t0 + (b + 0.5) * bw, bw}
TOFR_HD double bin_center(const HistSpec& h, int b) { return h.t0 + (b + 0.5) * h.bw; }

}  // namespace tofr_b200
