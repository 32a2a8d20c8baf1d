// tofr_ellipsoid.cuh -- path-length-constrained connection sampler: insert a
// vertex q on the constant-length prolate spheroid |q-x_d| + |q-L| = l_rem so
// the completed path lands exactly on the gate centre.
//
// Reference (restated, Length gate):
//   ellipsoid.hpp:22-37    ellipsoid_from_constraint
//   ellipsoid.hpp:46-80    unit-sphere frame, conservative node_overlaps
//   ellipsoid.hpp:128-135  32-point Gauss-Legendre integration (nodes built on
//                          the host exactly as Rule32 does and kept in
//                          constant memory)
//   ellipsoid.hpp:167-269  clip_ellipsoid_triangle (plane conic clipped to
//                          the triangle: <= 6 cut angles, <= 6 arc segments)
//   ellipsoid.hpp:273-296  sample_arc (arc-length bisection, <= 60 steps)
//   ellipsoid.hpp:310-380  area-weighted BVH descent and its pdf
//   transport.hpp:332-444  emit_ellipsoidal, ell_pdf_at, ell_length_gradient
#pragma once

#include "tofr_kernels.h"
#include "tofr_path.cuh"

namespace tofr_b200 {

#if defined(__CUDACC__)

__constant__ double c_gl_x[32];
__constant__ double c_gl_w[32];

struct Ellipsoid {
    V3 f1, f2, center, axis, w1, w2;  // w1, w2: onb(axis), hoisted out of every corner test
    double ell, a, b;
    M3 M;
};

__device__ inline bool ellipsoid_from_constraint(const V3& f1, const V3& f2, double ell, Ellipsoid& e) {
    double d = norm(f2 - f1);
    if (!(ell > d) || !(ell > 0)) return false;
    e.f1 = f1;
    e.f2 = f2;
    e.ell = ell;
    e.center = (f1 + f2) * 0.5;
    e.axis = d > 1e-12 * ell ? (f2 - f1) / d : V3{1, 0, 0};
    e.a = ell / 2;
    e.b = sqrt(dmax(0.0, e.a * e.a - d * d / 4));
    M3 aa = m3_outer(e.axis, e.axis);
    e.M = aa * (1.0 / (e.a * e.a)) + (m3_identity() - aa) * (1.0 / (e.b * e.b));
    onb(e.axis, e.w1, e.w2);
    return true;
}

__device__ inline bool node_overlaps(const Ellipsoid& e, const double lo[3], const double hi[3]) {
    double max2 = 0;
    V3 hlo{kInf, kInf, kInf}, hhi{-kInf, -kInf, -kInf};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        V3 c{(i & 1) ? hi[0] : lo[0], (i & 2) ? hi[1] : lo[1], (i & 4) ? hi[2] : lo[2]};
        V3 d = c - e.center;
        V3 u{dot(e.axis, d) / e.a, dot(e.w1, d) / e.b, dot(e.w2, d) / e.b};
        max2 = dmax(max2, norm2(u));
        hlo = vmin(hlo, u);
        hhi = vmax(hhi, u);
    }
    if (max2 < 1.0) return false;
    double min2 = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double l = comp(hlo, a), h = comp(hhi, a);
        double d = l > 0 ? l : (h < 0 ? -h : 0);
        min2 += d * d;
    }
    return min2 <= 1.0;
}

__device__ inline bool node_overlaps_i(const FrameView& F, const Ellipsoid& e, int ni) {
    const GNode& n = F.nodes[ni];
    return node_overlaps(e, n.lo, n.hi);
}

struct ConicArc {
    V3 origin;
    Frame2 frame;
    V2 center, ax1, ax2;
    double r1, r2;
    double t0[6], t1[6], len[6];
    int nseg;
    double total_len;
};

__device__ inline V2 arc_point2(const ConicArc& a, double th) {
    return a.center + a.ax1 * (a.r1 * cos(th)) + a.ax2 * (a.r2 * sin(th));
}
__device__ inline double arc_speed(const ConicArc& a, double th) {
    V2 d = a.ax1 * (-a.r1 * sin(th)) + a.ax2 * (a.r2 * cos(th));
    return norm(d);
}
__device__ inline double arc_integrate(const ConicArc& arc, double a, double b) {
    double mid = 0.5 * (a + b), half = 0.5 * (b - a);
    double s = 0;
    for (int i = 0; i < 32; ++i) s += c_gl_w[i] * arc_speed(arc, mid + half * c_gl_x[i]);
    return s * half;
}

struct HalfPlane {
    V2 n;
    double c;
};

__device__ inline HalfPlane make_edge(const V2& a, const V2& b, const V2& inside) {
    V2 n = rot90(b - a);
    double c = dot(n, a);
    if (dot(n, inside) < c) {
        n = -n;
        c = -c;
    }
    return HalfPlane{n, c};
}

__device__ inline bool arc_inside(const ConicArc& arc, const HalfPlane* edges, double th) {
    V2 q = arc_point2(arc, th);
    for (int i = 0; i < 3; ++i)
        if (dot(edges[i].n, q) < edges[i].c - 1e-12) return false;
    return true;
}

// clip_ellipsoid_triangle (ellipsoid.hpp:167-269), split in two: the conic,
// its cut angles and the kept segments [t0, t1] (clip_geometry), then the
// segments' arc lengths (arc_lengths: the 32-point Gauss-Legendre integrals,
// the expensive part).  A kept segment's length is always > 0 (the integrand
// |d/dth arc| >= min(r1, r2) > 0 and t1 - t0 >= 1e-12), so the reference's
// `len <= 0` skip never fires and the segment list is fixed by the geometry.
__device__ bool clip_geometry(const FrameView& F, const Ellipsoid& e, int tri, ConicArc& arc) {
    const GTriIsect& g = tri_geo(F, tri);
    arc.origin = g.v0;
    arc.frame = tangent_frame(F, tri);
    const V3 T = arc.frame.t, B = arc.frame.b;
    V3 d0 = g.v0 - e.center;
    V3 MT = e.M * T, MB = e.M * B, Md = e.M * d0;
    M2 Q{dot(T, MT), dot(T, MB), dot(B, MT), dot(B, MB)};
    V2 L{dot(T, Md), dot(B, Md)};
    double k = dot(d0, Md) - 1.0;
    V2 h;
    if (!solve2x2(Q, -L, h)) return false;
    double fh = dot(h, Q * h) + 2.0 * dot(L, h) + k;
    double rho = -fh;
    if (!(rho > 0)) return false;
    double tr = Q.a + Q.d, dt = det(Q);
    double disc = sqrt(dmax(0.0, tr * tr / 4 - dt));
    double l1 = tr / 2 + disc, l2 = tr / 2 - disc;
    if (!(l2 > 0)) return false;
    V2 c1{Q.b, l1 - Q.a};
    V2 c2{l1 - Q.d, Q.c};
    V2 v1 = norm(c1) >= norm(c2) ? c1 : c2;
    double nv = norm(v1);
    v1 = nv > 1e-14 * dmax(fabs(l1), 1e-30) ? v1 * (1.0 / nv) : V2{1, 0};
    arc.center = h;
    arc.ax1 = v1;
    arc.ax2 = rot90(v1);
    arc.r1 = sqrt(rho / l1);
    arc.r2 = sqrt(rho / l2);

    V2 p0{0, 0};
    V2 p1 = to_local(arc.frame, g.e1);
    V2 p2 = to_local(arc.frame, g.e2);
    HalfPlane edges[3] = {make_edge(p0, p1, p2), make_edge(p1, p2, p0), make_edge(p2, p0, p1)};

    double cuts[6];
    int nc = 0;
    for (int i = 0; i < 3; ++i) {
        double A = dot(edges[i].n, arc.ax1) * arc.r1;
        double B2 = dot(edges[i].n, arc.ax2) * arc.r2;
        double C = dot(edges[i].n, arc.center) - edges[i].c;
        double R = hypot(A, B2);
        if (R < fabs(C) || R < 1e-300) continue;
        double base = atan2(B2, A);
        double x = -C / R;
        x = x < -1.0 ? -1.0 : (x > 1.0 ? 1.0 : x);
        double off = acos(x);
        cuts[nc++] = base + off;
        cuts[nc++] = base - off;
    }
    for (int i = 0; i < nc; ++i) {
        double c = fmod(cuts[i], 2 * kPi);
        if (c < 0) c += 2 * kPi;
        cuts[i] = c;
    }
    for (int i = 1; i < nc; ++i) {  // insertion sort (values only)
        double v = cuts[i];
        int j = i - 1;
        while (j >= 0 && cuts[j] > v) {
            cuts[j + 1] = cuts[j];
            --j;
        }
        cuts[j + 1] = v;
    }
    arc.nseg = 0;
    arc.total_len = 0;
    auto add_seg = [&](double t0, double t1) {
        if (t1 - t0 < 1e-12) return;
        double mid = 0.5 * (t0 + t1);
        if (!arc_inside(arc, edges, mid)) return;
        arc.t0[arc.nseg] = t0;
        arc.t1[arc.nseg] = t1;
        arc.nseg++;
    };
    if (nc == 0) {
        if (!arc_inside(arc, edges, 0)) return false;
        add_seg(0, 2 * kPi);
    } else {
        for (int i = 0; i < nc; ++i) {
            double t0 = cuts[i];
            double t1 = i + 1 < nc ? cuts[i + 1] : cuts[0] + 2 * kPi;
            add_seg(t0, t1);
        }
    }
    return arc.nseg > 0;
}

__device__ inline void arc_lengths(ConicArc& arc) {
    arc.total_len = 0;
    for (int i = 0; i < arc.nseg; ++i) {
        arc.len[i] = arc_integrate(arc, arc.t0[i], arc.t1[i]);
        arc.total_len += arc.len[i];
    }
}

__device__ bool clip_ellipsoid_triangle(const FrameView& F, const Ellipsoid& e, int tri, ConicArc& arc) {
    if (!clip_geometry(F, e, tri, arc)) return false;
    arc_lengths(arc);
    return arc.total_len > 0;
}

// sample_arc (ellipsoid.hpp:273-296)
__device__ V3 sample_arc(const ConicArc& arc, Rng& rng, double& pdf_len) {
    double target = rng_next(rng) * arc.total_len;
    int si = arc.nseg - 1;
    for (int i = 0; i < arc.nseg; ++i) {
        if (target <= arc.len[i] || i == arc.nseg - 1) {
            si = i;
            break;
        }
        target -= arc.len[i];
    }
    double sl = arc.len[si];
    target = target < 0.0 ? 0.0 : (target > sl ? sl : target);
    double lo = arc.t0[si], hi = arc.t1[si];
    for (int it = 0; it < 60; ++it) {
        double mid = 0.5 * (lo + hi);
        double l = arc_integrate(arc, arc.t0[si], mid);
        if (l < target)
            lo = mid;
        else
            hi = mid;
        if ((hi - lo) * arc_speed(arc, 0.5 * (lo + hi)) < 1e-6 * dmax(arc.total_len, 1e-30)) break;
    }
    pdf_len = 1.0 / arc.total_len;
    return arc.origin + to_world(arc.frame, arc_point2(arc, 0.5 * (lo + hi)));
}

struct EllSample {
    V3 pos;
    int tri;
    double pdf_arc;
};

// area-weighted BVH descent + triangle pick of sample_connection_vertex
// (ellipsoid.hpp:310-340): the triangle and p_desc * p_tri
__device__ bool descend_pick(const FrameView& F, const Ellipsoid& e, Rng& rng, int& tri_out, double& p_dt) {
    if (!node_overlaps_i(F, e, 0)) return false;
    double p_desc = 1.0;
    int ni = 0;
    while (F.aux[ni].count == 0) {
        int li = F.aux[ni].left, ri = F.aux[ni].right;
        double wl = node_overlaps_i(F, e, li) ? F.aux[li].tri_area : 0.0;
        double wr = node_overlaps_i(F, e, ri) ? F.aux[ri].tri_area : 0.0;
        double sum = wl + wr;
        if (sum <= 0) return false;
        if (rng_next(rng) * sum < wl) {
            p_desc *= wl / sum;
            ni = li;
        } else {
            p_desc *= wr / sum;
            ni = ri;
        }
    }
    const GNodeAux& leaf = F.aux[ni];
    double pick = rng_next(rng) * leaf.tri_area;
    int tri_id = F.tri_id[leaf.first];
    double acc = 0;
    for (int i = 0; i < leaf.count; ++i) {
        int id = F.tri_id[leaf.first + i];
        acc += F.tri[id].area;
        if (pick <= acc || i == leaf.count - 1) {
            tri_id = id;
            break;
        }
    }
    double p_tri = F.tri[tri_id].area / leaf.tri_area;
    tri_out = tri_id;
    p_dt = p_desc * p_tri;
    return true;
}

// sample_connection_vertex (ellipsoid.hpp:310-352)
__device__ bool sample_connection_vertex(const FrameView& F, const Ellipsoid& e, Rng& rng, EllSample& s) {
    if (!node_overlaps_i(F, e, 0)) return false;
    double p_desc = 1.0;
    int ni = 0;
    while (F.aux[ni].count == 0) {
        int li = F.aux[ni].left, ri = F.aux[ni].right;
        double wl = node_overlaps_i(F, e, li) ? F.aux[li].tri_area : 0.0;
        double wr = node_overlaps_i(F, e, ri) ? F.aux[ri].tri_area : 0.0;
        double sum = wl + wr;
        if (sum <= 0) return false;
        if (rng_next(rng) * sum < wl) {
            p_desc *= wl / sum;
            ni = li;
        } else {
            p_desc *= wr / sum;
            ni = ri;
        }
    }
    const GNodeAux& leaf = F.aux[ni];
    double pick = rng_next(rng) * leaf.tri_area;
    int tri_id = F.tri_id[leaf.first];
    double acc = 0;
    for (int i = 0; i < leaf.count; ++i) {
        int id = F.tri_id[leaf.first + i];
        acc += F.tri[id].area;
        if (pick <= acc || i == leaf.count - 1) {
            tri_id = id;
            break;
        }
    }
    double p_tri = F.tri[tri_id].area / leaf.tri_area;
    ConicArc arc;
    if (!clip_ellipsoid_triangle(F, e, tri_id, arc)) return false;
    double pdf_len;
    s.pos = sample_arc(arc, rng, pdf_len);
    s.tri = tri_id;
    s.pdf_arc = p_desc * p_tri * pdf_len;
    return true;
}

// eval_connection_pdf (ellipsoid.hpp:356-380)
__device__ double eval_connection_pdf(const FrameView& F, const Ellipsoid& e, int tri_id) {
    int leaf_idx = F.tri[tri_id].leaf;
    if (leaf_idx < 0) return 0;
    double p_desc = 1.0;
    int ni = leaf_idx;
    while (F.aux[ni].parent >= 0) {
        int pi = F.aux[ni].parent;
        int li = F.aux[pi].left, ri = F.aux[pi].right;
        double wl = node_overlaps_i(F, e, li) ? F.aux[li].tri_area : 0.0;
        double wr = node_overlaps_i(F, e, ri) ? F.aux[ri].tri_area : 0.0;
        double sum = wl + wr;
        double mine = (li == ni) ? wl : wr;
        if (mine <= 0 || sum <= 0) return 0;
        p_desc *= mine / sum;
        ni = pi;
    }
    if (!node_overlaps_i(F, e, 0)) return 0;
    double p_tri = F.tri[tri_id].area / F.aux[leaf_idx].tri_area;
    ConicArc arc;
    if (!clip_ellipsoid_triangle(F, e, tri_id, arc)) return 0;
    return p_desc * p_tri / arc.total_len;
}

__device__ inline double ell_length_gradient(const Ellipsoid& e, const V3& q, const V3& n) {
    V3 s = normalize(e.f1 - q) + normalize(e.f2 - q);
    V3 in_plane = s - n * dot(n, s);
    return norm(in_plane);
}

// ell_pdf_at (transport.hpp:419-438): density of the ellipsoidal strategy
// producing the vertex at qpos on qtri from the prefix ending at `at`.
__device__ double ell_pdf_at(const FrameView& F, const PathCfg& cfg, const WalkV& at, const V3& qpos,
                             int qtri, double total_len) {
    if (cfg.ell_width <= 0) return 0;
    if (gate_w(cfg.ell_center, cfg.ell_width, total_len) <= 0) return 0;
    V3 lpos;
    if (F.light.regime == LIGHT_WIDE) {
        lpos = F.light.pos;
    } else {
        if (!F.lsub.valid) return 0;
        lpos = F.lsub.pos;
    }
    double two_seg = norm(qpos - at.p) + norm(lpos - qpos);
    Ellipsoid e;
    if (!ellipsoid_from_constraint(at.p, lpos, two_seg, e)) return 0;
    double pdf_arc = eval_connection_pdf(F, e, qtri);
    if (pdf_arc <= 0) return 0;
    double grad = ell_length_gradient(e, qpos, F.tri[qtri].n);
    if (grad <= 0) return 0;
    return pdf_arc * grad / cfg.ell_width;
}

// ---------------------------------------------------------------------------
// Wavefront ellipsoidal sampling (three launches instead of one per-lane
// sample_connection_vertex):
//   plan   (k_ell_plan)   the path trees' walks; every ellipsoidal step runs its
//                         BVH descent + triangle pick (the ellipsoid RNG draws)
//                         and the conic clip GEOMETRY, draws the arc target and
//                         records a job; no candidates, no NEE rays.
//   arcs   (k_ell_arcs)   one warp per job: the segment lengths and the <= 60
//                         bisection steps of sample_arc, each 32-point
//                         Gauss-Legendre integral with one node per lane and
//                         the terms summed in the reference's order.
//   replay (k_init_gated) the RIS initialisation with the jobs' vertices in
//                         place of sample_connection_vertex (the ellipsoid RNG
//                         counter restored from the plan).
// Every value is computed by the same operations as the per-lane sampler, so
// the vertices and pdfs are bit-identical to it (and to the reference's).

struct DirectSampler {
    __device__ bool sample(const FrameView& F, const Ellipsoid& e, Rng& rng, EllSample& q) {
        return sample_connection_vertex(F, e, rng, q);
    }
};

struct PlanSampler {
    EllScratch es;
    size_t slot0;
    int k;
    __device__ bool sample(const FrameView& F, const Ellipsoid& e, Rng& rng, EllSample&) {
        size_t slot = slot0 + size_t(k++);
        int tri = -1;
        double p_dt = 0;
        ConicArc arc;
        bool ok = descend_pick(F, e, rng, tri, p_dt) && clip_geometry(F, e, tri, arc);
        if (ok) {
            EllJob& j = es.jobs[slot];
            j.center = arc.center;
            j.ax1 = arc.ax1;
            j.ax2 = arc.ax2;
            j.r1 = arc.r1;
            j.r2 = arc.r2;
            for (int i = 0; i < arc.nseg; ++i) {
                j.t0[i] = arc.t0[i];
                j.t1[i] = arc.t1[i];
            }
            j.nseg = arc.nseg;
            j.tri = tri;
            j.p_dt = p_dt;
            j.u = rng_next(rng);
            es.list[atomicAdd(es.count, 1u)] = uint32_t(slot);
        }
        es.st[slot] = ok ? 1 : 0;
        es.ctr[slot] = rng.ctr;
        return false;  // the plan emits nothing
    }
};

struct ReplaySampler {
    EllScratch es;
    size_t slot0;
    int k;
    __device__ bool sample(const FrameView&, const Ellipsoid&, Rng& rng, EllSample& q) {
        size_t slot = slot0 + size_t(k++);
        rng.ctr = es.ctr[slot];
        if (!es.st[slot]) return false;
        EllRes r = es.res[slot];
        q.pos = r.pos;
        q.tri = es.jobs[slot].tri;
        q.pdf_arc = r.pdf_arc;
        return true;
    }
};

// emit_ellipsoidal (transport.hpp:332-415) as a walk hook.
template <class Sampler>
struct EllStepT {
    Sampler smp;
    __device__ double pdf_at(const FrameView& F, const PathCfg& cfg, const WalkV& at, const V3& qpos,
                             int qtri, double total_len) {
        return ell_pdf_at(F, cfg, at, qpos, qtri, total_len);
    }
    template <class Sink>
    __device__ void step(const FrameView& F, const PathCfg& cfg, const WalkV* v, int d, Rng& rng,
                         uint64_t lane_key, Sink& sink) {
        if (d + 2 > cfg.max_depth) return;
        const WalkV& x = v[d];
        V3 lpos;
        double suffix_len = 0;
        const bool wide = F.light.regime == LIGHT_WIDE;
        if (wide) {
            lpos = F.light.pos;
        } else {
            if (!F.lsub.valid) return;
            lpos = F.lsub.pos;
            suffix_len = F.lsub.chain_len;
        }
        double l_rem = cfg.ell_center - x.len - suffix_len;
        Ellipsoid e;
        if (!ellipsoid_from_constraint(x.p, lpos, l_rem, e)) return;
        EllSample q;
        if (!smp.sample(F, e, rng, q)) return;  // consumes the ellipsoid lane
        const GTriInfo& qt = F.tri[q.tri];
        const GMat& qm = F.mats[qt.mat];
        if (qm.kind == MAT_MIRROR) return;
        V3 d1 = q.pos - x.p;
        double dist1 = norm(d1);
        if (dist1 <= 2 * F.eps_ray) return;
        V3 w1 = d1 / dist1;
        V3 d2 = lpos - q.pos;
        double dist2 = norm(d2);
        if (dist2 <= 2 * F.eps_ray) return;
        V3 w2 = d2 / dist2;
        Cand c;
        c.len = x.len + dist1 + dist2 + suffix_len;
        if (!sink.wants(c.len)) return;  // gate-first culling (RNG already consumed)
        if (occluded(F, x.p, q.pos) || occluded(F, q.pos, lpos)) return;
        const GMat& m = F.mats[x.mat];
        V3 f_v = eval_bsdf(m, x.n, x.wi, w1);
        double g1 = geom_term(x.p, x.n, q.pos, qt.n);
        V3 f_q = eval_bsdf(qm, qt.n, -w1, w2);
        if (wide) {
            LightSample cone;
            if (!light_sample(F.light, q.pos, cone)) return;
            double cos_q = fabs(dot(qt.n, w2));
            c.f = x.fw * f_v * g1 * f_q * cos_q * cone.value;
        } else {
            V3 f_s = eval_bsdf(F.mats[F.lsub.mat], F.lsub.n, -w2, F.lsub.wo_light);
            double g2 = geom_term(q.pos, qt.n, F.lsub.pos, F.lsub.n);
            c.f = x.fw * f_v * g1 * f_q * g2 * f_s * F.lsub.power;
        }
        c.depth = d + 2;
        if (!(luminance(c.f) > 0) || !finite3(c.f)) return;
        double grad = ell_length_gradient(e, q.pos, qt.n);
        if (grad <= 0) return;
        double p_ell = q.pdf_arc * grad / cfg.ell_width;
        double surv = rr_survival(d, cfg.use_rr);
        double pdf_w = pdf_bsdf(m, x.n, x.wi, w1);
        double p_dir = surv * pdf_w * fabs(dot(qt.n, w1)) / (dist1 * dist1);
        double mis_m = p_ell / (p_ell + p_dir);
        c.pdf = x.pdf * p_ell;
        if (!(c.pdf > 0)) return;
        WalkV qv;
        qv.p = q.pos;
        qv.n = qt.n;
        qv.tri = q.tri;
        qv.mat = qt.mat;
        qv.wi = -w1;
        qv.fw = splat(0);
        qv.pdf = 0;
        qv.len = 0;
        qv.lane = 0;
        RecSrc rs{v, d, &qv, lane_key};
        sink.emit(c, mis_m, rs);
    }
};
using EllStep = EllStepT<DirectSampler>;

// one warp: 32-point Gauss-Legendre integral of |d arc / d th| over [a, b],
// node i on lane i, s += w_i f_i in i order (arc_integrate's operations)
__device__ inline double arc_integrate_warp(const ConicArc& arc, double a, double b, double glx, double glw) {
    double mid = 0.5 * (a + b), half = 0.5 * (b - a);
    double term = glw * arc_speed(arc, mid + half * glx);
    double s = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) s += __shfl_sync(0xffffffffu, term, i);
    return s * half;
}

#endif  // __CUDACC__

}  // namespace tofr_b200
