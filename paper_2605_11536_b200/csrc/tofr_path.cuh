// tofr_path.cuh -- device transport: path-tree walk with NEE, lazy
// reconnection records, weighted reservoirs, the hybrid path-length-
// preserving shift with its Newton solve, and GRIS merging.
//
// Semantics follow the CPU reference function by function (cited inline);
// data layout and control flow are GPU-first:
//   * Gate-first culling: a candidate's optical length is known before its
//     visibility ray, so candidates the sensor cannot see (outside the gate /
//     histogram) skip the shadow ray and shading.  The reference drops them in
//     the resampling sink (pipeline.hpp:121-123, p <= 0), and no random number
//     is drawn for them (ris.hpp:34-50), so the result is unchanged.
//   * Lazy records: the reconnection record (transport.hpp:448-582) is built
//     only for the candidate that wins the reservoir at the moment it wins;
//     the record never influences the weights.
//   * Primary hits come from a per-frame G-buffer instead of being re-cast by
//     every temporal reprojection and every replayed prefix
//     (pipeline.hpp:213-214, shiftmap.hpp:463-464); the hit is the same.
//   * Length-gate kernels carry no path-velocity bookkeeping (u); the Doppler
//     gate is a separate, not-yet-built variant.
#pragma once

#include "tofr_geom.h"

namespace tofr_b200 {

constexpr int kMaxVerts = 12;  // transport.hpp:132
constexpr int kMaxLanes = kMaxVerts - 2;

enum : int { SK_SURFACE = 0, SK_LIGHT = 1, SK_LIGHTSUB = 2 };  // transport.hpp:134-138
enum : int { GAUGE_FIXED = 0, GAUGE_RAW = 1, GAUGE_AVG = 2 };   // shiftmap.hpp:135

// Reconnection record (transport.hpp:143-170), Length-gate subset.  Normals
// and materials that are functions of a triangle id in the sample's own frame
// are looked up instead of stored (n1, m1 via tri1; pmat via ptri; m2 kept).
struct Rec {
    int valid, k, n_lanes, skind;
    uint64_t lane_key;
    uint16_t lane_ctr[kMaxLanes];
    double prefix_pdf, prefix_len;
    V3 prefix_fw, p1, wi1;
    int tri1;
    V3 p, pn;
    int ptri;
    V3 p2, n2;
    int m2, obj2;
    V3 wo2, suffix_f;
    double suffix_len;
    double prefix_u, suffix_u;  // path-velocity terms (Doppler gates)
};

struct Sample {  // PathSample (transport.hpp:172-179) without pdf
    V3 f;
    double len;
    double u;  // path velocity (transport.hpp:73-80)
    int depth;
    Rec rec;
};

TOFR_HD void rec_clear(Rec& r) {
    r.valid = 0;
    r.k = -1;
    r.n_lanes = 0;
    r.skind = SK_LIGHT;
    r.lane_key = 0;
    for (int i = 0; i < kMaxLanes; ++i) r.lane_ctr[i] = 0;
    r.prefix_pdf = 1;
    r.prefix_len = 0;
    r.prefix_fw = splat(1);
    r.p1 = splat(0);
    r.wi1 = splat(0);
    r.tri1 = -1;
    r.p = splat(0);
    r.pn = splat(0);
    r.ptri = -1;
    r.p2 = splat(0);
    r.n2 = splat(0);
    r.m2 = -1;
    r.obj2 = -1;
    r.prefix_u = 0;
    r.suffix_u = 0;
    r.wo2 = splat(0);
    r.suffix_f = splat(1);
    r.suffix_len = 0;
}

// Per-stage shift counters (ShiftCounts, shiftmap.hpp:398-417).
struct ShiftCtr {
    uint32_t attempts, newton_ok, newton_failed, occluded, jac_clamped, replay_failed, iterations,
        solves, success;
};
enum : int { SC_ATTEMPTS = 0, SC_NEWTON_OK, SC_NEWTON_FAILED, SC_OCCLUDED, SC_JAC_CLAMPED,
             SC_REPLAY_FAILED, SC_ITERATIONS, SC_SOLVES, SC_SUCCESS, SC_COUNT };

struct PathCfg {
    int max_depth;
    int use_rr;
    int ellipsoidal;
    double ell_center, ell_width;  // TraceConfig::ell_gate
    int gauge;
    int newton;
    double jac_min, jac_max;
    double m_cap;
    uint64_t seed;
    int gate_vel;  // velocity (Doppler) gate: the gated quantity is u, gate centre/width in u units
    int replay;  // the scene has non-reconnectable materials: records with k > 2 exist
    // end a path tree once its length passes the sink's reach (no later
    // candidate can be wanted; same candidates, fewer rays; TOFR_WALK_CUTOFF=0: off)
    int walk_cutoff;
    double shrink_k;           // shrink initialiser's gate widening K (JOB_SHRINK jobs)
    unsigned long long* work;  // device work counters [WK_COUNT] (may be null)
    // per-image-row shift cost (Newton iterations + 4 per job whose
    // destination lies in the row; null = off): the load-balancing probe of
    // multi-GPU row bands (tofr_gpu_session_row_cost)
    unsigned long long* row_cost;
};

// device work counters (cumulative per session): shift jobs, closest-hit rays,
// any-hit (shadow / occlusion) rays, transient histogram deposits
enum : int { WK_JOBS = 0, WK_CLOSEST = 1, WK_ANY = 2, WK_DEPOSITS = 3, WK_MERGES = 4, WK_COUNT = 5 };

#if defined(__CUDACC__)
// warp-aggregated add of a per-lane count (all lanes of the warp must call it)
__device__ __forceinline__ void work_add(unsigned long long* work, int k, uint32_t v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (work && (threadIdx.x & 31) == 0 && v) atomicAdd(&work[k], (unsigned long long)v);
}
#endif

// rr_survival (transport.hpp:193-196)
TOFR_HD double rr_survival(int bounce, int use_rr) { return (!use_rr || bounce < 3) ? 1.0 : 0.7; }

// G-buffer entry: primary hit of a pixel (t, triangle), tri < 0 on a miss.
struct GHit {
    double t;
    int tri;
    int pad;
};

#if defined(__CUDACC__)

__device__ __forceinline__ const GTriInfo& tri_info(const FrameView& F, int id) { return F.tri[id]; }
__device__ __forceinline__ const GMat& mat_of(const FrameView& F, int m) { return F.mats[m]; }
__device__ __forceinline__ const GTriIsect& tri_geo(const FrameView& F, int id) {
    return F.tri_isect[F.tri[id].leaf_slot];
}

// tangent_frame (geometry.hpp:51-63): precomputed per triangle (tangent_frame_of)
__device__ __forceinline__ Frame2 tangent_frame(const FrameView& F, int id) { return F.tframe[id]; }

// ---------------------------------------------------------------------------
// path-tree walk (Tracer::trace_tree, transport.hpp:224-275)

struct WalkV {
    V3 p, n, wi, fw;
    double pdf, len;
    int tri, mat;
    uint32_t lane;
    int pad;
};

// Velocity history of a walk (Doppler gates only; kept apart from WalkV so the
// length-gate kernels do not carry it)
struct WalkVel {
    V3 vel;       // velocity of the vertex (velocity_at)
    double u_in;  // path velocity of the segments camera .. this vertex
};

struct Cand {
    V3 f;
    double len, pdf;
    double u;
    int depth;
};

// the gated quantity of a sample: path length, or path velocity (Doppler)
__host__ __device__ __forceinline__ double gate_value(int gate_vel, double len, double u) {
    return gate_vel ? u : len;
}

// Inputs for building a record lazily: walk history plus the optional
// ellipsoidal insert q acting as vertex d+1.
struct RecSrc {
    const WalkV* v;
    int d;
    const WalkV* q;
    uint64_t lane_key;
    const WalkVel* wv;  // velocity history (null: no velocity terms)
};

__device__ inline WalkVel rs_vel(const RecSrc& s, int i) {
    if (!s.wv || (s.q && i == s.d + 1)) return WalkVel{splat(0), 0.0};
    return s.wv[i];
}

__device__ inline const WalkV& rs_vert(const RecSrc& s, int i) {
    return (s.q && i == s.d + 1) ? *s.q : s.v[i];
}

// build_record (transport.hpp:448-582); VEL adds the path-velocity terms
// (prefix_u, suffix_u, obj2) of Doppler gates
template <bool VEL>
static __device__ __noinline__ void build_record(const FrameView& F, const RecSrc& s, Rec& r) {
    rec_clear(r);
    int last = s.q ? s.d + 1 : s.d;
    int k = -1;
    for (int i = 2; i <= last; ++i) {
        if (F.mats[rs_vert(s, i - 1).mat].reconnectable && F.mats[rs_vert(s, i).mat].reconnectable &&
            (i == last || F.mats[rs_vert(s, i + 1).mat].kind != MAT_MIRROR)) {
            k = i;
            break;
        }
    }
    if (k < 0) return;
    r.valid = 1;
    r.k = k;
    r.n_lanes = k - 2 > 0 ? k - 2 : 0;
    r.lane_key = s.lane_key;
    for (int i = 1; i <= k - 2; ++i) r.lane_ctr[i - 1] = uint16_t(s.v[i].lane);

    const WalkV& pv1 = rs_vert(s, k - 1);
    r.prefix_pdf = pv1.pdf;
    r.prefix_len = pv1.len;
    if (VEL) r.prefix_u = rs_vel(s, k - 1).u_in;
    r.prefix_fw = pv1.fw;
    r.p1 = pv1.p;
    r.tri1 = pv1.tri;
    r.wi1 = pv1.wi;

    const WalkV& pv = rs_vert(s, k);
    r.p = pv.p;
    r.pn = pv.n;
    r.ptri = pv.tri;

    const bool wide = F.light.regime == LIGHT_WIDE;
    if (k == last) {
        if (wide) {
            r.skind = SK_LIGHT;
            r.p2 = F.light.pos;
            r.suffix_len = 0;
            r.suffix_u = 0;
        } else {
            r.skind = SK_LIGHTSUB;
            r.p2 = F.lsub.pos;
            r.suffix_len = F.lsub.chain_len;
            if (VEL) r.suffix_u = dot(velocity_at(F, F.lsub.obj, F.lsub.pos), F.lsub.wo_light);
        }
        return;
    }

    const WalkV& pv2 = rs_vert(s, k + 1);
    r.skind = SK_SURFACE;
    r.p2 = pv2.p;
    r.n2 = pv2.n;
    r.m2 = pv2.mat;
    if (VEL) r.obj2 = F.tri[pv2.tri].obj;
    V3 succ = (k + 1 == last) ? (wide ? F.light.pos : F.lsub.pos) : rs_vert(s, k + 2).p;
    r.wo2 = normalize(succ - pv2.p);

    V3 tail = splat(1);
    double tail_len = 0, tail_u = 0;
    V3 prev_p = pv2.p, prev_n = pv2.n, prev_vel = VEL ? rs_vel(s, k + 1).vel : splat(0);
    for (int i = k + 2; i <= last; ++i) {
        const WalkV& w = rs_vert(s, i);
        V3 wdir = normalize(w.p - prev_p);
        tail = tail * geom_term(prev_p, prev_n, w.p, w.n);
        if (i != last) {
            const GMat& wm = F.mats[w.mat];
            V3 out = normalize(rs_vert(s, i + 1).p - w.p);
            tail = tail * (wm.kind == MAT_MIRROR ? wm.albedo : eval_bsdf(wm, w.n, -wdir, out));
        }
        tail_len += norm(w.p - prev_p);
        if (VEL) {
            V3 wvel = rs_vel(s, i).vel;
            tail_u += dot(prev_vel - wvel, wdir);
            prev_vel = wvel;
        }
        prev_p = w.p;
        prev_n = w.n;
    }
    const WalkV& lastv = rs_vert(s, last);
    if (wide) {
        LightSample ls;
        if (!light_sample(F.light, lastv.p, ls)) {
            r.valid = 0;
            return;
        }
        if (k + 2 <= last) tail = tail * eval_bsdf(F.mats[lastv.mat], lastv.n, lastv.wi, ls.dir);
        tail = tail * (fabs(dot(lastv.n, ls.dir)) * ls.value);
        tail_len += ls.dist;
        if (VEL) tail_u += dot(rs_vel(s, last).vel, ls.dir);
    } else {
        V3 dvec = F.lsub.pos - lastv.p;
        double dist = norm(dvec);
        V3 wto = dvec / dist;
        if (k + 2 <= last) tail = tail * eval_bsdf(F.mats[lastv.mat], lastv.n, lastv.wi, wto);
        V3 f_s = eval_bsdf(F.mats[F.lsub.mat], F.lsub.n, -wto, F.lsub.wo_light);
        tail = tail * (geom_term(lastv.p, lastv.n, F.lsub.pos, F.lsub.n) * f_s * F.lsub.power);
        tail_len += dist + F.lsub.chain_len;
        if (VEL) {
            V3 vs = velocity_at(F, F.lsub.obj, F.lsub.pos);
            tail_u += dot(rs_vel(s, last).vel - vs, wto) + dot(vs, F.lsub.wo_light);
        }
    }
    r.suffix_f = tail;
    r.suffix_len = tail_len;
    r.suffix_u = tail_u;
}

// NEE completion at vertex d (Tracer::emit_nee, transport.hpp:280-328).
// Sink API:  bool wants(double len)  -- can a candidate of this optical
//            length contribute?  (gate-first culling)
//            void emit(const Cand&, double mis_m, const RecSrc&)
template <class Sink, class Ell>
__device__ void emit_nee(const FrameView& F, const PathCfg& cfg, const WalkV* v, int d,
                         uint64_t lane_key, Sink& sink, Ell& ell) {
    const WalkV& x = v[d];
    const GMat& m = F.mats[x.mat];
    Cand c;
    if (F.light.regime == LIGHT_WIDE) {
        LightSample ls;
        if (!light_sample(F.light, x.p, ls)) return;
        c.len = x.len + ls.dist;
        if (!sink.wants(c.len)) return;  // gate-first culling
        if (occluded(F, x.p, F.light.pos)) return;
        V3 f_at = eval_bsdf(m, x.n, x.wi, ls.dir);
        double cos_v = fabs(dot(x.n, ls.dir));
        c.f = x.fw * f_at * (cos_v) * ls.value;
        c.u = 0;  // legacy per-item trace: length gates only
        c.depth = d + 1;
    } else {
        if (!F.lsub.valid) return;
        V3 dvec = F.lsub.pos - x.p;
        double dist = norm(dvec);
        if (dist <= F.eps_ray * 2) return;
        V3 wto = dvec / dist;
        c.len = x.len + dist + F.lsub.chain_len;
        if (!sink.wants(c.len)) return;
        if (occluded(F, x.p, F.lsub.pos)) return;
        V3 f_at = eval_bsdf(m, x.n, x.wi, wto);
        V3 f_s = eval_bsdf(F.mats[F.lsub.mat], F.lsub.n, -wto, F.lsub.wo_light);
        double g = geom_term(x.p, x.n, F.lsub.pos, F.lsub.n);
        c.f = x.fw * f_at * g * f_s * F.lsub.power;
        c.u = 0;
        c.depth = d + 1;
    }
    if (c.len <= 0) return;
    c.pdf = x.pdf;
    if (!(luminance(c.f) > 0) || !finite3(c.f)) return;
    double mis_m = 1.0;
    if (cfg.ellipsoidal && d >= 2 && F.mats[v[d - 1].mat].kind != MAT_MIRROR) {
        double p_dir = x.pdf / v[d - 1].pdf;
        double p_ell = ell.pdf_at(F, cfg, v[d - 1], x.p, x.tri, c.len);
        if (p_ell > 0) mis_m = p_dir / (p_dir + p_ell);
    }
    RecSrc rs{v, d, nullptr, lane_key};
    sink.emit(c, mis_m, rs);
}

// Walk starting from a primary G-buffer hit.  `ell` supplies the ellipsoidal
// completion step and its density for the MIS weight (NoEll: disabled).
template <class Sink, class Ell>
__device__ void trace_tree(const FrameView& F, const PathCfg& cfg, int px, int py, const GHit& g,
                           Rng& rng, Rng& ell_rng, Sink& sink, WalkV* v, Ell& ell) {
    if (g.tri < 0) return;
    V3 d0 = primary_dir(F.cam, px, py);
    const GTriInfo& ti = F.tri[g.tri];
    v[1].p = F.cam.pos + d0 * g.t;
    v[1].n = ti.n;
    v[1].tri = g.tri;
    v[1].mat = ti.mat;
    v[1].wi = -d0;
    v[1].fw = splat(1);
    v[1].pdf = 1;
    v[1].len = g.t;
    v[1].lane = 0;
    for (int d = 1; d + 1 <= cfg.max_depth && d < kMaxVerts - 1; ++d) {
        const GMat& m = F.mats[v[d].mat];
        if (m.kind != MAT_MIRROR) {
            emit_nee(F, cfg, v, d, rng.key, sink, ell);
            if (cfg.ellipsoidal) ell.step(F, cfg, v, d, ell_rng, rng.key, sink);
        }
        if (d + 2 > cfg.max_depth) break;
        // walk cutoff: lengths only grow along the walk, so past the sink's reach
        // no later candidate (NEE, ellipsoidal or extension) can be wanted
        if (cfg.walk_cutoff && v[d].len > sink.walk_max()) break;
        v[d].lane = uint32_t(rng.ctr);
        double surv = rr_survival(d, cfg.use_rr);
        if (surv < 1.0 && rng_next(rng) >= surv) break;
        BsdfSample bs = sample_bsdf(m, v[d].n, v[d].wi, rng);
        if (!bs.valid) break;
        Hit nh;
        if (!intersect(F, v[d].p, bs.wo, nh)) break;
        WalkV& w = v[d + 1];
        const GTriInfo& wt = F.tri[nh.tri];
        w.p = nh.pos;
        w.n = wt.n;
        w.tri = nh.tri;
        w.mat = wt.mat;
        w.wi = -bs.wo;
        w.lane = 0;
        double gt = geom_term(v[d].p, v[d].n, w.p, w.n);
        V3 fr_val = m.kind == MAT_MIRROR ? m.albedo : eval_bsdf(m, v[d].n, v[d].wi, bs.wo);
        w.fw = v[d].fw * fr_val * gt;
        double cos_w = fabs(dot(w.n, bs.wo));
        w.pdf = v[d].pdf * surv * bs.pdf * cos_w / (nh.t * nh.t);
        w.len = v[d].len + nh.t;
    }
}

// Walk hook for runs without the ellipsoidal strategy.
struct NoEll {
    template <class Sink>
    __device__ void step(const FrameView&, const PathCfg&, const WalkV*, int, Rng&, uint64_t, Sink&) {}
    __device__ double pdf_at(const FrameView&, const PathCfg&, const WalkV&, const V3&, int, double) {
        return 0;
    }
};

// ---------------------------------------------------------------------------
// reservoirs (ris.hpp:20-56)

struct ResHdr {
    double W, M, phat, w_sum;
    int has;
};

// ---------------------------------------------------------------------------
// shift mapping (shiftmap.hpp:259-783), Length constraint

struct SurfPt {
    V3 pos, n;
    int tri;
};

struct Prefix {  // BaseShiftResult (shiftmap.hpp:448-454)
    int ok;
    double pdf, len, u;
    V3 fw, p1, n1, wi1;
    int tri1, m1;
};

struct Constraint {  // ConstraintEval (shiftmap.hpp:146-151)
    V2 F;
    M2 dFp, dF;
    V2 grad_cur;
};

__device__ inline double lc_value(const V3& p1, const V3& p2, const V3& p) {
    return norm(p1 - p) + norm(p2 - p);
}
__device__ inline V3 lc_grad(const V3& p1, const V3& p2, const V3& p) {
    return -(normalize(p1 - p) + normalize(p2 - p));
}
__device__ inline M3 lc_hess(const V3& p1, const V3& p2, const V3& p) {
    V3 e1 = p1 - p, e2 = p2 - p;
    double l1 = norm(e1), l2 = norm(e2);
    V3 d1 = e1 / l1, d2 = e2 / l2;
    M3 a = (m3_identity() - m3_outer(d1, d1)) * (1.0 / l1);
    M3 b = (m3_identity() - m3_outer(d2, d2)) * (1.0 / l2);
    return a + b;
}

// assemble_constraint (shiftmap.hpp:155-217)
__device__ inline Constraint assemble(const V3& p1, const V3& p2, const V3& ps, const Frame2& Js,
                               const V3& pc, const Frame2& Jc, double delta, int gauge) {
    Constraint e;
    V3 g3s = lc_grad(p1, p2, ps);
    V3 g3c = lc_grad(p1, p2, pc);
    V2 gs = to_local(Js, g3s);
    V2 gc = to_local(Jc, g3c);
    e.grad_cur = gc;
    V3 disp = pc - ps;
    V2 us = to_local(Js, disp);
    V2 uc = to_local(Jc, disp);
    e.F.x = lc_value(p1, p2, pc) - lc_value(p1, p2, ps) - delta;
    M2 Hs{0, 0, 0, 0}, Hc{0, 0, 0, 0};
    if (gauge != GAUGE_FIXED) {
        Hs = project_sym(Js, lc_hess(p1, p2, ps));
        Hc = project_sym(Jc, lc_hess(p1, p2, pc));
    }
    V2 row_c, row_s, m_c, m_s;
    if (gauge == GAUGE_FIXED) {
        V2 axis{1, 0};
        V3 aw = to_world(Js, axis);
        m_c = to_local(Jc, aw);
        m_s = axis;
        e.F.y = dot(rot90(m_c), uc);
        row_c = rot90(m_c);
        row_s = rot90(m_s);
    } else if (gauge == GAUGE_RAW) {
        V3 mw = g3s;
        m_c = to_local(Jc, mw);
        m_s = gs;
        e.F.y = dot(rot90(m_c), uc);
        row_c = rot90(m_c);
        row_s = rot90(m_s) + Hs * rot90(us);
    } else {
        V3 mw = (g3s + g3c) * 0.5;
        m_c = to_local(Jc, mw);
        m_s = to_local(Js, mw);
        e.F.y = dot(rot90(m_c), uc);
        row_c = rot90(m_c) - (Hc * rot90(uc)) * 0.5;
        row_s = rot90(m_s) + (Hs * rot90(us)) * 0.5;
    }
    e.dFp = M2{gc.x, gc.y, row_c.x, row_c.y};
    e.dF = M2{-gs.x, -gs.y, -row_s.x, -row_s.y};
    return e;
}

__device__ inline SurfPt surf_from_hit(const FrameView& F, const Hit& h) {
    return SurfPt{h.pos, F.tri[h.tri].n, h.tri};
}

// reproject_to_mesh (shiftmap.hpp:275-307)
static __device__ __noinline__ bool reproject(const FrameView& F, const SurfPt& cur, const V3& plane_pt, const V3& p1,
                          SurfPt& out) {
    const GTriIsect& g = tri_geo(F, cur.tri);
    V3 tn = F.tri[cur.tri].n;
    {
        V3 e1 = g.e1, e2 = g.e2, d = plane_pt - g.v0;
        double d11 = dot(e1, e1), d12 = dot(e1, e2), d22 = dot(e2, e2);
        double dv1 = dot(d, e1), dv2 = dot(d, e2);
        double dt = d11 * d22 - d12 * d12;
        if (dt > 0) {
            double u = (d22 * dv1 - d12 * dv2) / dt;
            double v = (d11 * dv2 - d12 * dv1) / dt;
            if (u >= 0 && v >= 0 && u + v <= 1) {
                out = cur;
                out.pos = plane_pt;
                return true;
            }
        }
    }
    V3 dir = plane_pt - p1;
    double dl = norm(dir);
    if (dl > 0) {
        dir = dir / dl;
        if (fabs(dot(dir, tn)) > 1e-4) {
            Hit h;
            if (intersect(F, p1, dir, h)) {
                out = surf_from_hit(F, h);
                return true;
            }
        }
    }
    double off = 1e-3 * F.diag;
    Hit h;
    if (trace_closest(F, plane_pt + tn * off, -tn, 0, 2 * off, h)) {
        out = surf_from_hit(F, h);
        return true;
    }
    if (trace_closest(F, plane_pt - tn * off, tn, 0, 2 * off, h)) {
        out = surf_from_hit(F, h);
        return true;
    }
    return false;
}

struct NewtonOut {
    int converged;
    SurfPt p;
    double jac;
    int iterations;
};

// newton_solve (shiftmap.hpp:314-378); max 5 iterations, 8 halvings
static __device__ __noinline__ NewtonOut newton_solve(const FrameView& F, const V3& p1, const V3& p2, const SurfPt& start,
                                  double delta, int gauge, double tol, double eps_grad) {
    NewtonOut res;
    res.converged = 0;
    res.jac = 0;
    res.iterations = 0;
    Frame2 Js = tangent_frame(F, start.tri);
    SurfPt cur = start;
    Frame2 Jc = Js;
    Constraint e = assemble(p1, p2, start.pos, Js, cur.pos, Jc, delta, gauge);
    double fnorm = hypot(e.F.x, e.F.y);
    // The reference's two nested loops (iterations x 9 halvings) run here as
    // ONE loop of trial steps with the (iteration, halving) position kept per
    // lane: lanes of a warp that are in different iterations or halvings
    // still execute the trial together instead of waiting at the inner
    // loop's exit.  Same decisions in the same order per lane.
    int iter = 0, bt = 0;
    bool need_dir = true;
    double scale = 1.0;
    V2 step{0, 0};
    for (;;) {
        if (need_dir) {
            res.iterations = iter;
            if (fabs(e.F.x) <= tol && fabs(e.F.y) <= tol) {
                res.p = cur;
                double dc = det(e.dFp);
                double j = dc == 0 ? 0 : det(e.dF) / dc;
                if (!(j > 0) || !isfinite(j)) return res;
                res.converged = 1;
                res.jac = j;
                return res;
            }
            if (iter >= 5) break;
            if (norm(e.grad_cur) < eps_grad) break;
            if (!solve2x2(e.dFp, -e.F, step)) break;
            need_dir = false;
            bt = 0;
            scale = 1.0;
        }
        V3 plane_pt = cur.pos + to_world(Jc, step * scale);
        SurfPt trial;
        if (reproject(F, cur, plane_pt, p1, trial)) {
            Frame2 Jt = tangent_frame(F, trial.tri);
            Constraint et = assemble(p1, p2, start.pos, Js, trial.pos, Jt, delta, gauge);
            double fn = hypot(et.F.x, et.F.y);
            if (fn < fnorm) {
                cur = trial;
                Jc = Jt;
                e = et;
                fnorm = fn;
                ++iter;
                need_dir = true;
                continue;
            }
        }
        if (++bt > 8) break;  // no halving accepted
        scale *= 0.5;
    }
    res.p = cur;
    return res;
}

// Domain (shiftmap.hpp:383-387): pixel, gate and frame snapshot.
struct Dom {
    int px, py;
    double center, width;
    const FrameView* F;
    const GHit* gbuf;  // that frame's primary hits
};

// hybrid_base_shift (shiftmap.hpp:459-528): random replay of the prefix from
// the destination pixel with the stored lanes.
static __device__ __noinline__ Prefix base_shift(const Dom& dom, const Rec& rec, const PathCfg& cfg) {
    Prefix out;
    out.ok = 0;
    const FrameView& F = *dom.F;
    GHit g = dom.gbuf[size_t(dom.py) * F.cam.w + dom.px];
    if (g.tri < 0) return out;
    V3 d0 = primary_dir(F.cam, dom.px, dom.py);
    V3 pos = F.cam.pos + d0 * g.t;
    int tri = g.tri;
    V3 n = F.tri[tri].n;
    int mat = F.tri[tri].mat;
    V3 wi = -d0;
    V3 fw = splat(1);
    double pdf = 1, len = g.t;
    V3 vel = velocity_at(F, F.tri[tri].obj, pos);
    double u = dot(F.cam_vel - vel, d0);
    bool rp2 = false;
    bool rp = F.mats[mat].reconnectable;
    for (int i = 1; i <= rec.k - 2; ++i) {
        const GMat& m = F.mats[mat];
        Rng lane{rec.lane_key, rec.lane_ctr[i - 1]};
        double surv = rr_survival(i, cfg.use_rr);
        if (surv < 1.0 && rng_next(lane) >= surv) return out;
        BsdfSample bs = sample_bsdf(m, n, wi, lane);
        if (!bs.valid) return out;
        Hit nh;
        if (!intersect(F, pos, bs.wo, nh)) return out;
        const GTriInfo& nt = F.tri[nh.tri];
        const GMat& nm = F.mats[nt.mat];
        if (i >= 2 && rp2 && rp && nm.kind != MAT_MIRROR) return out;
        double gt = geom_term(pos, n, nh.pos, nt.n);
        V3 fr_val = m.kind == MAT_MIRROR ? m.albedo : eval_bsdf(m, n, wi, bs.wo);
        fw = fw * (fr_val * gt);
        double cos_w = fabs(dot(nt.n, bs.wo));
        pdf = pdf * (surv * bs.pdf * cos_w / (nh.t * nh.t));
        len += nh.t;
        V3 nvel = velocity_at(F, nt.obj, nh.pos);
        u += dot(vel - nvel, bs.wo);
        pos = nh.pos;
        n = nt.n;
        tri = nh.tri;
        mat = nt.mat;
        wi = -bs.wo;
        vel = nvel;
        rp2 = rp;
        rp = nm.reconnectable;
    }
    if (rec.k >= 3 && rp2 && rp) return out;
    if (!rp) return out;
    if (!(pdf > 0) || !finite3(fw)) return out;
    out.ok = 1;
    out.pdf = pdf;
    out.len = len;
    out.u = u;
    out.fw = fw;
    out.p1 = pos;
    out.n1 = n;
    out.wi1 = wi;
    out.tri1 = tri;
    out.m1 = mat;
    return out;
}

struct Suffix {
    V3 p2, n2;
    double len;
    double u;  // suffix path velocity
    V3 v2;     // velocity of the p2 endpoint
    int ok;
    int vobj = -1;  // object whose velocity field v2 is (velocity_at(F, vobj, p2) == v2)
};

// suffix_geometry (shiftmap.hpp:546-575)
__device__ inline Suffix suffix_geometry(const FrameView& F, const Rec& rec) {
    Suffix s;
    s.ok = 0;
    s.n2 = splat(0);
    if (rec.skind == SK_SURFACE) {
        s.p2 = rec.p2;
        s.n2 = rec.n2;
        s.len = rec.suffix_len;
        s.ok = 1;
    } else if (rec.skind == SK_LIGHT) {
        s.p2 = F.light.pos;
        s.len = 0;
        s.ok = 1;
    } else {
        if (!F.lsub.valid) return s;
        s.p2 = F.lsub.pos;
        s.n2 = F.lsub.n;
        s.len = F.lsub.chain_len;
        s.ok = 1;
    }
    return s;
}

// rebuild_sample (shiftmap.hpp:579-654)
static __device__ __noinline__ bool rebuild_sample(const FrameView& F, const Rec& rec, const Prefix& pre, const SurfPt& p,
                               const Suffix& suf, Sample& out) {
    V3 d1 = p.pos - pre.p1;
    double l1 = norm(d1);
    if (l1 <= 2 * F.eps_ray) return false;
    V3 u1 = d1 / l1;
    V3 d2 = suf.p2 - p.pos;
    double l2 = norm(d2);
    if (l2 <= 2 * F.eps_ray) return false;
    V3 u2 = d2 / l2;

    const GMat& m1 = F.mats[pre.m1];
    V3 f = pre.fw * eval_bsdf(m1, pre.n1, pre.wi1, u1) * geom_term(pre.p1, pre.n1, p.pos, p.n);
    const GMat& mp = F.mats[F.tri[p.tri].mat];
    f = f * eval_bsdf(mp, p.n, -u1, u2);
    if (rec.skind == SK_SURFACE) {
        const GMat& m2 = F.mats[rec.m2];
        V3 f2 = m2.kind == MAT_MIRROR ? splat(0) : eval_bsdf(m2, rec.n2, -u2, rec.wo2);
        f = f * (geom_term(p.pos, p.n, rec.p2, rec.n2) * f2 * rec.suffix_f);
    } else if (rec.skind == SK_LIGHT) {
        LightSample ls;
        if (!light_sample(F.light, p.pos, ls)) {
            f = splat(0);
        } else {
            f = f * (fabs(dot(p.n, u2)) * ls.value);
        }
    } else {
        V3 fs = eval_bsdf(F.mats[F.lsub.mat], F.lsub.n, -u2, F.lsub.wo_light);
        f = f * (geom_term(p.pos, p.n, F.lsub.pos, F.lsub.n) * fs * F.lsub.power);
    }
    out.f = f;
    out.len = pre.len + l1 + l2 + suf.len;
    Rec& r = out.rec;
    r = rec;
    r.prefix_pdf = pre.pdf;
    r.prefix_len = pre.len;
    r.prefix_fw = pre.fw;
    r.p1 = pre.p1;
    r.tri1 = pre.tri1;
    r.wi1 = pre.wi1;
    r.p = p.pos;
    r.pn = p.n;
    r.ptri = p.tri;
    if (rec.skind == SK_LIGHTSUB) {
        r.p2 = F.lsub.pos;
        r.n2 = F.lsub.n;
        r.suffix_len = F.lsub.chain_len;
    } else if (rec.skind == SK_LIGHT) {
        r.p2 = F.light.pos;
    }
    return finite3(out.f);
}

__device__ inline void ctr_add(uint32_t* ctr, int i, uint32_t v = 1) {
    if (ctr) ctr[i] += v;
}

// Identity prefix: the stored one (same pixel, same frame).
__device__ inline Prefix stored_prefix(const FrameView& F, const Rec& rec) {
    Prefix pre;
    pre.ok = 1;
    pre.pdf = rec.prefix_pdf;
    pre.len = rec.prefix_len;
    pre.fw = rec.prefix_fw;
    pre.p1 = rec.p1;
    pre.n1 = F.tri[rec.tri1].n;
    pre.wi1 = rec.wi1;
    pre.tri1 = rec.tri1;
    pre.m1 = F.tri[rec.tri1].mat;
    return pre;
}

// shift_sample (shiftmap.hpp:662-783).  Returns true on a usable mapping.
static __device__ __noinline__ bool shift_sample(const Sample& src, const Dom& sd, const Dom& dd, const PathCfg& cfg,
                             uint32_t* ctr, Sample& mapped, double& jac_out) {
    ctr_add(ctr, SC_ATTEMPTS);
    const Rec& rec = src.rec;
    const FrameView& F = *dd.F;
    if (!rec.valid) {
        ctr_add(ctr, SC_REPLAY_FAILED);
        return false;
    }
    bool same_frame = sd.F->frame_id == dd.F->frame_id;
    if (!same_frame && rec.skind == SK_SURFACE && F.geo_motion) {
        ctr_add(ctr, SC_REPLAY_FAILED);
        return false;
    }
    Prefix pre;
    if (same_frame && sd.px == dd.px && sd.py == dd.py)
        pre = stored_prefix(F, rec);
    else
        pre = base_shift(dd, rec, cfg);
    if (!pre.ok) {
        ctr_add(ctr, SC_REPLAY_FAILED);
        return false;
    }
    Suffix suf = suffix_geometry(F, rec);
    if (!suf.ok) {
        ctr_add(ctr, SC_REPLAY_FAILED);
        return false;
    }
    SurfPt start{rec.p, rec.pn, rec.ptri};
    SurfPt solved = start;
    double j_newton = 1.0;
    if (cfg.newton) {
        double gate_delta = dd.center - sd.center;
        double target_local = src.len + gate_delta - pre.len - suf.len;
        double delta = target_local - lc_value(pre.p1, suf.p2, start.pos);
        double tol = 0.01 * dd.width;
        double eps_grad = 1e-8 * F.diag;
        ctr_add(ctr, SC_SOLVES);
        NewtonOut nres = newton_solve(F, pre.p1, suf.p2, start, delta, cfg.gauge, tol, eps_grad);
        ctr_add(ctr, SC_ITERATIONS, uint32_t(nres.iterations));
        if (!nres.converged) {
            ctr_add(ctr, SC_NEWTON_FAILED);
            return false;
        }
        ctr_add(ctr, SC_NEWTON_OK);
        solved = nres.p;
        j_newton = nres.jac;
        if (!F.mats[F.tri[solved.tri].mat].reconnectable) {
            ctr_add(ctr, SC_NEWTON_FAILED);
            return false;
        }
    }
    if (occluded(F, pre.p1, solved.pos) || occluded(F, solved.pos, suf.p2)) {
        ctr_add(ctr, SC_OCCLUDED);
        return false;
    }
    double jac = (rec.prefix_pdf / pre.pdf) * j_newton;
    if (!isfinite(jac) || jac < cfg.jac_min || jac > cfg.jac_max) {
        ctr_add(ctr, SC_JAC_CLAMPED);
        return false;
    }
    mapped.depth = src.depth;
    if (!rebuild_sample(F, rec, pre, solved, suf, mapped)) {
        ctr_add(ctr, SC_REPLAY_FAILED);
        return false;
    }
    jac_out = jac;
    if (ctr && gate_w(dd.center, dd.width, mapped.len) > 0 && luminance(mapped.f) > 0)
        ctr_add(ctr, SC_SUCCESS);
    return true;
}

// shrink_map (shiftmap.hpp:789-876): contract a wide-gate sample onto the fine
// gate (forward) or expand (inverse); identity prefix, no replay.
static __device__ __noinline__ bool shrink_map(const Sample& src, const Dom& dom, double K, bool forward,
                           const PathCfg& cfg, Sample& mapped, double& jac_out) {
    const Rec& rec = src.rec;
    const FrameView& F = *dom.F;
    if (!rec.valid || K < 1) return false;
    Prefix pre = stored_prefix(F, rec);
    Suffix suf = suffix_geometry(F, rec);
    if (!suf.ok) return false;
    double L0 = dom.center;
    double target_total = forward ? (src.len - L0) / K + L0 : (src.len - L0) * K + L0;
    double jac_scale = forward ? 1.0 / K : K;
    SurfPt start{rec.p, rec.pn, rec.ptri};
    double target_local = target_total - pre.len - suf.len;
    double delta = target_local - lc_value(pre.p1, suf.p2, start.pos);
    double tol = 0.01 * dom.width;
    double eps_grad = 1e-8 * F.diag;
    NewtonOut nres = newton_solve(F, pre.p1, suf.p2, start, delta, cfg.gauge, tol, eps_grad);
    if (!nres.converged) return false;
    if (!F.mats[F.tri[nres.p.tri].mat].reconnectable) return false;
    if (occluded(F, pre.p1, nres.p.pos) || occluded(F, nres.p.pos, suf.p2)) return false;
    if (!isfinite(nres.jac) || nres.jac < cfg.jac_min || nres.jac > cfg.jac_max) return false;
    double jac = nres.jac * jac_scale;
    mapped.depth = src.depth;
    if (!rebuild_sample(F, rec, pre, nres.p, suf, mapped)) return false;
    jac_out = jac;
    return true;
}

// ---------------------------------------------------------------------------
// GRIS merge (ris.hpp:78-104) over in-register reservoirs.

struct Res {
    Sample y;
    int has;
    double W, M, phat;
};

__device__ inline bool res_empty(const Res& r) { return !r.has || r.W <= 0; }

// reservoir_update for a merge output; `which` records the selected input.
__device__ inline void merge_update(double& w_sum, int& which, int id, double w, Rng& rng) {
    if (!isfinite(w) || w < 0) return;  // nonfinite_rejected (not reported)
    if (w <= 0) return;
    w_sum += w;
    if (rng_next(rng) * w_sum < w) which = id;
}

struct MergeShift {
    int valid;
    double jac;
    double phat_src_of_dst;
};

// Merges `src` (mapped into dst's domain as `mapped`) into dst.  Returns the
// selected input: 0 none (dst is now empty), 1 dst's own sample (kept, only W
// and M change), 2 the mapped source sample.
// `mapped_gv` is the mapped sample's gated quantity (length, or path velocity).
__device__ __forceinline__ int gris_merge(Res& dst, const Res& src, const MergeShift& ms, const Sample& mapped,
                           double mapped_gv, double dst_center, double dst_width, double m_cap, Rng& rng) {
    double Mc = dst.M, Ms = src.M;
    double w_sum = 0;
    int which = 0;
    double phat_out = 0;
    double py = 0;
    if (!res_empty(dst)) {
        double pc = dst.phat;
        double num = Mc * pc;
        double den = num + Ms * ms.phat_src_of_dst;
        double m_c = den > 0 ? num / den : 0;
        merge_update(w_sum, which, 1, m_c * pc * dst.W, rng);
    }
    if (!res_empty(src) && ms.valid && ms.jac > 0) {
        py = luminance(mapped.f) * gate_w(dst_center, dst_width, mapped_gv);
        if (py > 0) {
            double num = Ms * src.phat / ms.jac;
            double den = Mc * py + num;
            double m_s = den > 0 ? num / den : 0;
            merge_update(w_sum, which, 2, m_s * py * src.W * ms.jac, rng);
        }
    }
    double M = dmin(Mc + Ms, m_cap);
    if (which == 1) {
        phat_out = dst.phat;
    } else if (which == 2) {
        phat_out = py;
        dst.y = mapped;
    }
    dst.has = which != 0;
    dst.phat = phat_out;
    dst.W = (dst.has && phat_out > 0) ? w_sum / phat_out : 0;
    dst.M = M;
    return dst.W > 0 ? which : 0;
}

#endif  // __CUDACC__

}  // namespace tofr_b200
