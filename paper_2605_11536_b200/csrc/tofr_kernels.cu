// tofr_kernels.cu -- sm_100a kernels of the ToF ReSTIR frame pipeline.
//
//   k_gbuffer        primary hit per pixel (camera stage)
//   k_init_gated     RIS over m_init path trees (+ shrink initializer)
//   k_init_transient RIS into per-(pixel, bin) reservoirs
//   k_temporal       reprojection + path-length shift + GRIS merge
//   k_spatial        golden-angle neighbours, shift fwd/inv + GRIS merge
//   k_binreuse       +-1 bin merge with the bin pitch as shift delta
//   k_shade_gated    f * W * gate -> image (+ running frame sum)
//   k_shade_transient per-bin final shading accumulated into the histogram
//   k_hist_plain     trace-only transient deposits (Jarabo-style baseline)
//   k_reference      brute-force gated estimator (mean and standard error)
//
// One thread owns one pixel (or pixel-bin) for the whole stage, which keeps
// the reference's per-pixel sequential RNG semantics (the WRS pick stream is
// consumed in candidate emission order, spatial neighbours merge in order).
// Scenes are tiny, so each CTA stages the BVH nodes and triangle
// intersection records of the frames it touches in shared memory.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "tofr_ellipsoid.cuh"
#include "ktime.h"
#include "tofr_kcommon.cuh"
#include "tofr_store.cuh"

// Minimum resident CTAs per SM requested for the reuse/initial kernels
// (register cap 65536 / (128 * MINB)); tuned with ncu, overridable at build time.
#ifndef TOFR_REUSE_MINB
#define TOFR_REUSE_MINB 4
#endif

namespace tofr_b200 {

size_t frame_smem_bytes(const FrameView& F) {
    size_t nb = size_t(F.n_nodes) * sizeof(GNode);
    size_t tb = size_t(F.n_tris) * sizeof(GTriIsect);
    if (nb + tb > kSmemStageLimit) return 0;
    return ((nb + 15) & ~size_t(15)) + ((tb + 15) & ~size_t(15));
}

// ---------------------------------------------------------------------------
// work-ordering helpers (see k_cost_*)

constexpr int kCostBuckets = 8;

__device__ __forceinline__ bool nonempty(const ResStore& s, size_t i) { return ld2(s, 0, i).x > 0; }

__device__ __forceinline__ bool shiftable(const ResStore& s, size_t i) {
    return ld2(s, 0, i).x > 0 && ld_meta(s, i).valid;
}

// Warp-aggregated append of item `loc` into bucket c.
__device__ __forceinline__ void bucket_count(int c, uint32_t* counts) {
    unsigned peers = __match_any_sync(__activemask(), c);
    int leader = __ffs(peers) - 1;
    if ((threadIdx.x & 31) == leader) atomicAdd(&counts[c], uint32_t(__popc(peers)));
}

// ---------------------------------------------------------------------------
// camera stage

__global__ void __launch_bounds__(256) k_gbuffer(FrameView F, Band bd, GHit* g) {
    extern __shared__ __align__(16) unsigned char smem[];
    size_t off = 0;
    stage_frame(F, smem, off);
    __syncthreads();
    int W = F.cam.w;
    int n = (bd.r1 - bd.r0) * W;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
        int px = p % W, py = bd.r0 + p / W;
        V3 d = primary_dir(F.cam, px, py);
        Hit h;
        GHit o;
        o.pad = 0;
        if (intersect(F, F.cam.pos, d, h)) {
            o.t = h.t;
            o.tri = h.tri;
        } else {
            o.t = kInf;
            o.tri = -1;
        }
        g[p] = o;
    }
}

// ---------------------------------------------------------------------------
// initial candidates

// RIS into one in-register reservoir (stage::initial_sampling run_ris,
// pipeline.hpp:114-128); winner record built when it wins.
struct RisSink {
    const FrameView* F;
    double center, width, inv;
    Rng* pick;
    double w_sum;
    int has;
    double phat;
    Sample* win;
    __device__ bool wants(double len) const { return gate_w(center, width, len) > 0; }
    __device__ double walk_max() const { return center + width; }
    __device__ void emit(const Cand& c, double mis, const RecSrc& rs) {
        double p = luminance(c.f) * gate_w(center, width, c.len);
        if (p <= 0 || !(c.pdf > 0)) return;
        double w = mis * inv * p / c.pdf;
        if (!isfinite(w) || w < 0) return;
        if (w <= 0) return;
        w_sum += w;
        if (rng_next(*pick) * w_sum < w) {
            win->f = c.f;
            win->len = c.len;
            win->depth = c.depth;
            build_record<false>(*F, rs, win->rec);
            has = 1;
            phat = p;
        }
    }
};

template <class Ell>
__device__ void run_ris(const FrameView& F, const PathCfg& cfg, const GHit& g, int px, int py,
                        uint64_t pix, int frame_idx, int trees, double center, double width,
                        Rng& pick, Sample& win, Res& out, WalkV* v, Ell& ell) {
    out.has = 0;
    out.W = 0;
    out.phat = 0;
    out.M = 0;
    if (trees <= 0) return;
    RisSink sink{&F, center, width, 1.0 / trees, &pick, 0.0, 0, 0.0, &win};
    for (int s = 0; s < trees; ++s) {
        Rng rng = rng_make(cfg.seed, uint64_t(frame_idx), pix, uint64_t(s), 0);
        Rng erng = rng_make(cfg.seed, uint64_t(frame_idx), pix, uint64_t(s), 2);
        trace_tree(F, cfg, px, py, g, rng, erng, sink, v, ell);
    }
    out.has = sink.has;
    out.phat = sink.phat;
    out.W = (sink.has && sink.phat > 0) ? sink.w_sum / sink.phat : 0;
    out.M = 1;
}

template <class Ell>
__device__ void init_pixel(const FrameView& F, const PathCfg& cfg, const InitParams& ip, const GHit& g,
                           int px, int py, int frame_idx, Res& out, WalkV* v, Ell& ell) {
    uint64_t pix = uint64_t(py) * F.cam.w + px;
    Rng pick = rng_make(cfg.seed, uint64_t(frame_idx), pix, 0, 9);
    if (ip.mode != INIT_SHRINK) {
        run_ris(F, cfg, g, px, py, pix, frame_idx, ip.m_init, ip.center, ip.width, pick, out.y, out, v, ell);
        out.M = 1;
        return;
    }
    // shrink initializer (pipeline.hpp:137-183)
    int m_rough = int(llround(ip.shrink_r * ip.m_init));
    m_rough = m_rough < 0 ? 0 : (m_rough > ip.m_init ? ip.m_init : m_rough);
    int m_fine = ip.m_init - m_rough;
    Res rough;
    run_ris(F, cfg, g, px, py, pix, frame_idx, m_rough, ip.center, ip.width * ip.shrink_k, pick, rough.y,
            rough, v, ell);
    run_ris(F, cfg, g, px, py, pix, frame_idx, m_fine, ip.center, ip.width, pick, out.y, out, v, ell);
    out.M = 1;
    if (res_empty(rough)) return;
    Dom dom{px, py, ip.center, ip.width, &F, nullptr};
    Sample fwd;
    double fjac = 0;
    bool fok = shrink_map(rough.y, dom, ip.shrink_k, true, cfg, fwd, fjac);
    if (m_fine == 0) {
        double w_sum = 0;
        int has = 0;
        double ph = 0;
        if (fok) {
            double pyv = luminance(fwd.f) * gate_w(ip.center, ip.width, fwd.len);
            double w = pyv * rough.W * fjac;
            if (isfinite(w) && w > 0) {
                w_sum += w;
                if (rng_next(pick) * w_sum < w) {
                    has = 1;
                    ph = pyv;
                    out.y = fwd;
                }
            }
        }
        out.has = has;
        out.phat = ph;
        out.W = (has && ph > 0) ? w_sum / ph : 0;
        out.M = 1;
        return;
    }
    MergeShift ms{0, 1.0, 0.0};
    if (fok) {
        ms.valid = 1;
        ms.jac = fjac;
    }
    if (!res_empty(out)) {
        Sample inv;
        double ijac = 0;
        if (shrink_map(out.y, dom, ip.shrink_k, false, cfg, inv, ijac))
            ms.phat_src_of_dst =
                luminance(inv.f) * gate_w(ip.center, ip.width * ip.shrink_k, inv.len) * ijac;
    }
    gris_merge(out, rough, ms, fwd, fwd.len, ip.center, ip.width, cfg.m_cap, pick);
}

__global__ void __launch_bounds__(128, TOFR_REUSE_MINB) k_init_gated(FrameView F, Band bd, const GHit* gbuf, PathCfg cfg,
                                                    InitParams ip, int frame_idx, ResStore cur,
                                                    unsigned long long* q, EllScratch es) {
    extern __shared__ __align__(16) unsigned char smem[];
    size_t off = 0;
    stage_frame(F, smem, off);
    __syncthreads();
    int W = F.cam.w;
    WalkV v[kMaxVerts];
    size_t n = size_t(bd.y1 - bd.y0) * W;
    TOFR_FOR_ITEMS(i, n, q) {
        int p = bd.y0 * W + int(i);
        int px = p % W, py = p / W;
        Res r;
        GHit g = gbuf[p];
        if (cfg.ellipsoidal && es.jobs) {  // replay of the planned + bisected ellipsoidal vertices
            EllStepT<ReplaySampler> ell{ReplaySampler{es, i * size_t(es.per_pixel), 0}};
            init_pixel(F, cfg, ip, g, px, py, frame_idx, r, v, ell);
        } else if (cfg.ellipsoidal) {
            EllStep ell;
            init_pixel(F, cfg, ip, g, px, py, frame_idx, r, v, ell);
        } else {
            NoEll ell;
            init_pixel(F, cfg, ip, g, px, py, frame_idx, r, v, ell);
        }
        res_store_result(cur, size_t(p), r);
    }
}

// ---------------------------------------------------------------------------
// wavefront ellipsoidal sampling (tofr_ellipsoid.cuh): plan and arcs launches

// a sink that wants no candidate: emit_nee culls every NEE before its ray
struct NullSink {
    double reach;  // the replay's walk cutoff (the same walk, the same sampler calls)
    __device__ bool wants(double) const { return false; }
    __device__ double walk_max() const { return reach; }
    __device__ void emit(const Cand&, double, const RecSrc&) {}
};

// the path trees of run_ris (pipeline.hpp:114-128) with the ellipsoidal step
// recording jobs: same walk and ellipsoid RNG draws as the replay
__global__ void __launch_bounds__(128, TOFR_REUSE_MINB) k_ell_plan(FrameView F, Band bd, const GHit* gbuf,
                                                                  PathCfg cfg, int m_init, int frame_idx,
                                                                  EllScratch es, unsigned long long* q) {
    extern __shared__ __align__(16) unsigned char smem[];
    size_t off = 0;
    stage_frame(F, smem, off);
    __syncthreads();
    int W = F.cam.w;
    WalkV v[kMaxVerts];
    size_t n = size_t(bd.y1 - bd.y0) * W;
    TOFR_FOR_ITEMS(i, n, q) {
        int p = bd.y0 * W + int(i);
        int px = p % W, py = p / W;
        uint64_t pix = uint64_t(py) * W + px;
        GHit g = gbuf[p];
        NullSink sink{cfg.ell_center + cfg.ell_width};
        EllStepT<PlanSampler> ell{PlanSampler{es, i * size_t(es.per_pixel), 0}};
        for (int s = 0; s < m_init; ++s) {
            Rng rng = rng_make(cfg.seed, uint64_t(frame_idx), pix, uint64_t(s), 0);
            Rng erng = rng_make(cfg.seed, uint64_t(frame_idx), pix, uint64_t(s), 2);
            trace_tree(F, cfg, px, py, g, rng, erng, sink, v, ell);
        }
    }
}

// one warp per job: arc_lengths + sample_arc (ellipsoid.hpp:167-296) with
// warp-wide Gauss-Legendre integrals; lane 0 writes the vertex and its pdf
__global__ void __launch_bounds__(256) k_ell_arcs(FrameView F, EllScratch es, unsigned long long* q) {
    const int lane = threadIdx.x & 31;
    const double glx = c_gl_x[lane], glw = c_gl_w[lane];
    const unsigned n = *es.count;
    for (;;) {
        unsigned long long jn = 0;
        if (lane == 0) jn = atomicAdd(q, 1ull);
        jn = __shfl_sync(0xffffffffu, jn, 0);
        if (jn >= n) break;
        const uint32_t slot = es.list[jn];
        const EllJob& J = es.jobs[slot];
        ConicArc arc;
        const GTriIsect& tg = tri_geo(F, J.tri);
        arc.origin = tg.v0;
        arc.frame = tangent_frame(F, J.tri);
        arc.center = J.center;
        arc.ax1 = J.ax1;
        arc.ax2 = J.ax2;
        arc.r1 = J.r1;
        arc.r2 = J.r2;
        arc.nseg = J.nseg;
        arc.total_len = 0;
        for (int i = 0; i < arc.nseg; ++i) {  // arc_lengths
            arc.t0[i] = J.t0[i];
            arc.t1[i] = J.t1[i];
            arc.len[i] = arc_integrate_warp(arc, arc.t0[i], arc.t1[i], glx, glw);
            arc.total_len += arc.len[i];
        }
        // sample_arc (ellipsoid.hpp:273-296) with the planned draw
        double target = J.u * arc.total_len;
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
            double l = arc_integrate_warp(arc, arc.t0[si], mid, glx, glw);
            if (l < target)
                lo = mid;
            else
                hi = mid;
            if ((hi - lo) * arc_speed(arc, 0.5 * (lo + hi)) < 1e-6 * dmax(arc.total_len, 1e-30)) break;
        }
        if (lane == 0) {
            double pdf_len = 1.0 / arc.total_len;
            EllRes r;
            r.pos = arc.origin + to_world(arc.frame, arc_point2(arc, 0.5 * (lo + hi)));
            r.pdf_arc = J.p_dt * pdf_len;
            es.res[slot] = r;
        }
    }
}

// Transient RIS: candidates land in the reservoir of bin_of(len); p-hat is
// evaluated against that bin's (inclusive) gate (pipeline.hpp:421-445).
struct BinSink {
    const FrameView* F;
    HistSpec h;
    double inv;
    Rng* pick;
    ResStore st;
    size_t base;
    __device__ bool wants(double len) const {
        int b = bin_of(h, len);
        return b >= 0 && gate_w(bin_center(h, b), h.bw, len) > 0;
    }
    __device__ double walk_max() const { return h.t0 + (h.bins + 1) * h.bw; }
    __device__ void emit(const Cand& c, double mis, const RecSrc& rs) {
        int b = bin_of(h, c.len);
        if (b < 0 || !(c.pdf > 0)) return;
        double p = luminance(c.f) * gate_w(bin_center(h, b), h.bw, c.len);
        if (p <= 0) return;
        double w = mis * inv * p / c.pdf;
        if (!isfinite(w) || w < 0) return;
        if (w <= 0) return;
        size_t i = base + b;
        double2 c0 = ld2(st, 0, i);  // (w_sum during init, M)
        double w_sum = c0.x + w;
        st2(st, 0, i, w_sum, c0.y);
        if (rng_next(*pick) * w_sum < w) {
            Res r;
            r.W = w_sum;
            r.M = c0.y;
            r.has = 1;
            r.phat = p;
            r.y.f = c.f;
            r.y.len = c.len;
            r.y.depth = c.depth;
            build_record<false>(*F, rs, r.y.rec);
            res_store(st, i, r);
        }
    }
};

__global__ void __launch_bounds__(128, TOFR_REUSE_MINB) k_init_transient(FrameView F, Band bd, const GHit* gbuf, PathCfg cfg,
                                                        InitParams ip, HistSpec h, int frame_idx,
                                                        ResStore cur, unsigned long long* q) {
    extern __shared__ __align__(16) unsigned char smem[];
    size_t off = 0;
    stage_frame(F, smem, off);
    __syncthreads();
    int W = F.cam.w, B = h.bins;
    WalkV v[kMaxVerts];
    NoEll ell;
    size_t n = size_t(bd.y1 - bd.y0) * W;
    TOFR_FOR_ITEMS(i, n, q) {
        int p = bd.y0 * W + int(i);
        int px = p % W, py = p / W;
        uint64_t pix = uint64_t(py) * W + px;
        size_t base = size_t(p) * B;
        for (int b = 0; b < B; ++b) res_store_w(cur, base + b, 0.0, 0.0);
        Rng pick = rng_make(cfg.seed, uint64_t(frame_idx), pix, 0, 9);
        BinSink sink{&F, h, 1.0 / ip.m_init, &pick, cur, base};
        GHit g = gbuf[p];
        for (int s = 0; s < ip.m_init; ++s) {
            Rng rng = rng_make(cfg.seed, uint64_t(frame_idx), pix, uint64_t(s), 0);
            Rng erng = rng_make(cfg.seed, uint64_t(frame_idx), pix, uint64_t(s), 2);
            trace_tree(F, cfg, px, py, g, rng, erng, sink, v, ell);
        }
        for (int b = 0; b < B; ++b) {  // ris_finalize + M = 1
            size_t i = base + b;
            double2 c0 = ld2(cur, 0, i);  // (w_sum, -): w_sum > 0 iff a candidate was picked
            double Wv = 0;
            if (c0.x > 0) {
                double phat = ld2(cur, 1, i).x;
                Wv = phat > 0 ? c0.x / phat : 0;
            }
            st2(cur, 0, i, Wv, 1.0);
        }
    }
}

// ---------------------------------------------------------------------------
// temporal reuse (stage::temporal_reuse, pipeline.hpp:209-229)

__global__ void __launch_bounds__(128, TOFR_REUSE_MINB) k_temporal(FrameView Fc, Band bd, const GHit* gc, FrameView Fp,
                                                  const GHit* gp, PathCfg cfg, GateGrid cur_gate,
                                                  GateGrid prev_gate, int frame_idx, ResStore cur,
                                                  ResStore prev, const uint32_t* perm,
                                                  unsigned long long* ctr_out, unsigned long long* q) {
    extern __shared__ __align__(16) unsigned char smem[];
    size_t off = 0;
    stage_frame(Fc, smem, off);
    stage_frame(Fp, smem, off);
    __syncthreads();
    int W = Fc.cam.w, B = cur_gate.transient ? cur_gate.h.bins : 1;
    uint32_t ctr[SC_COUNT] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    TOFR_FOR_ITEMS(i, n, q) {
        size_t it = base + (perm ? size_t(perm[i]) : i);
        int p = int(it / B), b = int(it % B);
        int px = p % W, py = p / W;
        GHit g = gc[p];
        if (g.tri < 0) continue;
        V3 d0 = primary_dir(Fc.cam, px, py);
        V3 hp = Fc.cam.pos + d0 * g.t;
        int qx, qy;
        if (!project(Fp.cam, hp, qx, qy)) continue;
        if (qy < bd.t0 || qy >= bd.t1) {  // reprojection left the rows this band holds
            atomicAdd(bd.err, 1ull);
            continue;
        }
        size_t src_i = (size_t(qy) * W + qx) * B + b;
        Res dst, src;
        res_load_head(prev, src_i, src);
        if (src.M <= 0) continue;
        double dc, dw, sc, sw;
        gate_of(cur_gate, b, dc, dw);
        gate_of(prev_gate, b, sc, sw);
        res_load(cur, it, dst);
        if (src.has) {
            res_load_value(prev, src_i, src);
            res_load_rec(prev, src_i, src.y);
        }
        Dom dd{px, py, dc, dw, &Fc, gc};
        Dom sd{qx, qy, sc, sw, &Fp, gp};
        MergeShift ms{0, 1.0, 0.0};
        Sample mapped;
        if (!res_empty(src)) {
            double jac;
            if (shift_sample(src.y, sd, dd, cfg, ctr, mapped, jac)) {
                ms.valid = 1;
                ms.jac = jac;
            }
        }
        if (!res_empty(dst)) {
            Sample inv;
            double jac;
            if (shift_sample(dst.y, dd, sd, cfg, nullptr, inv, jac))
                ms.phat_src_of_dst = luminance(inv.f) * gate_w(sc, sw, inv.len) * jac;
        }
        uint64_t pix = uint64_t(py) * W + px;
        Rng rng = rng_make(cfg.seed, uint64_t(frame_idx), pix, uint64_t(b), 8);
        int which = gris_merge(dst, src, ms, mapped, mapped.len, dc, dw, cfg.m_cap, rng);
        if (which == 2)
            res_store(cur, it, dst);
        else  // in place: the kept sample and its p-hat are already stored
            res_store_w(cur, it, dst.W, dst.M);
    }
    flush_ctr(ctr, ctr_out);
}

// ---------------------------------------------------------------------------
// spatial reuse (stage::spatial_reuse + neighbor_offset, pipeline.hpp:232-269)

__global__ void __launch_bounds__(128, TOFR_REUSE_MINB) k_spatial(FrameView F, Band bd, const GHit* gbuf, PathCfg cfg,
                                                 GateGrid gate, SpatialParams sp, int pass,
                                                 int frame_idx, ResStore src_grid, ResStore dst_grid,
                                                 const uint32_t* perm, unsigned long long* ctr_out,
                                                 unsigned long long* q) {
    extern __shared__ __align__(16) unsigned char smem[];
    size_t off = 0;
    stage_frame(F, smem, off);
    __syncthreads();
    int W = F.cam.w, H = F.cam.h, B = gate.transient ? gate.h.bins : 1;
    uint32_t ctr[SC_COUNT] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    TOFR_FOR_ITEMS(i, n, q) {
        size_t it = base + (perm ? size_t(perm[i]) : i);
        int p = int(it / B), b = int(it % B);
        int px = p % W, py = p / W;
        Res out;
        res_load(src_grid, it, out);
        if (sp.neighbors > 0 && sp.radius > 0) {
            double dc, dw;
            gate_of(gate, b, dc, dw);
            uint64_t pix = uint64_t(py) * W + px;
            Rng rng = rng_make(cfg.seed, uint64_t(frame_idx), pix, uint64_t(pass * 131 + b), 10);
            Dom dd{px, py, dc, dw, &F, gbuf};
            uint64_t rk = mix64(pix * 1315423911u + (unsigned)(pass * 2654435761u) + uint64_t(cfg.seed) +
                                uint64_t(frame_idx) * 97);
            for (int j = 0; j < sp.neighbors; ++j) {
                int dx, dy;
                neighbor_offset(j, sp.neighbors, sp.radius, rk, dx, dy);
                int nx = px + dx, ny = py + dy;
                if (nx == px && ny == py) continue;
                if (nx < 0 || nx >= W || ny < 0 || ny >= H) continue;
                if (ny < bd.r0 || ny >= bd.r1) {  // beyond the exchanged halo
                    atomicAdd(bd.err, 1ull);
                    continue;
                }
                size_t si = (size_t(ny) * W + nx) * B + b;
                Res src;
                res_load_head(src_grid, si, src);
                if (src.M <= 0) continue;
                if (src.has) {
                    res_load_value(src_grid, si, src);
                    res_load_rec(src_grid, si, src.y);
                }
                Dom sd{nx, ny, dc, dw, &F, gbuf};
                MergeShift ms{0, 1.0, 0.0};
                Sample mapped;
                if (!res_empty(src)) {
                    double jac;
                    if (shift_sample(src.y, sd, dd, cfg, ctr, mapped, jac)) {
                        ms.valid = 1;
                        ms.jac = jac;
                    }
                }
                if (!res_empty(out)) {
                    Sample inv;
                    double jac;
                    if (shift_sample(out.y, dd, sd, cfg, nullptr, inv, jac))
                        ms.phat_src_of_dst = luminance(inv.f) * gate_w(dc, dw, inv.len) * jac;
                }
                gris_merge(out, src, ms, mapped, mapped.len, dc, dw, cfg.m_cap, rng);
            }
        }
        res_store_result(dst_grid, it, out);
    }
    flush_ctr(ctr, ctr_out);
}

// ---------------------------------------------------------------------------
// Spatial reuse split into phases.  k_spatial runs a pixel's whole merge chain
// in one thread: per neighbour j a forward shift (neighbour sample -> pixel),
// an inverse shift (running output -> neighbour) and a GRIS merge.  On B200
// that chain diverges badly (lanes of one warp sit in different shifts and
// Newton iterations).  The forward shifts do not depend on the merge order,
// so they run first as one flat, compacted list of (neighbour, pixel) jobs;
// the inverse shift + merge of neighbour j then runs as one kernel per j with
// the running output and the lane-10 RNG counter carried in HBM.  Same
// arithmetic, same RNG draws in the same order, same counters.


__global__ void k_spatial_fwd_list(FrameView F, Band bd, PathCfg cfg, GateGrid gate, SpatialParams sp, int pass,
                                   int frame_idx, ResStore src_grid, SpatialScratch sc) {
    int W = F.cam.w, H = F.cam.h, B = gate.transient ? gate.h.bins : 1;
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t n_round = (n + 31) & ~size_t(31);
    int lane = threadIdx.x & 31;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n_round; i += stride) {
        bool live = i < n;
        size_t it = base + (live ? i : 0);
        int p = int(it / B), b = int(it % B);
        int px = p % W, py = p / W;
        uint64_t rk = spatial_rot_key(uint64_t(py) * W + px, pass, cfg.seed, frame_idx);
        for (int j = 0; j < sp.neighbors; ++j) {
            int nx, ny;
            size_t si = 0;
            // every non-empty neighbour is a forward shift attempt (counted even
            // when its record has no reconnection vertex, as the reference does)
            bool want = live && spatial_neighbor(bd, W, H, B, px, py, b, sp, rk, j, src_grid, nx, ny, si) &&
                        nonempty(src_grid, si);
            unsigned m = __ballot_sync(0xffffffffu, want);
            if (!m) continue;
            uint32_t start = 0;
            if (lane == __ffs(m) - 1) start = atomicAdd(sc.count, uint32_t(__popc(m)));
            start = __shfl_sync(0xffffffffu, start, __ffs(m) - 1);
            if (want) sc.list[start + __popc(m & ((1u << lane) - 1))] = uint32_t(size_t(j) * n + i);
        }
    }
}

__global__ void __launch_bounds__(128, TOFR_REUSE_MINB)
    k_spatial_fwd(FrameView F, Band bd, const GHit* gbuf, PathCfg cfg, GateGrid gate, SpatialParams sp, int pass,
                  int frame_idx, ResStore src_grid, SpatialScratch sc, unsigned long long* ctr_out,
                  unsigned long long* q) {
    extern __shared__ __align__(16) unsigned char smem[];
    size_t off = 0;
    stage_frame(F, smem, off);
    __syncthreads();
    int W = F.cam.w, B = gate.transient ? gate.h.bins : 1;
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    uint32_t ctr[SC_COUNT] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    size_t jobs = *sc.count;
    TOFR_FOR_ITEMS(jq, jobs, q) {
        uint32_t e = sc.list[jq];
        int j = int(e / n);
        size_t i = e % n, it = base + i;
        int p = int(it / B), b = int(it % B);
        int px = p % W, py = p / W;
        double dc, dw;
        gate_of(gate, b, dc, dw);
        uint64_t rk = spatial_rot_key(uint64_t(py) * W + px, pass, cfg.seed, frame_idx);
        int nx, ny, dx, dy;
        neighbor_offset(j, sp.neighbors, sp.radius, rk, dx, dy);
        nx = px + dx;
        ny = py + dy;
        size_t si = (size_t(ny) * W + nx) * B + b;
        Res src;
        res_load(src_grid, si, src);
        Dom dd{px, py, dc, dw, &F, gbuf};
        Dom sd{nx, ny, dc, dw, &F, gbuf};
        Res m;
        double jac;
        if (shift_sample(src.y, sd, dd, cfg, ctr, m.y, jac)) {
            m.has = 1;
            m.W = jac;
            m.M = 0;
            m.phat = 0;
            res_store(sc.mapped, e, m);
            sc.ok[e] = 1;
        }
    }
    flush_ctr(ctr, ctr_out);
}

__global__ void __launch_bounds__(128, TOFR_REUSE_MINB)
    k_spatial_merge(FrameView F, Band bd, const GHit* gbuf, PathCfg cfg, GateGrid gate, SpatialParams sp, int pass,
                    int j, int frame_idx, ResStore src_grid, ResStore dst_grid, SpatialScratch sc,
                    unsigned long long* q) {
    extern __shared__ __align__(16) unsigned char smem[];
    size_t off = 0;
    stage_frame(F, smem, off);
    __syncthreads();
    int W = F.cam.w, H = F.cam.h, B = gate.transient ? gate.h.bins : 1;
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    TOFR_FOR_ITEMS(i, n, q) {
        size_t it = base + i;
        int p = int(it / B), b = int(it % B);
        int px = p % W, py = p / W;
        uint64_t pix = uint64_t(py) * W + px;
        uint64_t rk = spatial_rot_key(pix, pass, cfg.seed, frame_idx);
        int nx, ny;
        size_t si = 0;
        bool use = spatial_neighbor(bd, W, H, B, px, py, b, sp, rk, j, src_grid, nx, ny, si);
        if (!use) {
            if (j == 0) {  // the output starts as the pass input
                Res out;
                res_load(src_grid, it, out);
                res_store_result(dst_grid, it, out);
            }
            if (j + 1 < sp.neighbors && j == 0) sc.rng_ctr[i] = 0;
            continue;
        }
        Res out;
        res_load(j == 0 ? src_grid : dst_grid, it, out);
        Rng rng = rng_make(cfg.seed, uint64_t(frame_idx), pix, uint64_t(pass * 131 + b), 10);
        if (j > 0) rng.ctr = sc.rng_ctr[i];
        double dc, dw;
        gate_of(gate, b, dc, dw);
        Res src;  // header only: gris_merge reads W, M, phat, has
        res_load_head(src_grid, si, src);
        if (src.has) src.phat = ld2(src_grid, 1, si).x;
        size_t e = size_t(j) * n + i;
        MergeShift ms{0, 1.0, 0.0};
        Res mapped;  // f, len, jac now; the record only if it is selected
        if (!res_empty(src) && sc.ok[e]) {
            res_load_head(sc.mapped, e, mapped);
            res_load_value(sc.mapped, e, mapped);
            ms.valid = 1;
            ms.jac = mapped.W;
        }
        if (!res_empty(out)) {
            Dom dd{px, py, dc, dw, &F, gbuf};
            Dom sd{nx, ny, dc, dw, &F, gbuf};
            Sample inv;
            double jac;
            if (shift_sample(out.y, dd, sd, cfg, nullptr, inv, jac))
                ms.phat_src_of_dst = luminance(inv.f) * gate_w(dc, dw, inv.len) * jac;
        }
        int which = gris_merge(out, src, ms, mapped.y, mapped.y.len, dc, dw, cfg.m_cap, rng);
        if (which == 2) {
            res_load_rec(sc.mapped, e, out.y);
            res_store(dst_grid, it, out);
        } else if (which == 1 && j > 0) {  // in place: sample and p-hat already stored
            res_store_w(dst_grid, it, out.W, out.M);
        } else {
            res_store_result(dst_grid, it, out);
        }
        if (j + 1 < sp.neighbors) sc.rng_ctr[i] = rng.ctr;
    }
}

// ---------------------------------------------------------------------------
// bin reuse (stage::bin_reuse, pipeline.hpp:273-299)

__global__ void __launch_bounds__(128, TOFR_REUSE_MINB) k_binreuse(FrameView F, Band bd, const GHit* gbuf, PathCfg cfg,
                                                  HistSpec h, int frame_idx, ResStore src_grid,
                                                  ResStore dst_grid, unsigned long long* ctr_out,
                                                  unsigned long long* q) {
    extern __shared__ __align__(16) unsigned char smem[];
    size_t off = 0;
    stage_frame(F, smem, off);
    __syncthreads();
    int W = F.cam.w, B = h.bins;
    uint32_t ctr[SC_COUNT] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    TOFR_FOR_ITEMS(i, n, q) {
        size_t it = base + i;
        int p = int(it / B), b = int(it % B);
        int px = p % W, py = p / W;
        Res out;
        res_load(src_grid, it, out);
        double dc = bin_center(h, b), dw = h.bw;
        Dom dd{px, py, dc, dw, &F, gbuf};
        uint64_t pix = uint64_t(py) * W + px;
        Rng rng = rng_make(cfg.seed, uint64_t(frame_idx), pix, uint64_t(b), 12);
        for (int k = 0; k < 2; ++k) {
            int nb = k == 0 ? b - 1 : b + 1;
            if (nb < 0 || nb >= B) continue;
            size_t si = size_t(p) * B + nb;
            Res src;
            res_load_head(src_grid, si, src);
            if (src.M <= 0) continue;
            if (src.has) {
                res_load_value(src_grid, si, src);
                res_load_rec(src_grid, si, src.y);
            }
            double sc = bin_center(h, nb);
            Dom sd{px, py, sc, dw, &F, gbuf};
            MergeShift ms{0, 1.0, 0.0};
            Sample mapped;
            if (!res_empty(src)) {
                double jac;
                if (shift_sample(src.y, sd, dd, cfg, ctr, mapped, jac)) {
                    ms.valid = 1;
                    ms.jac = jac;
                }
            }
            if (!res_empty(out)) {
                Sample inv;
                double jac;
                if (shift_sample(out.y, dd, sd, cfg, nullptr, inv, jac))
                    ms.phat_src_of_dst = luminance(inv.f) * gate_w(sc, dw, inv.len) * jac;
            }
            gris_merge(out, src, ms, mapped, mapped.len, dc, dw, cfg.m_cap, rng);
        }
        res_store_result(dst_grid, it, out);
    }
    flush_ctr(ctr, ctr_out);
}

// ---------------------------------------------------------------------------
// Work ordering for the reuse kernels.  One thread owns one reservoir item for
// the whole merge chain (the reference's per-pixel sequential semantics), and
// the cost of an item is dominated by the shifts it attempts (replay, Newton,
// re-projection and occlusion rays).  A cheap pre-pass estimates that count
// from the reservoir headers, and the items are then processed heaviest first
// in cost buckets, so that a warp's lanes carry similar shift loads instead of
// mixing 6-shift pixels with empty ones.  Results do not depend on the order:
// items are independent given the pass-input grid, counters are sums.

__global__ void k_cost_temporal(FrameView Fc, Band bd, const GHit* gc, FrameView Fp, GateGrid cur_gate,
                                ResStore cur, ResStore prev, uint8_t* cls, uint32_t* counts) {
    int W = Fc.cam.w, B = cur_gate.transient ? cur_gate.h.bins : 1;
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t n_round = (n + 31) & ~size_t(31);
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n_round; i += stride) {
        if (i >= n) continue;
        size_t it = base + i;
        int p = int(it / B), b = int(it % B);
        int px = p % W, py = p / W;
        int c = 0;
        GHit g = gc[p];
        if (g.tri >= 0) {
            V3 d0 = primary_dir(Fc.cam, px, py);
            V3 hp = Fc.cam.pos + d0 * g.t;
            int qx, qy;
            if (project(Fp.cam, hp, qx, qy) && qy >= bd.t0 && qy < bd.t1) {
                size_t si = (size_t(qy) * W + qx) * B + b;
                c = 1 + int(shiftable(prev, si)) * 3 + int(shiftable(cur, it)) * 3;
            }
        }
        c = c > kCostBuckets - 1 ? kCostBuckets - 1 : c;
        cls[i] = uint8_t(c);
        bucket_count(c, counts);
    }
}

__global__ void k_cost_spatial(FrameView F, Band bd, PathCfg cfg, GateGrid gate, SpatialParams sp, int pass,
                               int frame_idx, ResStore src_grid, uint8_t* cls, uint32_t* counts) {
    int W = F.cam.w, H = F.cam.h, B = gate.transient ? gate.h.bins : 1;
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t n_round = (n + 31) & ~size_t(31);
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n_round; i += stride) {
        if (i >= n) continue;
        size_t it = base + i;
        int p = int(it / B), b = int(it % B);
        int px = p % W, py = p / W;
        int c = 0;
        if (sp.neighbors > 0 && sp.radius > 0) {
            bool self = shiftable(src_grid, it);
            uint64_t pix = uint64_t(py) * W + px;
            uint64_t rk = mix64(pix * 1315423911u + (unsigned)(pass * 2654435761u) + uint64_t(cfg.seed) +
                                uint64_t(frame_idx) * 97);
            for (int j = 0; j < sp.neighbors; ++j) {
                int dx, dy;
                neighbor_offset(j, sp.neighbors, sp.radius, rk, dx, dy);
                int nx = px + dx, ny = py + dy;
                if (nx == px && ny == py) continue;
                if (nx < 0 || nx >= W || ny < 0 || ny >= H || ny < bd.r0 || ny >= bd.r1) continue;
                size_t si = (size_t(ny) * W + nx) * B + b;
                bool nb = shiftable(src_grid, si);
                c += int(nb) + int(self || nb);  // fwd shift; inverse once the output is non-empty
            }
        }
        c = c > kCostBuckets - 1 ? kCostBuckets - 1 : c;
        cls[i] = uint8_t(c);
        bucket_count(c, counts);
    }
}

// Heaviest bucket first: offsets from the counts, positions by warp-aggregated
// cursors (counts[kCostBuckets + c]).
__global__ void k_cost_scatter(const uint8_t* cls, size_t n, uint32_t* counts, uint32_t* perm) {
    __shared__ uint32_t off[kCostBuckets];
    if (threadIdx.x == 0) {
        uint32_t o = 0;
        for (int c = kCostBuckets - 1; c >= 0; --c) {
            off[c] = o;
            o += counts[c];
        }
    }
    __syncthreads();
    size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t n_round = (n + 31) & ~size_t(31);
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n_round; i += stride) {
        if (i >= n) continue;
        int c = cls[i];
        unsigned peers = __match_any_sync(__activemask(), c);
        int leader = __ffs(peers) - 1;
        int lane = threadIdx.x & 31;
        uint32_t start = 0;
        if (lane == leader) start = atomicAdd(&counts[kCostBuckets + c], uint32_t(__popc(peers)));
        start = __shfl_sync(peers, start, leader);
        uint32_t rank = __popc(peers & ((1u << lane) - 1));
        perm[off[c] + start + rank] = uint32_t(i);
    }
}

// ---------------------------------------------------------------------------
// final shading (ris.hpp:108-111)

// final_shading (ris.hpp:108-111): f * (W * gate weight of the sample's
// length, or of its path velocity for Doppler gates)
__device__ __forceinline__ V3 shade_item(const ResStore& s, size_t i, double c, double w, int gate_vel = 0) {
    double W, M;
    int has;
    res_load_hdr(s, i, W, M, has);
    if (!has || W <= 0) return splat(0);
    const size_t row = res_row(s, i);
    double2 c1 = ld2r(s, 1, row), c2 = ld2r(s, 2, row), c3 = ld2r(s, 3, row);
    V3 f{c2.x, c2.y, c3.x};
    double gv = gate_vel ? ld2r(s, 22, row).x : c1.y;
    return f * (W * gate_w(c, w, gv));
}

__global__ void k_shade_gated(ResStore cur, int p0, int p1, double center, double width, int gate_vel,
                              double* image, double* accum) {
    for (int p = p0 + blockIdx.x * blockDim.x + threadIdx.x; p < p1; p += gridDim.x * blockDim.x) {
        V3 v = shade_item(cur, size_t(p), center, width, gate_vel);
        image[3 * size_t(p) + 0] = v.x;
        image[3 * size_t(p) + 1] = v.y;
        image[3 * size_t(p) + 2] = v.z;
        accum[3 * size_t(p) + 0] += v.x;
        accum[3 * size_t(p) + 1] += v.y;
        accum[3 * size_t(p) + 2] += v.z;
    }
}

__global__ void k_shade_transient(ResStore cur, size_t i0, size_t i1, HistSpec h, double* hist) {
    for (size_t it = i0 + blockIdx.x * size_t(blockDim.x) + threadIdx.x; it < i1;
         it += size_t(gridDim.x) * blockDim.x) {
        int b = int(it % h.bins);
        V3 v = shade_item(cur, it, bin_center(h, b), h.bw);
        if (v.x != 0 || v.y != 0 || v.z != 0) {
            hist[3 * it + 0] += v.x;
            hist[3 * it + 1] += v.y;
            hist[3 * it + 2] += v.z;
        }
    }
}

// Wide-band image of a transient histogram (pipeline.hpp:521-526): per pixel the
// sum over its B bins, times `scale` (1/frames).  One warp per pixel row
// segment; bins are contiguous per pixel so reads are coalesced.
__global__ void k_hist_image(const double* hist, int p0, int p1, int B, double scale, double* image) {
    int lane = threadIdx.x & 31;
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int p = p0 + warp; p < p1; p += nwarps) {
        const double* h = hist + 3 * size_t(p) * B;
        double sx = 0, sy = 0, sz = 0;
        for (int b = lane; b < B; b += 32) {
            sx += __ldcs(&h[3 * b + 0]);
            sy += __ldcs(&h[3 * b + 1]);
            sz += __ldcs(&h[3 * b + 2]);
        }
        for (int o = 16; o > 0; o >>= 1) {
            sx += __shfl_down_sync(0xffffffffu, sx, o);
            sy += __shfl_down_sync(0xffffffffu, sy, o);
            sz += __shfl_down_sync(0xffffffffu, sz, o);
        }
        if (lane == 0) {
            image[3 * size_t(p) + 0] = sx * scale;
            image[3 * size_t(p) + 1] = sy * scale;
            image[3 * size_t(p) + 2] = sz * scale;
        }
    }
}

// ---------------------------------------------------------------------------
// trace-only transient deposits (render_transient_plain, pipeline.hpp:531-571;
// TransientHistogram::deposit, transport.hpp:121-126): nested-loop walk
// (default; TOFR_TRACE=wave: the k_trace<PlainSink2> state machine).
#ifndef TOFR_PLAIN_HISTORY
#define TOFR_PLAIN_HISTORY 0
#endif

struct PlainSink {
    HistSpec h;
    int m_init;
    double* hist;
    double* img;
    size_t base, pix;
    uint32_t* n_dep;
    __device__ bool wants(double len) const { return bin_of(h, len) >= 0; }
    __device__ double walk_max() const { return h.t0 + (h.bins + 1) * h.bw; }
    __device__ void emit(const Cand& c, double mis, const RecSrc&) {
        if (!(c.pdf > 0)) return;
        V3 val = c.f * (mis / c.pdf / m_init);
        int b = bin_of(h, c.len);
        if (b < 0) return;
        hist_deposit(hist, img, base + b, pix, val);
        ++*n_dep;
    }
};

// Path tree of a plain deposit run (Tracer::trace_tree + emit_nee,
// transport.hpp:224-328, with build_rec = false and no ellipsoidal strategy,
// pipeline.hpp:535-555): the same operations as trace_tree / emit_nee in the
// same order, but only the current vertex is kept (no record is ever built,
// and without the ellipsoidal MIS no earlier vertex is read), so the walk
// needs no per-thread vertex history in local memory.
template <class Sink>
__device__ void trace_tree_deposit(const FrameView& F, const PathCfg& cfg, int px, int py, const GHit& g, Rng& rng,
                                   Sink& sink) {
    if (g.tri < 0) return;
    V3 d0 = primary_dir(F.cam, px, py);
    const GTriInfo& ti = F.tri[g.tri];
    WalkV x;
    x.p = F.cam.pos + d0 * g.t;
    x.n = ti.n;
    x.tri = g.tri;
    x.mat = ti.mat;
    x.wi = -d0;
    x.fw = splat(1);
    x.pdf = 1;
    x.len = g.t;
    const RecSrc none{nullptr, 0, nullptr, 0};
    for (int d = 1; d + 1 <= cfg.max_depth && d < kMaxVerts - 1; ++d) {
        const GMat& m = F.mats[x.mat];
        if (m.kind != MAT_MIRROR) {  // emit_nee at x
            Cand c;
            bool ok = true;
            if (F.light.regime == LIGHT_WIDE) {
                LightSample ls;
                ok = light_sample(F.light, x.p, ls);
                if (ok) {
                    c.len = x.len + ls.dist;
                    ok = sink.wants(c.len) && !occluded(F, x.p, F.light.pos);
                }
                if (ok) {
                    V3 f_at = eval_bsdf(m, x.n, x.wi, ls.dir);
                    double cos_v = fabs(dot(x.n, ls.dir));
                    c.f = x.fw * f_at * (cos_v) * ls.value;
                }
            } else {
                ok = F.lsub.valid;
                V3 dvec, wto;
                if (ok) {
                    dvec = F.lsub.pos - x.p;
                    double dist = norm(dvec);
                    ok = !(dist <= F.eps_ray * 2);
                    if (ok) {
                        wto = dvec / dist;
                        c.len = x.len + dist + F.lsub.chain_len;
                        ok = sink.wants(c.len) && !occluded(F, x.p, F.lsub.pos);
                    }
                }
                if (ok) {
                    V3 f_at = eval_bsdf(m, x.n, x.wi, wto);
                    V3 f_s = eval_bsdf(F.mats[F.lsub.mat], F.lsub.n, -wto, F.lsub.wo_light);
                    double gg = geom_term(x.p, x.n, F.lsub.pos, F.lsub.n);
                    c.f = x.fw * f_at * gg * f_s * F.lsub.power;
                }
            }
            if (ok && c.len > 0) {
                c.pdf = x.pdf;
                c.u = 0;
                c.depth = d + 1;
                if (luminance(c.f) > 0 && finite3(c.f)) sink.emit(c, 1.0, none);
            }
        }
        if (d + 2 > cfg.max_depth) break;
        if (cfg.walk_cutoff && x.len > sink.walk_max()) break;  // no later candidate can be wanted
        double surv = rr_survival(d, cfg.use_rr);
        if (surv < 1.0 && rng_next(rng) >= surv) break;
        BsdfSample bs = sample_bsdf(m, x.n, x.wi, rng);
        if (!bs.valid) break;
        Hit nh;
        if (!intersect(F, x.p, bs.wo, nh)) break;
        const GTriInfo& wt = F.tri[nh.tri];
        WalkV w;
        w.p = nh.pos;
        w.n = wt.n;
        w.tri = nh.tri;
        w.mat = wt.mat;
        w.wi = -bs.wo;
        double gt = geom_term(x.p, x.n, w.p, w.n);
        V3 fr_val = m.kind == MAT_MIRROR ? m.albedo : eval_bsdf(m, x.n, x.wi, bs.wo);
        w.fw = x.fw * fr_val * gt;
        double cos_w = fabs(dot(w.n, bs.wo));
        w.pdf = x.pdf * surv * bs.pdf * cos_w / (nh.t * nh.t);
        w.len = x.len + nh.t;
        x = w;
    }
}

#ifndef TOFR_PLAIN_MINB
#define TOFR_PLAIN_MINB 5
#endif
__global__ void __launch_bounds__(128, TOFR_PLAIN_MINB) k_hist_plain(FrameView F, Band bd, const GHit* gbuf, PathCfg cfg,
                                                    HistSpec h, int m_init, int frame_idx, double* hist,
                                                    double* img, unsigned long long* q) {
    extern __shared__ __align__(16) unsigned char smem[];
    size_t off = 0;
    stage_frame(F, smem, off);
    __syncthreads();
    int W = F.cam.w;
    size_t n = size_t(bd.y1 - bd.y0) * W;
    uint32_t n_dep = 0;
#if TOFR_PLAIN_HISTORY
    WalkV vh[kMaxVerts];
#endif
    TOFR_FOR_ITEMS(i, n, q) {
        int p = bd.y0 * W + int(i);
        int px = p % W, py = p / W;
        uint64_t pix = uint64_t(py) * W + px;
        PlainSink sink{h, m_init, hist, img, size_t(p) * h.bins, size_t(p), &n_dep};
        GHit g = gbuf[p];
        for (int s = 0; s < m_init; ++s) {
            Rng rng = rng_make(cfg.seed, uint64_t(frame_idx), pix, uint64_t(s), 0);
#if TOFR_PLAIN_HISTORY  // A/B variant: the generic walk with its vertex history
            Rng erng = rng_make(cfg.seed, uint64_t(frame_idx), pix, uint64_t(s), 2);
            NoEll ell;
            trace_tree(F, cfg, px, py, g, rng, erng, sink, vh, ell);
#else
            trace_tree_deposit(F, cfg, px, py, g, rng, sink);
#endif
        }
    }
    work_add(cfg.work, WK_DEPOSITS, n_dep);
}

// ---------------------------------------------------------------------------
// brute-force gated reference (reference_gated_pixel, transport.hpp:591-617)

struct RefSink {
    double center, width;
    V3 est;
    __device__ bool wants(double len) const { return gate_w(center, width, len) > 0; }
    __device__ double walk_max() const { return center + width; }
    __device__ void emit(const Cand& c, double mis, const RecSrc&) {
        double w = gate_w(center, width, c.len);
        if (w > 0 && c.pdf > 0) est = est + c.f * (mis * w / c.pdf);
    }
};

__global__ void __launch_bounds__(128) k_reference(FrameView F, Band bd, const GHit* gbuf, PathCfg cfg,
                                                   double center, double width, int spp, uint64_t frame_key,
                                                   double* mean, double* se, unsigned long long* q) {
    extern __shared__ __align__(16) unsigned char smem[];
    size_t off = 0;
    stage_frame(F, smem, off);
    __syncthreads();
    int W = F.cam.w;
    WalkV v[kMaxVerts];
    NoEll ell;
    size_t n = size_t(bd.y1 - bd.y0) * W;
    TOFR_FOR_ITEMS(i, n, q) {
        int p = bd.y0 * W + int(i);
        int px = p % W, py = p / W;
        uint64_t pix = uint64_t(py) * W + px;
        GHit g = gbuf[p];
        V3 sum = splat(0), sum2 = splat(0);
        for (int s = 0; s < spp; ++s) {
            RefSink sink{center, width, splat(0)};
            Rng rng = rng_make(cfg.seed, frame_key, pix, uint64_t(s), 0);
            Rng erng = rng_make(cfg.seed, frame_key, pix, uint64_t(s), 2);
            trace_tree(F, cfg, px, py, g, rng, erng, sink, v, ell);
            sum = sum + sink.est;
            sum2 = sum2 + sink.est * sink.est;
        }
        V3 m = sum / double(spp);
        V3 var = sum2 / double(spp) - m * m;
        var = V3{dmax(0.0, var.x), dmax(0.0, var.y), dmax(0.0, var.z)};
        mean[3 * size_t(p) + 0] = m.x;
        mean[3 * size_t(p) + 1] = m.y;
        mean[3 * size_t(p) + 2] = m.z;
        se[3 * size_t(p) + 0] = sqrt(var.x / spp);
        se[3 * size_t(p) + 1] = sqrt(var.y / spp);
        se[3 * size_t(p) + 2] = sqrt(var.z / spp);
    }
}

// ---------------------------------------------------------------------------
// debug / parity probes

__global__ void k_probe_rays(FrameView F, const double* rays, int n, int mode, double* out_t, int* out_tri) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* r = rays + 8 * size_t(i);  // o.xyz, d.xyz, tmin, tmax
    V3 o{r[0], r[1], r[2]}, d{r[3], r[4], r[5]};
    if (mode == 0) {
        Hit h;
        if (trace_closest(F, o, d, r[6], r[7], h)) {
            out_t[i] = h.t;
            out_tri[i] = h.tri;
        } else {
            out_t[i] = kInf;
            out_tri[i] = -1;
        }
    } else {
        // occluded(a = o, b = d)
        out_tri[i] = occluded(F, o, d) ? 1 : 0;
        out_t[i] = 0;
    }
}

// Self-test of the shared-reciprocal division (v3_div_shared / ddiv_by,
// tofr_core.h) against the compiler's a / b: counts quotients whose bits
// differ.  Operands: raw 64-bit patterns (every exponent, subnormals, inf, NaN)
// for odd k, and geometry-range values (|a| < 2^20, |b| in [2^-30, 2^30]) for
// even k; the three numerators of a V3 share one divisor.
__device__ __forceinline__ uint64_t st_mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__global__ void k_selftest_div(uint64_t n, uint64_t seed, unsigned long long* bad) {
    unsigned long long local = 0;
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n; k += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t h = st_mix(seed ^ (k * 0x2545f4914f6cdd1dull));
        double a[3], b;
        if (k & 1) {
            b = __longlong_as_double((long long)st_mix(h));
            for (int j = 0; j < 3; ++j) a[j] = __longlong_as_double((long long)st_mix(h + 1 + j));
        } else {
            uint64_t hb = st_mix(h);
            double m = 1.0 + double(hb >> 12) * 0x1p-52;
            b = ldexp(m, int((hb & 63) - 30)) * ((hb >> 7) & 1 ? -1.0 : 1.0);
            for (int j = 0; j < 3; ++j) {
                uint64_t ha = st_mix(h + 1 + j);
                a[j] = (double(ha >> 11) * 0x1p-53 * 2.0 - 1.0) * ldexp(1.0, int(ha & 31) - 10);
            }
        }
        V3 q = v3_div_shared(V3{a[0], a[1], a[2]}, b);
        double ref[3] = {a[0] / b, a[1] / b, a[2] / b};
        double got[3] = {q.x, q.y, q.z};
        for (int j = 0; j < 3; ++j)
            local += __double_as_longlong(got[j]) != __double_as_longlong(ref[j]);
    }
    if (local) atomicAdd(bad, local);
}

// FP64 issue peak (the FP64 roofline's denominator, measured, not a data-sheet
// number): 8 independent DFMA chains per thread, enough warps per SM to hide
// the pipe latency.  flops = 2 per DFMA.
__global__ void __launch_bounds__(256) k_fp64_peak(double* out, int iters, double m, double c) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
           a7 = a0 + 7;
    for (int i = 0; i < iters; ++i) {
        a0 = __fma_rn(a0, m, c);
        a1 = __fma_rn(a1, m, c);
        a2 = __fma_rn(a2, m, c);
        a3 = __fma_rn(a3, m, c);
        a4 = __fma_rn(a4, m, c);
        a5 = __fma_rn(a5, m, c);
        a6 = __fma_rn(a6, m, c);
        a7 = __fma_rn(a7, m, c);
    }
    double sum = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (sum == 12345.678) out[0] = sum;  // keeps the chains alive
}
double measure_fp64_peak_gflops(cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out = nullptr;
    if (cudaMalloc(&out, 8) != cudaSuccess) return 0;
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0, s);
        k_fp64_peak<<<blocks, threads, 0, s>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 8.0 * double(iters) * blocks * threads;
        if (rep > 0 && ms > 0) best = fl / (ms * 1e-3) / 1e9 > best ? fl / (ms * 1e-3) / 1e9 : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return best;
}

void launch_selftest_div(uint64_t n, uint64_t seed, unsigned long long* bad, cudaStream_t s) {
    KScope ks("k_selftest_div", s);
    k_selftest_div<<<148 * 8, 256, 0, s>>>(n, seed, bad);
}

// ---------------------------------------------------------------------------
// halo staging (row-band sharding): one 16 B chunk per thread, coalesced on
// both sides

__global__ void k_halo_pack(ResStore grid, size_t item0, size_t n, double2* buf) {
    size_t total = n * kResChunks;
    for (size_t j = blockIdx.x * size_t(blockDim.x) + threadIdx.x; j < total; j += size_t(gridDim.x) * blockDim.x) {
        size_t c = j / n, i = j % n;
        buf[j] = __ldcg(&grid.base[c * grid.stride + item0 + i]);
    }
}

__global__ void k_halo_unpack(ResStore grid, size_t item0, size_t n, const double2* buf) {
    size_t total = n * kResChunks;
    for (size_t j = blockIdx.x * size_t(blockDim.x) + threadIdx.x; j < total; j += size_t(gridDim.x) * blockDim.x) {
        size_t c = j / n, i = j % n;
        __stcg(&grid.base[c * grid.stride + item0 + i], __ldcg(&buf[j]));
    }
}

// Sparse grids travel compacted (HaloLayout): the dense header plane of the
// halo rows, then only the non-empty reservoirs' sample rows with their item
// offsets.  Rows are handed out warp-aggregated so consecutive lanes write
// consecutive payload rows (coalesced chunk planes).
struct HaloLayout {
    unsigned int* count;  // payload rows
    double2* hdr;         // n headers
    uint32_t* idx;        // cap item offsets
    double2* pl;          // chunk c (1..23) of payload row r at pl[(c - 1) * cap + r]
    size_t cap;
};
__device__ __forceinline__ HaloLayout halo_layout(double2* buf, size_t n, size_t cap) {
    HaloLayout h;
    h.count = reinterpret_cast<unsigned int*>(buf);
    h.hdr = buf + 1;
    h.idx = reinterpret_cast<uint32_t*>(buf + 1 + n);
    h.pl = buf + 1 + n + (cap * 4 + 15) / 16;
    h.cap = cap;
    return h;
}

__global__ void k_halo_pack_sparse(ResStore grid, size_t item0, size_t n, double2* buf, size_t cap) {
    HaloLayout h = halo_layout(buf, n, cap);
    const int lane = threadIdx.x & 31;
    size_t n_round = (n + 31) / 32 * 32;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n_round; i += size_t(gridDim.x) * blockDim.x) {
        bool live = i < n;
        double2 c0 = live ? __ldcg(&grid.base[item0 + i]) : make_double2(0.0, 0.0);
        if (live) __stcg(&h.hdr[i], c0);
        bool ne = live && c0.x > 0;
        unsigned m = __ballot_sync(0xffffffffu, ne);
        unsigned r0 = 0;
        if (m && lane == __ffs(m) - 1) r0 = atomicAdd(h.count, unsigned(__popc(m)));
        r0 = __shfl_sync(0xffffffffu, r0, __ffs(m ? m : 1u) - 1);
        if (!ne) continue;
        size_t r = r0 + __popc(m & ((1u << lane) - 1));
        if (r >= cap) {
            atomicOr(grid.err, kErrHalo);
            continue;
        }
        __stcg(&h.idx[r], uint32_t(i));
        const size_t row = res_row(grid, item0 + i);
        for (int c = 1; c < grid.planes; ++c) __stcg(&h.pl[size_t(c - 1) * cap + r], ld2r(grid, c, row));
    }
}

__global__ void k_halo_unpack_hdr(ResStore grid, size_t item0, size_t n, const double2* buf, size_t cap) {
    HaloLayout h = halo_layout(const_cast<double2*>(buf), n, cap);
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        __stcg(&grid.base[item0 + i], __ldcg(&h.hdr[i]));
}

__global__ void k_halo_unpack_rows(ResStore grid, size_t item0, size_t n, const double2* buf, size_t cap) {
    HaloLayout h = halo_layout(const_cast<double2*>(buf), n, cap);
    size_t cnt = min(size_t(__ldcg(h.count)), cap);
    for (size_t r = blockIdx.x * size_t(blockDim.x) + threadIdx.x; r < cnt; r += size_t(gridDim.x) * blockDim.x) {
        const size_t row = res_row_w(grid, item0 + __ldcg(&h.idx[r]));
        for (int c = 1; c < grid.planes; ++c) st2r(grid, c, row, __ldcg(&h.pl[size_t(c - 1) * cap + r]));
    }
}

// ---------------------------------------------------------------------------
// launchers

// One wave of resident CTAs for a persistent kernel (occupancy calculator,
// cached per kernel), never more than the items need.
int persistent_grid(const void* kernel, int block, size_t smem, size_t n) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
    if (per_sm < 1) per_sm = 1;
    size_t need = (n + block - 1) / block;
    size_t g = size_t(sms) * per_sm;
    if (g > need) g = need;
    return int(g < 1 ? 1 : g);
}

static int grid_for(size_t n, int block) {
    size_t g = (n + block - 1) / block;
    if (g > 148 * 64) g = 148 * 64;
    if (g < 1) g = 1;
    return int(g);
}

void set_gauss_rule(const double* x, const double* w, cudaStream_t s) {
    cudaMemcpyToSymbolAsync(c_gl_x, x, 32 * sizeof(double), 0, cudaMemcpyHostToDevice, s);
    cudaMemcpyToSymbolAsync(c_gl_w, w, 32 * sizeof(double), 0, cudaMemcpyHostToDevice, s);
}

static size_t band_pixels(const Band& bd, int W) { return size_t(bd.y1 - bd.y0) * W; }

// TOFR_TRACE=legacy keeps the nested-loop trace kernels (A/B and debugging)
static bool trace_wave() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("TOFR_TRACE");
        v = (e && std::strcmp(e, "legacy") == 0) ? 0 : 1;
    }
    return v == 1;
}

void launch_gbuffer(const FrameView& F, const Band& bd, GHit* g, cudaStream_t s) {
    size_t n = size_t(bd.r1 - bd.r0) * F.cam.w;
    if (!n) return;
    {
        KScope ks("k_gbuffer", s);
        k_gbuffer<<<grid_for(n, 256), 256, frame_smem_bytes(F), s>>>(F, bd, g);
    }
}

// zeroed work counter + persistent launch configuration
#define TOFR_PERSISTENT(kernel, n, smem) \
    cudaMemsetAsync(q, 0, sizeof(unsigned long long), s); \
    kernel<<<persistent_grid(reinterpret_cast<const void*>(kernel), 128, smem, n), 128, smem, s>>>

void launch_init_gated(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg,
                       const InitParams& ip, int frame_idx, ResStore cur, unsigned long long* q, cudaStream_t s,
                       const EllScratch* es) {
    size_t n = band_pixels(bd, F.cam.w);
    if (!n) return;
    if (ip.mode == INIT_DIRECT && !cfg.ellipsoidal && trace_wave()) {
        launch_trace_gated(F, bd, g, cfg, ip.m_init, ip.center, ip.width, frame_idx, cur, q, s);
        return;
    }
    size_t sm = frame_smem_bytes(F);
    EllScratch none{};
    const bool wave_ell = cfg.ellipsoidal && ip.mode == INIT_ELLIPSOIDAL && es && es->jobs;
    if (wave_ell) {
        cudaMemsetAsync(es->count, 0, sizeof(unsigned int), s);
        {
            KScope ks("k_ell_plan", s);
            TOFR_PERSISTENT(k_ell_plan, n, sm)(F, bd, g, cfg, ip.m_init, frame_idx, *es, q);
        }
        {
            cudaMemsetAsync(q, 0, sizeof(unsigned long long), s);
            KScope ks("k_ell_arcs", s);
            k_ell_arcs<<<persistent_grid(reinterpret_cast<const void*>(k_ell_arcs), 256, 0, n * 32), 256, 0, s>>>(
                F, *es, q);
        }
    }
    {
        KScope ks("k_init_gated", s);
        TOFR_PERSISTENT(k_init_gated, n, sm)(F, bd, g, cfg, ip, frame_idx, cur, q, wave_ell ? *es : none);
    }
}

void launch_init_transient(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg,
                           const InitParams& ip, const HistSpec& h, int frame_idx, ResStore cur,
                           unsigned long long* q, cudaStream_t s) {
    size_t n = band_pixels(bd, F.cam.w);
    if (!n) return;
    if (trace_wave()) {
        launch_trace_transient(F, bd, g, cfg, ip.m_init, h, frame_idx, cur, q, s);
        return;
    }
    size_t sm = frame_smem_bytes(F);
    {
        KScope ks("k_init_transient", s);
        TOFR_PERSISTENT(k_init_transient, n, sm)(F, bd, g, cfg, ip, h, frame_idx, cur, q);
    }
}

static void order_items(const uint8_t* cls, size_t n, const WorkOrder& wo, cudaStream_t s) {
    {
        KScope ks("k_cost_scatter", s);
        k_cost_scatter<<<grid_for(n, 256), 256, 0, s>>>(cls, n, wo.counts, wo.perm);
    }
}

void launch_temporal(const FrameView& Fc, const Band& bd, const GHit* gc, const FrameView& Fp, const GHit* gp,
                     const PathCfg& cfg, const GateGrid& cg, const GateGrid& pg, int frame_idx,
                     ResStore cur, ResStore prev, const WorkOrder& wo, unsigned long long* ctr,
                     unsigned long long* q, cudaStream_t s) {
    size_t n = band_pixels(bd, Fc.cam.w) * (cg.transient ? cg.h.bins : 1);
    if (!n) return;
    const uint32_t* perm = nullptr;
    if (wo.perm) {
        cudaMemsetAsync(wo.counts, 0, 2 * kCostBuckets * sizeof(uint32_t), s);
        {
            KScope ks("k_cost_temporal", s);
            k_cost_temporal<<<grid_for(n, 256), 256, 0, s>>>(Fc, bd, gc, Fp, cg, cur, prev, wo.cls, wo.counts);
        }
        order_items(wo.cls, n, wo, s);
        perm = wo.perm;
    }
    size_t sm = frame_smem_bytes(Fc) + frame_smem_bytes(Fp);
    {
        KScope ks("k_temporal", s);
        TOFR_PERSISTENT(k_temporal, n, sm)(Fc, bd, gc, Fp, gp, cfg, cg, pg, frame_idx, cur, prev, perm, ctr, q);
    }
}

void launch_spatial(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, const GateGrid& gg,
                    const SpatialParams& sp, int pass, int frame_idx, ResStore src, ResStore dst,
                    const WorkOrder& wo, const SpatialScratch* sc, unsigned long long* ctr, unsigned long long* q,
                    cudaStream_t s) {
    size_t n = band_pixels(bd, F.cam.w) * (gg.transient ? gg.h.bins : 1);
    if (!n) return;
    size_t sm = frame_smem_bytes(F);
    if (sc && sp.neighbors > 0 && sp.radius > 0) {
        cudaMemsetAsync(sc->count, 0, sizeof(uint32_t), s);
        cudaMemsetAsync(sc->ok, 0, n * size_t(sp.neighbors), s);
        {
            KScope ks("k_spatial_fwd_list", s);
            k_spatial_fwd_list<<<grid_for(n, 256), 256, 0, s>>>(F, bd, cfg, gg, sp, pass, frame_idx, src, *sc);
        }
        size_t jobs_max = n * size_t(sp.neighbors);
        {
            KScope ks("k_spatial_fwd", s);
            TOFR_PERSISTENT(k_spatial_fwd, jobs_max, sm)(F, bd, g, cfg, gg, sp, pass, frame_idx, src, *sc, ctr, q);
        }
        for (int j = 0; j < sp.neighbors; ++j) {
            {
                KScope ks("k_spatial_merge", s);
                TOFR_PERSISTENT(k_spatial_merge, n, sm)(F, bd, g, cfg, gg, sp, pass, j, frame_idx, src, dst, *sc, q);
            }
        }
        return;
    }
    const uint32_t* perm = nullptr;
    if (wo.perm) {
        cudaMemsetAsync(wo.counts, 0, 2 * kCostBuckets * sizeof(uint32_t), s);
        {
            KScope ks("k_cost_spatial", s);
            k_cost_spatial<<<grid_for(n, 256), 256, 0, s>>>(F, bd, cfg, gg, sp, pass, frame_idx, src, wo.cls,
                                                             wo.counts);
        }
        order_items(wo.cls, n, wo, s);
        perm = wo.perm;
    }
    {
        KScope ks("k_spatial", s);
        TOFR_PERSISTENT(k_spatial, n, sm)(F, bd, g, cfg, gg, sp, pass, frame_idx, src, dst, perm, ctr, q);
    }
}

void launch_binreuse(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, const HistSpec& h,
                     int frame_idx, ResStore src, ResStore dst, unsigned long long* ctr, unsigned long long* q,
                     cudaStream_t s) {
    size_t n = band_pixels(bd, F.cam.w) * h.bins;
    if (!n) return;
    size_t sm = frame_smem_bytes(F);
    {
        KScope ks("k_binreuse", s);
        TOFR_PERSISTENT(k_binreuse, n, sm)(F, bd, g, cfg, h, frame_idx, src, dst, ctr, q);
    }
}

void launch_shade_gated(ResStore cur, const Band& bd, int W, double center, double width, int gate_vel,
                        double* image, double* accum, cudaStream_t s) {
    size_t n = band_pixels(bd, W);
    if (!n) return;
    {
        KScope ks("k_shade_gated", s);
        k_shade_gated<<<grid_for(n, 256), 256, 0, s>>>(cur, bd.y0 * W, bd.y1 * W, center, width, gate_vel, image,
                                                                 accum);
    }
}

void launch_shade_transient(ResStore cur, const Band& bd, int W, const HistSpec& h, double* hist,
                            cudaStream_t s) {
    size_t n = band_pixels(bd, W) * h.bins;
    if (!n) return;
    size_t i0 = size_t(bd.y0) * W * h.bins;
    {
        KScope ks("k_shade_transient", s);
        k_shade_transient<<<grid_for(n, 256), 256, 0, s>>>(cur, i0, i0 + n, h, hist);
    }
}

void launch_hist_plain(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, const HistSpec& h,
                       int m_init, int frame_idx, double* hist, double* img, unsigned long long* q,
                       cudaStream_t s) {
    size_t n = band_pixels(bd, F.cam.w);
    if (!n) return;
    // nested-loop walk without vertex history (trace_tree_deposit): measured
    // faster than the path-tree state machine for plain deposits, where every
    // candidate in the histogram range is traced and lanes stay in step
    // (C4 plain 0.99 vs 1.17 ms per frame); the state machine with TOFR_TRACE=wave
    if (std::getenv("TOFR_TRACE") && std::strcmp(std::getenv("TOFR_TRACE"), "wave") == 0) {
        launch_trace_plain(F, bd, g, cfg, h, m_init, frame_idx, hist, img, q, s);
        return;
    }
    size_t sm = frame_smem_bytes(F);
    {
        KScope ks("k_hist_plain", s);
        TOFR_PERSISTENT(k_hist_plain, n, sm)(F, bd, g, cfg, h, m_init, frame_idx, hist, img, q);
    }
}

// image = accumulator * scale (plain sessions keep the wide-band image per deposit)
__global__ void k_scale3(const double* a, size_t n, double scale, double* out) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        out[i] = a[i] * scale;
}
void launch_scale3(const double* a, size_t n_pixels, double scale, double* out, cudaStream_t s) {
    if (!n_pixels) return;
    KScope ks("k_scale3", s);
    k_scale3<<<grid_for(n_pixels * 3, 256), 256, 0, s>>>(a, n_pixels * 3, scale, out);
}

// device-to-device copy of an image on the SMs (the copy engine's D2D path
// measured several times slower, on the frame's critical path)
__global__ void k_copy_f64(const double* a, size_t n, double* out) {
    const size_t n2 = n / 2;
    const double2* a2 = reinterpret_cast<const double2*>(a);
    double2* o2 = reinterpret_cast<double2*>(out);
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n2; i += size_t(gridDim.x) * blockDim.x)
        __stcs(&o2[i], __ldcs(&a2[i]));
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) out[n - 1] = a[n - 1];
}
void launch_copy_f64(const double* a, size_t n, double* out, cudaStream_t s) {
    if (!n) return;
    KScope ks("k_copy_f64", s);
    k_copy_f64<<<grid_for(n / 2 + 1, 256), 256, 0, s>>>(a, n, out);
}

void launch_reference(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, double center,
                      double width, int spp, uint64_t frame_key, double* mean, double* se, unsigned long long* q,
                      cudaStream_t s) {
    size_t n = band_pixels(bd, F.cam.w);
    if (!n) return;
    if (trace_wave()) {
        launch_trace_reference(F, bd, g, cfg, center, width, spp, frame_key, mean, se, q, s);
        return;
    }
    size_t sm = frame_smem_bytes(F);
    {
        KScope ks("k_reference", s);
        TOFR_PERSISTENT(k_reference, n, sm)(F, bd, g, cfg, center, width, spp, frame_key, mean, se, q);
    }
}

void launch_hist_image(const double* hist, const Band& bd, int W, int B, double scale, double* image,
                       cudaStream_t s) {
    size_t n = band_pixels(bd, W);
    if (!n) return;
    {
        KScope ks("k_hist_image", s);
        k_hist_image<<<grid_for(n * 32, 256), 256, 0, s>>>(hist, bd.y0 * W, bd.y1 * W, B, scale, image);
    }
}

size_t halo_bytes(size_t n_items, size_t cap, bool sparse) {
    if (!n_items) return 0;
    if (!sparse) return n_items * kResChunks * 16;
    return 16 + n_items * 16 + (cap * 4 + 15) / 16 * 16 + (kResChunks - 1) * cap * 16;
}

void launch_halo_pack(ResStore grid, size_t item0, size_t n_items, double2* buf, size_t cap, cudaStream_t s) {
    if (!n_items) return;
    if (grid.slot) {
        cudaMemsetAsync(buf, 0, 16, s);
        KScope ks("k_halo_pack_sparse", s);
        k_halo_pack_sparse<<<grid_for(n_items, 256), 256, 0, s>>>(grid, item0, n_items, buf, cap);
        return;
    }
    KScope ks("k_halo_pack", s);
    k_halo_pack<<<grid_for(n_items * kResChunks, 256), 256, 0, s>>>(grid, item0, n_items, buf);
}
void launch_halo_unpack(ResStore grid, size_t item0, size_t n_items, const double2* buf, size_t cap,
                        cudaStream_t s) {
    if (!n_items) return;
    if (grid.slot) {
        {
            KScope ks("k_halo_unpack_hdr", s);
            k_halo_unpack_hdr<<<grid_for(n_items, 256), 256, 0, s>>>(grid, item0, n_items, buf, cap);
        }
        KScope ks("k_halo_unpack_rows", s);
        k_halo_unpack_rows<<<grid_for(cap, 256), 256, 0, s>>>(grid, item0, n_items, buf, cap);
        return;
    }
    KScope ks("k_halo_unpack", s);
    k_halo_unpack<<<grid_for(n_items * kResChunks, 256), 256, 0, s>>>(grid, item0, n_items, buf);
}

void launch_probe_rays(const FrameView& F, const double* rays, int n, int mode, double* out_t, int* out_tri,
                       cudaStream_t s) {
    {
        KScope ks("k_probe_rays", s);
        k_probe_rays<<<(n + 127) / 128, 128, 0, s>>>(F, rays, n, mode, out_t, out_tri);
    }
}

}  // namespace tofr_b200
