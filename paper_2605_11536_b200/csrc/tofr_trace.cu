// tofr_trace.cu -- path-tree tracing (Tracer::trace_tree + emit_nee,
// transport.hpp:224-328) as a per-lane state machine.
//
// A path tree alternates shadow rays (NEE at every non-delta vertex) and
// extension rays.  Written as nested loops per pixel, the lanes of a warp drift
// apart: some are in the NEE branch, some extend, some start the next tree, and
// the two traversal call sites run one after the other with a few lanes each.
// Here every lane owns one pixel at a time and, in every iteration of the loop,
//
//   1. prepares at most one ray (advancing its tree through any steps that
//      need no ray: culled NEE candidates, mirror vertices, finished trees,
//      the next pixel -- lanes refill from a per-launch work counter);
//   2. traces it through ONE traversal call shared by all lanes
//      (trace_ray_impl: closest hit or first hit on the shadow segment);
//   3. consumes the result (emit the NEE candidate, or add the new vertex).
//
// Same operations per path in the same order, same RNG draws (walk stream lane
// 0, RIS pick stream lane 9), same candidate emission order: results are
// identical to the nested-loop trace.  The vertex history needed by lazily
// built reconnection records (build_record) lives in a per-lane local array.
//
// Sinks: RIS into one gated reservoir (initial sampling, pipeline.hpp:100-135),
// RIS into per-bin transient reservoirs (pipeline.hpp:421-445), plain histogram
// deposits (render_transient_plain, pipeline.hpp:531-571) and the brute-force
// gated reference (transport.hpp:591-617).
#include <cuda_runtime.h>

#include <type_traits>

#define TOFR_OUTLINE_MATH 0
#ifndef TOFR_TRACE_SHARED_DIV
#define TOFR_TRACE_SHARED_DIV 0
#endif
#define TOFR_SHARED_DIV TOFR_TRACE_SHARED_DIV

#include "ktime.h"
#include "tofr_kcommon.cuh"
#include "tofr_store.cuh"

#ifndef TOFR_TRACE_MINB
#define TOFR_TRACE_MINB 4
#endif
#ifndef TOFR_TRACE_BLOCK
#define TOFR_TRACE_BLOCK 128
#endif


namespace tofr_b200 {

// ---------------------------------------------------------------------------
// sinks

// gated grids are never sparse: a store view the compiler knows is dense
__device__ __forceinline__ ResStore dense(ResStore s) {
    s.slot = nullptr;
    return s;
}

// RIS into the pixel's gated reservoir; the winning sample's record is written
// to the grid when it wins, chunk 0 (W, M) when the pixel is done.
// VEL: velocity (Doppler) gate, the gated quantity is the path velocity u
template <bool VEL>
struct GatedSink {
    ResStore cur;
    double center, width, inv;
    double w_sum, phat;
    int has;
    Rng pick;
    size_t item;
    // the pick stream's counter carried between RIS runs of one pixel (the
    // shrink initialiser's rough then fine runs share the stream): read at
    // begin, written at end, indexed by item - pbase (null: a fresh stream)
    const uint64_t* pick_in = nullptr;
    uint64_t* pick_out = nullptr;
    size_t pbase = 0;
    __device__ void begin(const PathCfg& cfg, uint64_t fk, uint64_t pix, size_t p, int) {
        w_sum = 0;
        phat = 0;
        has = 0;
        pick = rng_make(cfg.seed, fk, pix, 0, 9);
        if (pick_in) pick.ctr = pick_in[p - pbase];
        item = p;
    }
    __device__ void tree_begin() {}
    __device__ void tree_end() {}
    __device__ bool wants(double len, double u) const { return gate_w(center, width, VEL ? u : len) > 0; }
    // lengths only grow along a walk: beyond this no candidate of the tree can
    // be in the gate (a full width of margin over center + width / 2); velocity
    // gates are not monotone
    __device__ double walk_max() const { return VEL ? kInf : center + width; }
    __device__ void emit(const FrameView& F, const Cand& c, double mis, const RecSrc& rs) {
        double p = luminance(c.f) * gate_w(center, width, VEL ? c.u : c.len);
        if (p <= 0 || !(c.pdf > 0)) return;
        double w = mis * inv * p / c.pdf;
        if (!isfinite(w) || w < 0) return;
        if (w <= 0) return;
        w_sum += w;
        if (rng_next(pick) * w_sum < w) {
            Res r;
            r.W = w_sum;  // chunk 0 is rewritten by end()
            r.M = 1;
            r.has = 1;
            r.phat = p;
            r.y.f = c.f;
            r.y.len = c.len;
            r.y.u = c.u;
            r.y.depth = c.depth;
            build_record<VEL>(F, rs, r.y.rec);
            res_store(dense(cur), item, r, VEL);
            has = 1;
            phat = p;
        }
    }
    __device__ void end() {
        double W = (has && phat > 0) ? w_sum / phat : 0;
        res_store_w(dense(cur), item, W, 1.0);
        if (pick_out) pick_out[item - pbase] = pick.ctr;
    }
    __device__ void flush(unsigned long long*) {}
};

// RIS into per-(pixel, bin) reservoirs: chunk 0 holds (w_sum, -) during the
// launch (zeroed before it), k_ris_finalize turns it into (W, 1).
struct BinsSink {
    ResStore st;
    HistSpec h;
    double inv;
    Rng pick;
    size_t base;
    __device__ void begin(const PathCfg& cfg, uint64_t fk, uint64_t pix, size_t p, int) {
        pick = rng_make(cfg.seed, fk, pix, 0, 9);
        base = p * size_t(h.bins);
    }
    __device__ void tree_begin() {}
    __device__ void tree_end() {}
    __device__ bool wants(double len, double) const {
        int b = bin_of(h, len);
        return b >= 0 && gate_w(bin_center(h, b), h.bw, len) > 0;
    }
    __device__ double walk_max() const { return h.t0 + (h.bins + 1) * h.bw; }
    __device__ void emit(const FrameView& F, const Cand& c, double mis, const RecSrc& rs) {
        int b = bin_of(h, c.len);
        if (b < 0 || !(c.pdf > 0)) return;
        double p = luminance(c.f) * gate_w(bin_center(h, b), h.bw, c.len);
        if (p <= 0) return;
        double w = mis * inv * p / c.pdf;
        if (!isfinite(w) || w < 0) return;
        if (w <= 0) return;
        size_t i = base + b;
        double2 c0 = ld2(st, 0, i);  // (w_sum, -)
        double w_sum = c0.x + w;
        st2(st, 0, i, w_sum, c0.y);
        if (rng_next(pick) * w_sum < w) {
            Res r;
            r.W = w_sum;
            r.M = c0.y;
            r.has = 1;
            r.phat = p;
            r.y.f = c.f;
            r.y.len = c.len;
            r.y.u = c.u;
            r.y.depth = c.depth;
            build_record<false>(F, rs, r.y.rec);
            res_store(st, i, r);
        }
    }
    __device__ void end() {}
    __device__ void flush(unsigned long long*) {}
};

// TransientHistogram::deposit of every candidate (f * mis / pdf / m_init,
// pipeline.hpp:547-556, transport.hpp:121-126) -- see hist_deposit
struct PlainSink2 {
    HistSpec h;
    int m_init;
    double* hist;  // 32 B bin records (HistBin)
    double* img;   // per-pixel wide-band accumulator (3 doubles)
    size_t base, pix;
    uint32_t deposits;
    __device__ void begin(const PathCfg&, uint64_t, uint64_t, size_t p, int) {
        base = p * size_t(h.bins);
        pix = p;
    }
    __device__ void tree_begin() {}
    __device__ void tree_end() {}
    __device__ bool wants(double len, double) const { return bin_of(h, len) >= 0; }
    __device__ void emit(const FrameView&, const Cand& c, double mis, const RecSrc&) {
        if (!(c.pdf > 0)) return;
        V3 val = c.f * (mis / c.pdf / m_init);
        int b = bin_of(h, c.len);
        if (b < 0) return;
        hist_deposit(hist, img, base + b, pix, val);
        ++deposits;
    }
    __device__ double walk_max() const { return h.t0 + (h.bins + 1) * h.bw; }
    __device__ void end() {}
    __device__ void flush(unsigned long long* work) { work_add(work, WK_DEPOSITS, deposits); }
};

// reference_gated_pixel: per-tree estimate, mean and standard error
struct RefSink2 {
    double center, width;
    double* mean;
    double* se;
    V3 est, sum, sum2;
    size_t item;
    int spp;
    __device__ void begin(const PathCfg&, uint64_t, uint64_t, size_t p, int trees) {
        sum = splat(0);
        sum2 = splat(0);
        item = p;
        spp = trees;
    }
    __device__ void tree_begin() { est = splat(0); }
    __device__ void tree_end() {
        sum = sum + est;
        sum2 = sum2 + est * est;
    }
    __device__ bool wants(double len, double) const { return gate_w(center, width, len) > 0; }
    __device__ void emit(const FrameView&, const Cand& c, double mis, const RecSrc&) {
        double w = gate_w(center, width, c.len);
        if (w > 0 && c.pdf > 0) est = est + c.f * (mis * w / c.pdf);
    }
    __device__ double walk_max() const { return center + width; }
    __device__ void end() {
        V3 m = sum / double(spp);
        V3 var = sum2 / double(spp) - m * m;
        var = V3{dmax(0.0, var.x), dmax(0.0, var.y), dmax(0.0, var.z)};
        mean[3 * item + 0] = m.x;
        mean[3 * item + 1] = m.y;
        mean[3 * item + 2] = m.z;
        se[3 * item + 0] = sqrt(var.x / spp);
        se[3 * item + 1] = sqrt(var.y / spp);
        se[3 * item + 2] = sqrt(var.z / spp);
    }
    __device__ void flush(unsigned long long*) {}
};

// ---------------------------------------------------------------------------
// the state machine

enum : int { ST_IDLE = 0, ST_NEE = 1, ST_EXT = 2, ST_SHADOW = 3, ST_EXTEND = 4 };

template <class Sink, bool VEL>
__global__ void __launch_bounds__(TOFR_TRACE_BLOCK, TOFR_TRACE_MINB * 128 / TOFR_TRACE_BLOCK)
    k_trace(FrameView F, Band bd, const GHit* gbuf, PathCfg cfg, int trees, uint64_t frame_key, Sink proto,
            unsigned long long* q) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ FrameView sF;
    {
        size_t off = 0;
        stage_frame(F, smem, off);
        if (threadIdx.x == 0) sF = F;
        __syncthreads();
    }
    const FrameView& Fs = sF;
    const int W = Fs.cam.w;
    const size_t n = size_t(bd.y1 - bd.y0) * W;
    const int lane = threadIdx.x & 31;
    const double eps = Fs.eps_ray;
    const bool wide = Fs.light.regime == LIGHT_WIDE;

    Sink sk = proto;
    WalkV v[kMaxVerts];  // vertex history of the current tree (build_record)
    int state = ST_IDLE;
    bool exhausted = false;
    int px = 0, py = 0, s = 0, d = 1;
    GHit g{0, -1, 0};
    uint64_t pix = 0;
    Rng rng{0, 0};
    WalkV x;  // current vertex (= v[d])
    WalkVel vv[VEL ? kMaxVerts : 1];  // velocity history (Doppler gates)
    V3 xvel{0, 0, 0};                 // current vertex velocity and path velocity so far
    double xu = 0;
    Cand c;   // NEE candidate waiting for its shadow ray
    c.pdf = 0;
    c.u = 0;
    V3 rd{0, 0, 1};
    double rtmax = 0, bs_pdf = 0, surv = 1;
    uint32_t n_closest = 0, n_any = 0;

    for (;;) {
        // ---- refill: lanes without a pixel take the next ones
        bool need = state == ST_IDLE && !exhausted;
        unsigned m = __ballot_sync(0xffffffffu, need);
        if (m) {
            int leader = __ffs(m) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(q, (unsigned long long)__popc(m));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (need) {
                size_t i = size_t(base) + __popc(m & ((1u << lane) - 1));
                if (i >= n) {
                    exhausted = true;
                } else {
                    int p = bd.y0 * W + int(i);
                    px = p % W;
                    py = p / W;
                    pix = uint64_t(py) * W + px;
                    g = gbuf[p];
                    sk.begin(cfg, frame_key, pix, size_t(p), trees);
                    s = -1;
                    state = ST_EXT;  // "tree done" below starts tree 0
                    d = cfg.max_depth + 2;
                }
            }
        }
        if (__all_sync(0xffffffffu, exhausted)) {
            work_add(cfg.work, WK_CLOSEST, n_closest);
            work_add(cfg.work, WK_ANY, n_any);
            sk.flush(cfg.work);
            break;
        }

        // ---- advance to the next ray (no ray needed for these steps)
        bool ray = false, any = false;
        while (state != ST_IDLE && !ray) {
            if (state == ST_NEE) {
                // for (d = 1; d + 1 <= max_depth && d < kMaxVerts - 1; ++d): loop test
                if (!(d + 1 <= cfg.max_depth && d < kMaxVerts - 1)) {
                    state = ST_EXT;
                    d = cfg.max_depth + 2;  // forces "tree done"
                    continue;
                }
                state = ST_EXT;
                const GMat& mx = Fs.mats[x.mat];
                if (mx.kind == MAT_MIRROR) continue;
                // emit_nee (transport.hpp:280-328), candidate prepared before its shadow ray
                V3 lp;
                if (wide) {
                    LightSample ls;
                    if (!light_sample(Fs.light, x.p, ls)) continue;
                    c.len = x.len + ls.dist;
                    if (VEL) c.u = xu + dot(xvel, ls.dir);
                    if (!sk.wants(c.len, c.u)) continue;
                    V3 f_at = eval_bsdf(mx, x.n, x.wi, ls.dir);
                    double cos_v = fabs(dot(x.n, ls.dir));
                    c.f = x.fw * f_at * (cos_v) * ls.value;
                    lp = Fs.light.pos;
                } else {
                    if (!Fs.lsub.valid) continue;
                    V3 dvec = Fs.lsub.pos - x.p;
                    double dist = norm(dvec);
                    if (dist <= eps * 2) continue;
                    V3 wto = dvec / dist;
                    c.len = x.len + dist + Fs.lsub.chain_len;
                    if (VEL) {
                        V3 vs = velocity_at(Fs, Fs.lsub.obj, Fs.lsub.pos);
                        c.u = xu + dot(xvel - vs, wto) + dot(vs, Fs.lsub.wo_light);
                    }
                    if (!sk.wants(c.len, c.u)) continue;
                    V3 f_at = eval_bsdf(mx, x.n, x.wi, wto);
                    V3 f_s = eval_bsdf(Fs.mats[Fs.lsub.mat], Fs.lsub.n, -wto, Fs.lsub.wo_light);
                    double gg = geom_term(x.p, x.n, Fs.lsub.pos, Fs.lsub.n);
                    c.f = x.fw * f_at * gg * f_s * Fs.lsub.power;
                    lp = Fs.lsub.pos;
                }
                c.depth = d + 1;
                c.pdf = x.pdf;
                // candidates the sink drops anyway need no shadow ray
                if (c.len <= 0 || !(luminance(c.f) > 0) || !finite3(c.f)) continue;
                // occluded(x.p, light): open segment shrunk by eps_ray
                V3 dd = lp - x.p;
                double dist = norm(dd);
                if (dist <= 2 * eps) {  // never occluded
                    RecSrc rs{v, d, nullptr, rng.key, VEL ? vv : nullptr};
                    sk.emit(Fs, c, 1.0, rs);
                    continue;
                }
                rd = dd / dist;
                rtmax = dist - eps;
                ray = true;
                any = true;
                state = ST_SHADOW;
            } else if (state == ST_EXT) {
                if (d + 2 > cfg.max_depth) {  // tree done
                    if (s >= 0) sk.tree_end();
                    ++s;
                    if (s >= trees) {
                        sk.end();
                        state = ST_IDLE;
                        continue;
                    }
                    sk.tree_begin();
                    rng = rng_make(cfg.seed, frame_key, pix, uint64_t(s), 0);
                    if (g.tri < 0) continue;  // no primary hit: an empty tree
                    V3 d0 = primary_dir(Fs.cam, px, py);
                    const GTriInfo& ti = Fs.tri[g.tri];
                    x.p = Fs.cam.pos + d0 * g.t;
                    x.n = ti.n;
                    x.tri = g.tri;
                    x.mat = ti.mat;
                    x.wi = -d0;
                    x.fw = splat(1);
                    x.pdf = 1;
                    x.len = g.t;
                    x.lane = 0;
                    v[1] = x;
                    if (VEL) {
                        xvel = velocity_at(Fs, ti.obj, x.p);
                        xu = dot(Fs.cam_vel - xvel, d0);
                        vv[1] = WalkVel{xvel, xu};
                    }
                    d = 1;
                    state = ST_NEE;
                    continue;
                }
                // walk cutoff: path lengths only grow (every segment adds a
                // non-negative length), so once x.len passes the sink's reach no
                // NEE or later candidate of this tree can be wanted -- the tree
                // ends here with the same candidates (the next tree has its own
                // RNG stream)
                if (cfg.walk_cutoff && x.len > sk.walk_max()) {
                    d = cfg.max_depth + 2;
                    continue;
                }
                const GMat& mx = Fs.mats[x.mat];
                x.lane = uint32_t(rng.ctr);
                v[d].lane = x.lane;
                surv = rr_survival(d, cfg.use_rr);
                if (surv < 1.0 && rng_next(rng) >= surv) {
                    d = cfg.max_depth + 2;
                    continue;
                }
                BsdfSample bs = sample_bsdf(mx, x.n, x.wi, rng);
                if (!bs.valid) {
                    d = cfg.max_depth + 2;
                    continue;
                }
                rd = bs.wo;
                bs_pdf = bs.pdf;
                rtmax = kInf;
                ray = true;
                any = false;
                state = ST_EXTEND;
            }
        }

        // ---- trace: one traversal for every lane with a ray
        TraceHit th{0, -1};
        if (ray) {
            th = trace_ray_impl(Fs.nodes, Fs.tri_isect, x.p, rd, eps, rtmax, any);
            if (any)
                ++n_any;
            else
                ++n_closest;
        }

        // ---- consume
        if (state == ST_SHADOW) {
            if (th.slot < 0) {
                RecSrc rs{v, d, nullptr, rng.key, VEL ? vv : nullptr};
                sk.emit(Fs, c, 1.0, rs);
            }
            state = ST_EXT;
        } else if (state == ST_EXTEND) {
            if (th.slot < 0) {
                d = cfg.max_depth + 2;  // no hit: tree done
                state = ST_EXT;
            } else {
                const GMat& mx = Fs.mats[x.mat];
                int tri = Fs.tri_id[th.slot];
                const GTriInfo& wt = Fs.tri[tri];
                WalkV w;
                w.p = x.p + rd * th.t;
                w.n = wt.n;
                w.tri = tri;
                w.mat = wt.mat;
                w.wi = -rd;
                w.lane = 0;
                double gt = geom_term(x.p, x.n, w.p, w.n);
                V3 fr_val = mx.kind == MAT_MIRROR ? mx.albedo : eval_bsdf(mx, x.n, x.wi, rd);
                w.fw = x.fw * fr_val * gt;
                double cos_w = fabs(dot(w.n, rd));
                w.pdf = x.pdf * surv * bs_pdf * cos_w / (th.t * th.t);
                w.len = x.len + th.t;
                ++d;
                v[d] = w;
                x = w;
                if (VEL) {
                    V3 wvel = velocity_at(Fs, wt.obj, w.p);
                    xu = xu + dot(xvel - wvel, rd);
                    xvel = wvel;
                    vv[d] = WalkVel{xvel, xu};
                }
                state = ST_NEE;
            }
        }
    }
}

// chunk 0 (w_sum, -) of every (pixel, bin) -> (W, 1) (ris_finalize + M = 1)
__global__ void k_ris_finalize(ResStore st, size_t i0, size_t i1) {
    for (size_t i = i0 + blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < i1; i += size_t(gridDim.x) * blockDim.x) {
        double2 c0 = ld2(st, 0, i);
        double Wv = 0;
        if (c0.x > 0) {
            double phat = ld2(st, 1, i).x;
            Wv = phat > 0 ? c0.x / phat : 0;
        }
        st2(st, 0, i, Wv, 1.0);
    }
}

// ---------------------------------------------------------------------------
// launchers

template <class Sink, bool VEL = false>
static void launch_trace(const char* kname, const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg,
                         int trees, uint64_t frame_key, const Sink& sk, unsigned long long* q, cudaStream_t s) {
    size_t n = size_t(bd.y1 - bd.y0) * F.cam.w;
    if (!n) return;
    size_t sm = frame_smem_bytes(F);
    cudaMemsetAsync(q, 0, sizeof(unsigned long long), s);
    const void* kf = reinterpret_cast<const void*>(k_trace<Sink, VEL>);
    {
        KScope ks(kname, s);
        k_trace<Sink, VEL><<<persistent_grid(kf, TOFR_TRACE_BLOCK, sm, n), TOFR_TRACE_BLOCK, sm, s>>>(F, bd, g, cfg,
                                                                                               trees, frame_key, sk, q);
    }
}

void launch_trace_gated(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, int m_init,
                        double center, double width, int frame_idx, ResStore cur, unsigned long long* q,
                        cudaStream_t s) {
    auto run = [&](auto sk, auto vel) {
        sk.cur = cur;
        sk.center = center;
        sk.width = width;
        sk.inv = 1.0 / m_init;
        launch_trace<decltype(sk), decltype(vel)::value>("k_trace_gated", F, bd, g, cfg, m_init,
                                                         uint64_t(frame_idx), sk, q, s);
    };
    if (cfg.gate_vel)
        run(GatedSink<true>{}, std::true_type{});
    else
        run(GatedSink<false>{}, std::false_type{});
}

void launch_trace_gated_ris(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, int trees,
                            double center, double width, int frame_idx, ResStore cur, const uint64_t* pick_in,
                            uint64_t* pick_out, unsigned long long* q, cudaStream_t s) {
    GatedSink<false> sk{};
    sk.cur = cur;
    sk.center = center;
    sk.width = width;
    sk.inv = 1.0 / trees;
    sk.pick_in = pick_in;
    sk.pick_out = pick_out;
    sk.pbase = size_t(bd.y0) * F.cam.w;
    launch_trace<GatedSink<false>, false>("k_trace_gated", F, bd, g, cfg, trees, uint64_t(frame_idx), sk, q, s);
}

void launch_trace_transient(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, int m_init,
                            const HistSpec& h, int frame_idx, ResStore cur, unsigned long long* q, cudaStream_t s) {
    size_t n = size_t(bd.y1 - bd.y0) * F.cam.w * h.bins;
    if (!n) return;
    size_t i0 = size_t(bd.y0) * F.cam.w * h.bins;
    cudaMemsetAsync(cur.base + i0, 0, n * sizeof(double2), s);  // chunk 0 plane of the band
    BinsSink sk;
    sk.st = cur;
    sk.h = h;
    sk.inv = 1.0 / m_init;
    launch_trace("k_trace_bins", F, bd, g, cfg, m_init, uint64_t(frame_idx), sk, q, s);
    size_t blocks = (n + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    {
        KScope ks("k_ris_finalize", s);
        k_ris_finalize<<<int(blocks), 256, 0, s>>>(cur, i0, i0 + n);
    }
}

void launch_trace_plain(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, const HistSpec& h,
                        int m_init, int frame_idx, double* hist, double* img, unsigned long long* q,
                        cudaStream_t s) {
    PlainSink2 sk;
    sk.h = h;
    sk.m_init = m_init;
    sk.hist = hist;
    sk.img = img;
    sk.deposits = 0;
    launch_trace("k_trace_plain", F, bd, g, cfg, m_init, uint64_t(frame_idx), sk, q, s);
}

void launch_trace_reference(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, double center,
                            double width, int spp, uint64_t frame_key, double* mean, double* se,
                            unsigned long long* q, cudaStream_t s) {
    RefSink2 sk;
    sk.center = center;
    sk.width = width;
    sk.mean = mean;
    sk.se = se;
    launch_trace("k_trace_reference", F, bd, g, cfg, spp, frame_key, sk, q, s);
}

}  // namespace tofr_b200
