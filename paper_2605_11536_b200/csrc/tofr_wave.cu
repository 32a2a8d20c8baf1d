// tofr_wave.cu -- wavefront shift engine and the reuse stages built on it.
//
// The path-length-preserving shift (shift_sample, shiftmap.hpp:662-783) is the
// hot operation of temporal and spatial reuse.  Run as one monolithic device
// function per reservoir it keeps whole samples in local memory and serialises
// very different phases (prefix replay, Newton, occlusion, rebuild) inside a
// warp.  Here a reuse stage is a short pipeline over compacted job queues:
//
//   prep     one thread per reservoir item decides which shifts the merge
//            needs (forward: neighbour sample -> pixel; inverse: the pixel's
//            sample -> neighbour) and appends them to the queue with warp
//            ballots + one atomic per warp;
//   solve    k_shift_solve: record checks, prefix (stored / G-buffer / lane
//            replay), suffix and the Newton solve.  Lanes refill from the
//            queue as soon as their job finishes, so a warp always runs 32
//            Newton trials together (persistent threads, per-lane refill);
//   finish   k_shift_finish: the two occlusion rays, Jacobian clamp, rebuild
//            of the shifted sample, output (the mapped record for forward
//            shifts, p-hat of the source gate for inverse shifts);
//   apply    one thread per item runs the GRIS merge with the reference's RNG
//            stream and writes the reservoir (chunk 0 only when the kept sample
//            is already in place).
//
// Same IEEE operations in the same order as the per-reservoir code, same RNG
// draws, same integer counters: results are bit-identical to it.
#include <cuda_runtime.h>

// The shift kernels are small enough to take FP64 division and square root
// inline: out-of-line math (tofr_core.h) would force the Newton state across
// call boundaries (caller-saved registers -> local memory).
#define TOFR_OUTLINE_MATH 0

#include "ktime.h"
#include "tofr_kcommon.cuh"
#include "tofr_store.cuh"

#ifndef TOFR_WAVE_MINB
#define TOFR_WAVE_MINB 4
#endif
#ifndef TOFR_FINISH_MINB
#define TOFR_FINISH_MINB TOFR_WAVE_MINB
#endif
// threads per CTA of the persistent solve (TOFR_WAVE_MINB CTAs of 128 per SM)
#ifndef TOFR_SOLVE_BLOCK
#define TOFR_SOLVE_BLOCK 128
#endif
// idle lanes a warp of k_shift_solve collects before it refills them
#ifndef TOFR_REFILL
#define TOFR_REFILL 12
#endif
// lanes needing re-projection rays a warp collects before it traces them
#ifndef TOFR_RAYBATCH
#define TOFR_RAYBATCH 12
#endif
#ifndef TOFR_SOLVE_REVERSE
#define TOFR_SOLVE_REVERSE 0
#endif
// 1: lanes waiting for a refill help too (measured slower: it disables ray parking)
#ifndef TOFR_HELP_IDLE
#define TOFR_HELP_IDLE 0
#endif
// 1: a batch with fewer jobs than 32 per warp of the grid is spread over all
// warps (at most ceil(jobs / warps) busy lanes per warp), so every busy lane
// has idle lanes of its own warp to run its halving ladder from the first
// round (without it the first warps take 32 jobs each and the rest exit)
#ifndef TOFR_SHARE
#define TOFR_SHARE 1
#endif
// >0: a lane whose solve has rejected TOFR_ESCALATE halvings in a row (or
// passed two Newton iterations) is "slow": its warp stops refilling until its
// slow lanes finish, and the lanes that free up run their halving ladders
// (the tail-phase helpers) -- the long serial chains that end every shift
// batch get helpers before the queue drains
#ifndef TOFR_ESCALATE
#define TOFR_ESCALATE 0
#endif

namespace tofr_b200 {

// ---------------------------------------------------------------------------
// job records (chunk-major, kJobChunks x 16 B)
//   0: item (u64), meta (u32), -      2: s_center, d_center     4-6: solve -> finish
//   1: spx, spy, dpx, dpy (i32)       3: d_width, -                  (see sol_*)

struct Job {
    size_t item;
    uint32_t meta;
    int spx, spy, dpx, dpy;
    double sc, dc, dw;
};

__device__ __forceinline__ double2 jld(const ShiftQueue& q, int c, uint32_t k) {
    TOFR_CHK(c >= 0 && c < kJobChunks && size_t(k) < q.cap);
    return __ldcg(&q.jobs[size_t(c) * q.cap + k]);
}
__device__ __forceinline__ void jst(const ShiftQueue& q, int c, uint32_t k, double2 v) {
    TOFR_CHK(c >= 0 && c < kJobChunks && size_t(k) < q.cap);
    __stcg(&q.jobs[size_t(c) * q.cap + k], v);
}

__device__ __forceinline__ void job_put(const ShiftQueue& q, uint32_t k, size_t item, uint32_t meta, int spx, int spy,
                                        int dpx, int dpy, double sc, double dc, double dw) {
    double2 c0;
    uint64_t it = item;
    uint2 mm = make_uint2(meta, 0);
    memcpy(&c0.x, &it, 8);
    memcpy(&c0.y, &mm, 8);
    jst(q, 0, k, c0);
    int4 px = make_int4(spx, spy, dpx, dpy);
    double2 c1;
    memcpy(&c1, &px, 16);
    jst(q, 1, k, c1);
    jst(q, 2, k, make_double2(sc, dc));
    jst(q, 3, k, make_double2(dw, 0.0));
}

__device__ __forceinline__ Job job_get(const ShiftQueue& q, uint32_t k) {
    Job j;
    double2 c0 = jld(q, 0, k), c1 = jld(q, 1, k), c2 = jld(q, 2, k), c3 = jld(q, 3, k);
    uint64_t it;
    uint2 mm;
    memcpy(&it, &c0.x, 8);
    memcpy(&mm, &c0.y, 8);
    int4 px;
    memcpy(&px, &c1, 16);
    j.item = size_t(it);
    j.meta = mm.x;
    j.spx = px.x;
    j.spy = px.y;
    j.dpx = px.z;
    j.dpy = px.w;
    j.sc = c2.x;
    j.dc = c2.y;
    j.dw = c3.x;
    return j;
}

// solve -> finish hand-off: solved point and triangle, J_newton, status
// (bit 0: proceed to occlusion; bit 1: the point's normal is still the
// record's pn -- it never left the start triangle -- else it is the normal of
// the triangle a re-projection ray hit, reproject_to_mesh)
__device__ __forceinline__ void sol_put(const ShiftQueue& q, uint32_t k, const V3& pos, int tri, double jn,
                                        int status) {
    jst(q, 4, k, make_double2(pos.x, pos.y));
    jst(q, 5, k, make_double2(pos.z, jn));
    double2 c6;
    c6.x = 0;
    int2 ts = make_int2(tri, status);
    memcpy(&c6.y, &ts, 8);
    jst(q, 6, k, c6);
    if (q.done) {  // publish: hand-off first, then the mark (release)
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(q.done + k), "r"(q.epoch) : "memory");
    }
}
// finish side: wait until the solve of job k has published its hand-off
__device__ __forceinline__ void sol_wait(const ShiftQueue& q, uint32_t k) {
    if (!q.done) return;
    for (;;) {
        uint32_t v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(q.done + k) : "memory");
        if (v == q.epoch) break;
        __nanosleep(64);
    }
}
__device__ __forceinline__ void sol_fail(const ShiftQueue& q, uint32_t k) { sol_put(q, k, splat(0), -1, 0.0, 0); }

// Warp-aggregated append: every lane of the warp must call it (converged).
// Returns the job slot for lanes with `want`, kNoJob otherwise; a full queue
// raises the overflow bit of the band error flag.
__device__ __forceinline__ uint32_t queue_append(const ShiftQueue& q, bool want, unsigned long long* err) {
    unsigned m = __ballot_sync(0xffffffffu, want);
    if (!m) return kNoJob;
    int lane = threadIdx.x & 31;
    int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(&q.ctl[1], uint32_t(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, leader);
    uint32_t k = base + __popc(m & ((1u << lane) - 1));
    if (!want) return kNoJob;
    if (k >= q.cap) {
        atomicAdd(err, 1ull << 32);
        return kNoJob;
    }
    return k;
}

// Warp-aggregated append to the merge list (items whose merge needs a sample:
// at least one side non-empty); count in q.ctl[3].  All lanes must call it.
__device__ __forceinline__ void mlist_append(const WaveScratch& ws, bool want, uint32_t item,
                                             unsigned long long* work) {
    unsigned m = __ballot_sync(0xffffffffu, want);
    if (!m) return;
    int lane = threadIdx.x & 31;
    int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) {
        base = atomicAdd(&ws.q.ctl[3], uint32_t(__popc(m)));
        if (work) atomicAdd(&work[WK_MERGES], (unsigned long long)__popc(m));
    }
    base = __shfl_sync(0xffffffffu, base, leader);
    if (want) ws.mlist[base + __popc(m & ((1u << lane) - 1))] = item;
}

// Block-aggregated appends for the per-item prep kernels: one global atomic
// per block and list per loop iteration instead of one per warp (the warps of
// a 67 M-item transient grid otherwise serialise on the queue counters).  All
// threads of the block must call them; `sh` is nwarps + 1 words of shared memory.
__device__ __forceinline__ uint32_t block_append(uint32_t* gctr, bool want, uint32_t* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned m = __ballot_sync(0xffffffffu, want);
    if (lane == 0) sh[warp] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (int w = 0; w < nw; ++w) {
            uint32_t c = sh[w];
            sh[w] = tot;
            tot += c;
        }
        sh[nw] = tot ? atomicAdd(gctr, tot) : 0u;
    }
    __syncthreads();
    uint32_t k = sh[nw] + sh[warp] + __popc(m & ((1u << lane) - 1));
    __syncthreads();  // `sh` is reused by the next call
    return want ? k : kNoJob;
}

__device__ __forceinline__ uint32_t block_queue_append(const ShiftQueue& q, bool want, unsigned long long* err,
                                                       uint32_t* sh) {
    uint32_t k = block_append(&q.ctl[1], want, sh);
    if (k != kNoJob && k >= q.cap) {
        atomicAdd(err, 1ull << 32);
        return kNoJob;
    }
    return k;
}

// One block-wide append of up to 2 jobs per thread to the shift queue and of
// the item to the merge list (2 barriers + 1 instead of 3 per append): returns
// the thread's first job slot (its jobs are consecutive), kNoJob if none or
// the queue is full (overflow bit raised).  `sh`: 2 * nwarps + 2 words.
__device__ __forceinline__ uint32_t block_append_jobs(const WaveScratch& ws, uint32_t njobs, bool merge,
                                                      uint32_t item, unsigned long long* err,
                                                      unsigned long long* work, uint32_t* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t incl = njobs;  // inclusive warp scan of the job counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    const uint32_t wtot = __shfl_sync(0xffffffffu, incl, 31);
    const unsigned mm = __ballot_sync(0xffffffffu, merge);
    if (lane == 0) {
        sh[warp] = wtot;
        sh[nw + warp] = __popc(mm);
        if (work && mm) atomicAdd(&work[WK_MERGES], (unsigned long long)__popc(mm));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tj = 0, tm = 0;
        for (int w = 0; w < nw; ++w) {
            uint32_t cj = sh[w], cm = sh[nw + w];
            sh[w] = tj;
            sh[nw + w] = tm;
            tj += cj;
            tm += cm;
        }
        sh[2 * nw] = tj ? atomicAdd(&ws.q.ctl[1], tj) : 0u;
        sh[2 * nw + 1] = tm ? atomicAdd(&ws.q.ctl[3], tm) : 0u;
    }
    __syncthreads();
    const uint32_t k = sh[2 * nw] + sh[warp] + (incl - njobs);
    if (merge) ws.mlist[sh[2 * nw + 1] + sh[nw + warp] + __popc(mm & ((1u << lane) - 1))] = item;
    __syncthreads();  // `sh` is reused by the next call
    if (!njobs) return kNoJob;
    if (size_t(k) + njobs > ws.q.cap) {
        atomicAdd(err, 1ull << 32);
        return kNoJob;
    }
    return k;
}

// The multi-item form: a thread appends `njobs` consecutive job slots and
// `nmerge` consecutive merge-list slots (its items' entries, in its item
// order).  Returns the first job slot (kNoJob if none or the queue is full:
// overflow bit raised) and the first merge-list slot in *mfirst.
__device__ __forceinline__ uint32_t block_append_jobs_n(const WaveScratch& ws, uint32_t njobs, uint32_t nmerge,
                                                        uint32_t* mfirst, unsigned long long* err,
                                                        unsigned long long* work, uint32_t* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t incl = njobs, minc = nmerge;  // inclusive warp scans
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        uint32_t vm = __shfl_up_sync(0xffffffffu, minc, o);
        if (lane >= o) {
            incl += v;
            minc += vm;
        }
    }
    const uint32_t wtot = __shfl_sync(0xffffffffu, incl, 31), mtot = __shfl_sync(0xffffffffu, minc, 31);
    if (lane == 0) {
        sh[warp] = wtot;
        sh[nw + warp] = mtot;
        if (work && mtot) atomicAdd(&work[WK_MERGES], (unsigned long long)mtot);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tj = 0, tm = 0;
        for (int w = 0; w < nw; ++w) {
            uint32_t cj = sh[w], cm = sh[nw + w];
            sh[w] = tj;
            sh[nw + w] = tm;
            tj += cj;
            tm += cm;
        }
        sh[2 * nw] = tj ? atomicAdd(&ws.q.ctl[1], tj) : 0u;
        sh[2 * nw + 1] = tm ? atomicAdd(&ws.q.ctl[3], tm) : 0u;
    }
    __syncthreads();
    const uint32_t k = sh[2 * nw] + sh[warp] + (incl - njobs);
    *mfirst = sh[2 * nw + 1] + sh[nw + warp] + (minc - nmerge);
    __syncthreads();  // `sh` is reused by the next call
    if (!njobs) return kNoJob;
    if (size_t(k) + njobs > ws.q.cap) {
        atomicAdd(err, 1ull << 32);
        return kNoJob;
    }
    return k;
}

__device__ __forceinline__ void block_mlist_append(const WaveScratch& ws, bool want, uint32_t item,
                                                   unsigned long long* work, uint32_t* sh) {
    uint32_t k = block_append(&ws.q.ctl[3], want, sh);
    if (k != kNoJob) ws.mlist[k] = item;
    unsigned m = __ballot_sync(0xffffffffu, want);
    if (work && (threadIdx.x & 31) == 0 && m) atomicAdd(&work[WK_MERGES], (unsigned long long)__popc(m));
}

// ---------------------------------------------------------------------------
// record fields straight from the reservoir store (tofr_store.cuh layout)

__device__ __forceinline__ V3 rec_p(const ResStore& s, size_t i) {
    double2 a = ld2(s, 10, i), b = ld2(s, 11, i);
    return V3{a.y, b.x, b.y};
}
__device__ __forceinline__ V3 rec_pn(const ResStore& s, size_t i) {
    double2 a = ld2(s, 12, i), b = ld2(s, 13, i);
    return V3{a.x, a.y, b.x};
}
__device__ __forceinline__ V3 rec_p2(const ResStore& s, size_t i) {
    double2 a = ld2(s, 13, i), b = ld2(s, 14, i);
    return V3{a.y, b.x, b.y};
}
__device__ __forceinline__ V3 rec_n2(const ResStore& s, size_t i) {
    double2 a = ld2(s, 15, i), b = ld2(s, 16, i);
    return V3{a.x, a.y, b.x};
}
__device__ __forceinline__ V3 rec_wo2(const ResStore& s, size_t i) {
    double2 a = ld2(s, 16, i), b = ld2(s, 17, i);
    return V3{a.y, b.x, b.y};
}
__device__ __forceinline__ V3 rec_suffix_f(const ResStore& s, size_t i, int& m2) {
    double2 a = ld2(s, 18, i), b = ld2(s, 19, i);
    int2 mi;
    memcpy(&mi, &b.y, 8);
    m2 = mi.x;
    return V3{a.x, a.y, b.x};
}

// stored_prefix (identity shift: same pixel and frame), from the store
__device__ __forceinline__ Prefix stored_prefix_at(const FrameView& F, const ResStore& s, size_t i, int tri1,
                                                   bool vel) {
    Prefix pre;
    pre.ok = 1;
    if (s.compact) {
        const PrefixCache pc = res_prefix_derived(s, i);
        pre.pdf = pc.pdf;
        pre.len = pc.len;
        pre.fw = pc.fw;
        pre.p1 = pc.p1;
        pre.wi1 = pc.wi1;
    } else {
        double2 c5 = ld2(s, 5, i), c6 = ld2(s, 6, i), c7 = ld2(s, 7, i), c8 = ld2(s, 8, i), c9 = ld2(s, 9, i),
                c10 = ld2(s, 10, i);
        pre.pdf = c5.x;
        pre.len = c5.y;
        pre.fw = V3{c6.x, c6.y, c7.x};
        pre.p1 = V3{c7.y, c8.x, c8.y};
        pre.wi1 = V3{c9.x, c9.y, c10.x};
    }
    pre.n1 = F.tri[tri1].n;
    pre.tri1 = tri1;
    pre.m1 = F.tri[tri1].mat;
    pre.u = vel ? ld2(s, 22, i).y : 0.0;
    return pre;
}

// hybrid_base_shift for k = 2 (shiftmap.hpp:459-528 with no replayed bounce):
// the prefix is the destination pixel's primary hit.
__device__ __forceinline__ Prefix gbuffer_prefix(const FrameView& F, const GHit* gbuf, int px, int py, bool vel) {
    Prefix out;
    out.ok = 0;
    GHit g = gbuf[size_t(py) * F.cam.w + px];
    if (g.tri < 0) return out;
    V3 d0 = primary_dir(F.cam, px, py);
    int mat = F.tri[g.tri].mat;
    if (!F.mats[mat].reconnectable) return out;
    out.ok = 1;
    out.pdf = 1;
    out.len = g.t;
    out.fw = splat(1);
    out.p1 = F.cam.pos + d0 * g.t;
    out.u = vel ? dot(F.cam_vel - velocity_at(F, F.tri[g.tri].obj, out.p1), d0) : 0.0;
    out.n1 = F.tri[g.tri].n;
    out.wi1 = -d0;
    out.tri1 = g.tri;
    out.m1 = mat;
    return out;
}

// hybrid_base_shift with k - 2 replayed bounces (mirror / low-roughness
// scenes): lanes read from the store.  Out of line: rare and ray-heavy.
static __device__ __noinline__ Prefix replay_prefix(const FrameView* Fp, const GHit* gbuf, int px, int py,
                                                    ResStore s, size_t item, int k, int use_rr) {
    Rec rec;
    rec.k = k;
    double2 c20 = ld2(s, 20, item), c21 = ld2(s, 21, item);
    memcpy(&rec.lane_key, &c20.x, 8);
    memcpy(&rec.lane_ctr[0], &c20.y, 8);
    memcpy(&rec.lane_ctr[4], &c21, 12);
    Dom dom{px, py, 0.0, 0.0, Fp, gbuf};
    PathCfg cfg;
    cfg.use_rr = use_rr;
    return base_shift(dom, rec, cfg);
}

// replayed prefix of job k (k_shift_replay) in job chunks 7-12
__device__ __forceinline__ void replay_put(const ShiftQueue& q, uint32_t k, const Prefix& p) {
    jst(q, 7, k, make_double2(p.pdf, p.len));
    jst(q, 8, k, make_double2(p.fw.x, p.fw.y));
    jst(q, 9, k, make_double2(p.fw.z, p.p1.x));
    jst(q, 10, k, make_double2(p.p1.y, p.p1.z));
    jst(q, 11, k, make_double2(p.wi1.x, p.wi1.y));
    double2 c12;
    c12.x = p.wi1.z;
    int2 to = make_int2(p.ok ? p.tri1 : -1, p.ok);
    memcpy(&c12.y, &to, 8);
    jst(q, 12, k, c12);
    jst(q, 13, k, make_double2(p.u, 0.0));
}
__device__ __forceinline__ Prefix replay_get(const FrameView& F, const ShiftQueue& q, uint32_t k) {
    Prefix p;
    double2 c7 = jld(q, 7, k), c8 = jld(q, 8, k), c9 = jld(q, 9, k), c10 = jld(q, 10, k), c11 = jld(q, 11, k),
            c12 = jld(q, 12, k);
    int2 to;
    memcpy(&to, &c12.y, 8);
    p.ok = to.y;
    if (!p.ok) return p;
    p.pdf = c7.x;
    p.len = c7.y;
    p.fw = V3{c8.x, c8.y, c9.x};
    p.p1 = V3{c9.y, c10.x, c10.y};
    p.wi1 = V3{c11.x, c11.y, c12.x};
    p.tri1 = to.x;
    p.n1 = F.tri[p.tri1].n;  // hybrid_base_shift: n = the hit triangle's normal
    p.m1 = F.tri[p.tri1].mat;
    p.u = jld(q, 13, k).x;
    return p;
}

// prefix of the destination path: stored (identity), the primary hit (k = 2)
// or the replayed bounces computed by k_shift_replay (k > 2)
__device__ __forceinline__ Prefix job_prefix(const FrameView& F, const GHit* gbuf, const Job& jb, bool identity,
                                             const ResStore& st, const Meta& mt, const ShiftQueue& q, uint32_t k,
                                             bool vel) {
    if (identity) return stored_prefix_at(F, st, jb.item, mt.tri1, vel);
    if (mt.k == 2) return gbuffer_prefix(F, gbuf, jb.dpx, jb.dpy, vel);
    return replay_get(F, q, k);
}

// suffix_geometry (shiftmap.hpp:546-575)
__device__ __forceinline__ Suffix job_suffix(const FrameView& F, const ResStore& st, size_t item, int skind,
                                             bool vel) {
    Suffix s;
    s.ok = 0;
    s.n2 = splat(0);
    if (skind == SK_SURFACE) {
        s.p2 = rec_p2(st, item);
        s.n2 = rec_n2(st, item);
        s.len = ld2(st, 3, item).y;
        s.u = 0;
        s.v2 = splat(0);
        if (vel) {
            s.u = ld2(st, 23, item).x;
            int2 mo;
            double m19 = ld2(st, 19, item).y;
            memcpy(&mo, &m19, 8);
            s.v2 = velocity_at(F, mo.y, s.p2);  // obj2
            s.vobj = mo.y;
        }
        s.ok = 1;
    } else if (skind == SK_LIGHT) {
        s.p2 = F.light.pos;
        s.len = 0;
        s.u = 0;
        s.v2 = splat(0);
        s.ok = 1;
    } else {
        if (!F.lsub.valid) return s;
        s.p2 = F.lsub.pos;
        s.n2 = F.lsub.n;
        s.len = F.lsub.chain_len;
        s.v2 = vel ? velocity_at(F, F.lsub.obj, F.lsub.pos) : splat(0);
        s.vobj = F.lsub.obj;
        s.u = vel ? dot(s.v2, F.lsub.wo_light) : 0.0;
        s.ok = 1;
    }
    return s;
}

// reproject_to_mesh (shiftmap.hpp:275-307), ray fallbacks: the plane point left
// the current triangle.  Out of line, arguments by value.
struct SurfR {
    V3 pos, n;
    int tri, ok;
    int rays;  // closest-hit rays traced
};
static __device__ __noinline__ SurfR reproject_rays(const FrameView* Fp, int cur_tri, V3 plane_pt, V3 p1) {
    const FrameView& F = *Fp;
    SurfR out;
    out.ok = 0;
    out.rays = 0;
    V3 tn = F.tri[cur_tri].n;
    V3 dir = plane_pt - p1;
    double dl = norm(dir);
    Hit h;
    if (dl > 0) {
        dir = dir / dl;
        if (fabs(dot(dir, tn)) > 1e-4) {
            out.rays = 1;
            if (intersect(F, p1, dir, h)) {
                out.pos = h.pos;
                out.n = F.tri[h.tri].n;
                out.tri = h.tri;
                out.ok = 1;
                return out;
            }
        }
    }
    double off = 1e-3 * F.diag;
    out.rays += 1;
    bool hit = trace_closest(F, plane_pt + tn * off, -tn, 0, 2 * off, h);
    if (!hit) {
        out.rays += 1;
        hit = trace_closest(F, plane_pt - tn * off, tn, 0, 2 * off, h);
    }
    if (hit) {
        out.pos = h.pos;
        out.n = F.tri[h.tri].n;
        out.tri = h.tri;
        out.ok = 1;
    }
    return out;
}

// in-triangle test of reproject_to_mesh
__device__ __forceinline__ bool in_triangle(const FrameView& F, int tri, const V3& plane_pt) {
    const GTriIsect& g = tri_geo(F, tri);
    V3 e1 = g.e1, e2 = g.e2, d = plane_pt - g.v0;
    double d11 = dot(e1, e1), d12 = dot(e1, e2), d22 = dot(e2, e2);
    double dv1 = dot(d, e1), dv2 = dot(d, e2);
    double dt = d11 * d22 - d12 * d12;
    if (!(dt > 0)) return false;
    double u = (d22 * dv1 - d12 * dv2) / dt;
    double v = (d11 * dv2 - d12 * dv1) / dt;
    return u >= 0 && v >= 0 && u + v <= 1;
}

// per-thread shift counters in registers (constant indices only)
struct Ctr {
    uint32_t v[SC_COUNT];
};
__device__ __forceinline__ void ctr_flush(const Ctr& c, unsigned long long* out) {
    uint32_t t[SC_COUNT];
#pragma unroll
    for (int k = 0; k < SC_COUNT; ++k) t[k] = c.v[k];
    flush_ctr(t, out);
}

// stage the two frames of a reuse stage in shared memory (once when equal)
__device__ __forceinline__ void stage_two(FrameView& F0, FrameView& F1, FrameView* sF, unsigned char* smem) {
    size_t off = 0;
    bool same = F1.nodes == F0.nodes && F1.tri_isect == F0.tri_isect;
    stage_frame(F0, smem, off);
    if (same) {
        F1.nodes = F0.nodes;
        F1.tri_isect = F0.tri_isect;
    } else {
        stage_frame(F1, smem, off);
    }
    if (threadIdx.x == 0) {
        sF[0] = F0;
        sF[1] = F1;
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Newton constraint, split into its start-point half (constant per job) and
// its trial-point half.  assemble_constraint (shiftmap.hpp:155-217) evaluates
// both at every trial; the start-point terms (gradient, length, projected
// Hessian at the start point) are computed once here with the same operations,
// so every value is bit-identical to assemble().

// lc_value / lc_grad / lc_hess at p, sharing the edge vectors
struct LcEval {
    double val;   // |p1 - p| + |p2 - p|
    V3 grad;      // -(normalize(p1 - p) + normalize(p2 - p))
    M2 hess;      // project_sym(J, lc_hess(p1, p2, p)), only when `with_hess`
};
__device__ __forceinline__ LcEval lc_eval(const V3& p1, const V3& p2, const V3& p, const Frame2& J, bool with_hess) {
    LcEval r;
    V3 e1 = p1 - p, e2 = p2 - p;
    double l1 = norm(e1), l2 = norm(e2);
    V3 d1 = e1 / l1, d2 = e2 / l2;
    r.val = l1 + l2;
    r.grad = -(d1 + d2);
    r.hess = M2{0, 0, 0, 0};
    if (with_hess) {
        // A = (I - d1 d1^T) * (1/l1) + (I - d2 d2^T) * (1/l2), row by row
        double s1 = 1.0 / l1, s2 = 1.0 / l2;
        double At[3], Ab[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            double di1 = comp(d1, i), di2 = comp(d2, i);
            double a0 = ((i == 0 ? 1.0 : 0.0) - di1 * d1.x) * s1 + ((i == 0 ? 1.0 : 0.0) - di2 * d2.x) * s2;
            double a1 = ((i == 1 ? 1.0 : 0.0) - di1 * d1.y) * s1 + ((i == 1 ? 1.0 : 0.0) - di2 * d2.y) * s2;
            double a2 = ((i == 2 ? 1.0 : 0.0) - di1 * d1.z) * s1 + ((i == 2 ? 1.0 : 0.0) - di2 * d2.z) * s2;
            At[i] = a0 * J.t.x + a1 * J.t.y + a2 * J.t.z;
            Ab[i] = a0 * J.b.x + a1 * J.b.y + a2 * J.b.z;
        }
        V3 vt{At[0], At[1], At[2]}, vb{Ab[0], Ab[1], Ab[2]};
        r.hess = M2{dot(J.t, vt), dot(J.t, vb), dot(J.b, vt), dot(J.b, vb)};
    }
    return r;
}

// Velocity (Doppler) constraint field, LocalConstraint in velocity mode
// (shiftmap.hpp:28-122): u(p) = (v1 - v(p)).r1 + (v(p) - v2).r2 with v the rigid
// velocity field of the object p sits on (bound per evaluation point).
struct VelField {
    V3 v1, v2;
};

__device__ __forceinline__ V3 transpose_mul(const M3& A, const V3& v) {
    return V3{A.m[0][0] * v.x + A.m[1][0] * v.y + A.m[2][0] * v.z,
              A.m[0][1] * v.x + A.m[1][1] * v.y + A.m[2][1] * v.z,
              A.m[0][2] * v.x + A.m[1][2] * v.y + A.m[2][2] * v.z};
}

// detail::vel_term_grad / vel_term_hess (shiftmap.hpp:52-76)
__device__ __forceinline__ V3 vel_term_grad(const V3& p, const V3& a, const V3& cvec, double s_r, double alpha,
                                            const M3& V, bool moving) {
    V3 e = p - a;
    double l = norm(e);
    V3 n = e / l;
    M3 P = m3_identity() - m3_outer(n, n);
    V3 g = (P * cvec) * (s_r / l);
    if (moving) g = g + transpose_mul(V, n) * (alpha * s_r);
    return g;
}
__device__ __forceinline__ M3 vel_term_hess(const V3& p, const V3& a, const V3& cvec, double s_r, double alpha,
                                            const M3& V, bool moving) {
    V3 e = p - a;
    double l = norm(e);
    V3 n = e / l;
    M3 P = m3_identity() - m3_outer(n, n);
    V3 Pc = P * cvec;
    M3 h = (P * (-dot(n, cvec)) - m3_outer(n, Pc) - m3_outer(Pc, n)) * (s_r / (l * l));
    if (moving) {
        M3 PV = P * V;
        h = h + (PV + transpose(PV)) * (alpha * s_r / l);
    }
    return h;
}

// value, world gradient and projected Hessian of the velocity field at p,
// bound to object `obj`'s velocity field
__device__ __noinline__ LcEval vel_eval(const FrameView* Fp, int obj, VelField vf, V3 p1, V3 p2, V3 p, Frame2 J,
                                        bool with_hess) {
    const FrameView& F = *Fp;
    bool moving = obj >= 0 && obj < F.n_obj && F.vel[obj].moving;
    M3 A = moving ? F.vel[obj].A : m3_zero();
    V3 c = moving ? F.vel[obj].c : splat(0);
    V3 v = moving ? A * p + c : splat(0);
    LcEval r;
    r.val = dot(vf.v1 - v, normalize(p - p1)) + dot(v - vf.v2, normalize(p2 - p));
    r.grad = vel_term_grad(p, p1, vf.v1 - v, +1, -1, A, moving) + vel_term_grad(p, p2, v - vf.v2, -1, +1, A, moving);
    r.hess = M2{0, 0, 0, 0};
    if (with_hess)
        r.hess = project_sym(J, vel_term_hess(p, p1, vf.v1 - v, +1, -1, A, moving) +
                                    vel_term_hess(p, p2, v - vf.v2, -1, +1, A, moving));
    return r;
}

template <bool VEL>
__device__ __forceinline__ LcEval field_eval(const FrameView& F, int obj, const VelField& vf, const V3& p1,
                                             const V3& p2, const V3& p, const Frame2& J, bool with_hess) {
    if (VEL) return vel_eval(&F, obj, vf, p1, p2, p, J, with_hess);
    return lc_eval(p1, p2, p, J, with_hess);
}

struct StartTerms {
    V3 g3s;     // gradient at the start point
    V2 gs;      // ... in the start frame
    double lvs; // path length through the start point
    M2 Hs;      // projected Hessian at the start point (gauge != FIXED)
};

struct TrialEval {
    V2 F;
    M2 dFp;
    double det_dF;   // det(dF), dF = d F / d(start coordinates)
    double ngrad;    // |grad_cur|
};

// the trial half given the field evaluation e at the trial point pc
__device__ __forceinline__ TrialEval trial_from(const LcEval& e, const V3& ps, const Frame2& Js, const StartTerms& st,
                                                const V3& pc, const Frame2& Jc, double delta, int gauge) {
    TrialEval r;
    V2 gc = to_local(Jc, e.grad);
    r.ngrad = norm(gc);
    V3 disp = pc - ps;
    V2 us = to_local(Js, disp);
    V2 uc = to_local(Jc, disp);
    r.F.x = e.val - st.lvs - delta;
    V2 row_c, row_s, m_c, m_s;
    if (gauge == GAUGE_FIXED) {
        m_c = to_local(Jc, to_world(Js, V2{1, 0}));
        m_s = V2{1, 0};
        r.F.y = dot(rot90(m_c), uc);
        row_c = rot90(m_c);
        row_s = rot90(m_s);
    } else if (gauge == GAUGE_RAW) {
        m_c = to_local(Jc, st.g3s);
        m_s = st.gs;
        r.F.y = dot(rot90(m_c), uc);
        row_c = rot90(m_c);
        row_s = rot90(m_s) + st.Hs * rot90(us);
    } else {
        V3 mw = (st.g3s + e.grad) * 0.5;
        m_c = to_local(Jc, mw);
        m_s = to_local(Js, mw);
        r.F.y = dot(rot90(m_c), uc);
        row_c = rot90(m_c) - (e.hess * rot90(uc)) * 0.5;
        row_s = rot90(m_s) + (st.Hs * rot90(us)) * 0.5;
    }
    r.dFp = M2{gc.x, gc.y, row_c.x, row_c.y};
    r.det_dF = det(M2{-st.gs.x, -st.gs.y, -row_s.x, -row_s.y});
    return r;
}

// Trial 0 evaluates the start point itself, which is where the start-point
// terms come from (gradient, length and projected Hessian at the start point:
// the same field evaluation), so one evaluation serves both: the start terms
// are taken from it and the trial continues from it.
__device__ __forceinline__ void start_from(const LcEval& e, const Frame2& Js, StartTerms& t) {
    t.g3s = e.grad;
    t.gs = to_local(Js, e.grad);
    t.lvs = e.val;
    t.Hs = e.hess;
}

// ---------------------------------------------------------------------------
// replay: prefixes with k - 2 > 0 replayed bounces (hybrid_base_shift,
// shiftmap.hpp:459-528).  Only scenes with a non-reconnectable material (mirror,
// glossy roughness < 0.2) have records with k > 2; the host skips this stage
// for the others.

__global__ void __launch_bounds__(128)
    k_shift_replay(FrameView F0, FrameView F1, const GHit* g0, const GHit* g1, ResStore st0, ResStore st1,
                   ShiftQueue q, PathCfg cfg, unsigned long long* wq) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ FrameView sF[2];
    stage_two(F0, F1, sF, smem);
    const uint32_t j0 = q.ctl[0];
    uint32_t j1 = q.ctl[1];
    if (j1 > q.cap) j1 = uint32_t(q.cap);
    size_t njobs = j1 > j0 ? j1 - j0 : 0;
    TOFR_FOR_ITEMS(i, njobs, wq) {
        uint32_t k = j0 + uint32_t(i);
        Job jb = job_get(q, k);
        int dsel = (jb.meta & JOB_DST1) ? 1 : 0;
        const ResStore st = res_pin((jb.meta & JOB_REC1) ? st1 : st0, jb.item);
        Meta mt = ld_meta(st, jb.item);
        bool same_frame = ((jb.meta & JOB_SRC1) != 0) == (dsel != 0);
        bool identity = same_frame && jb.spx == jb.dpx && jb.spy == jb.dpy;
        if (!mt.valid || identity || mt.k == 2) continue;
        const FrameView& F = sF[dsel];
        if (!same_frame && mt.skind == SK_SURFACE && F.geo_motion) continue;
        Prefix p = replay_prefix(&F, dsel ? g1 : g0, jb.dpx, jb.dpy, st, jb.item, mt.k, cfg.use_rr);
        replay_put(q, k, p);
    }
}

// ---------------------------------------------------------------------------
// solve: checks, prefix, suffix, Newton (newton_solve, shiftmap.hpp:314-378)

// SP: the grids may be sparse (transient); !SP instantiations (gated grids)
// see slot == nullptr at compile time and drop the slot-map branches.
// Diagnostic build (-DTOFR_SOLVE_PROFILE=1, a tools variant): per solved job,
// {cycles from its refill to its finish, trial rounds it took part in, Newton
// iterations, re-projection rays, global timer (ns) at finish} for the latency-floor
// analysis of DESIGN 8 (tofr_gpu_debug_solve_profile).
#ifndef TOFR_SOLVE_PROFILE
#define TOFR_SOLVE_PROFILE 0
#endif
#if TOFR_SOLVE_PROFILE
constexpr unsigned kSolveProfCap = 1u << 22;
__device__ unsigned long long g_solve_prof[kSolveProfCap][3];
__device__ unsigned int g_solve_prof_n;
#endif

template <bool VEL, bool SP>
__global__ void __launch_bounds__(TOFR_SOLVE_BLOCK, TOFR_WAVE_MINB * 128 / TOFR_SOLVE_BLOCK)
    k_shift_solve(FrameView F0, FrameView F1, const GHit* g0, const GHit* g1, ResStore st0, ResStore st1,
                  ShiftQueue q, PathCfg cfg, unsigned long long* ctr_out, unsigned long long* wq) {
    if (!SP) st0.slot = st1.slot = nullptr;
    q.out.slot = nullptr;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ FrameView sF[2];
    stage_two(F0, F1, sF, smem);
    const uint32_t j0 = q.ctl[0];
    uint32_t j1 = q.ctl[1];
    if (j1 > q.cap) j1 = uint32_t(q.cap);
    const int lane = threadIdx.x & 31;
    // shift counters: CTA-wide in shared memory (keeps 9 registers free for the
    // Newton state); one global atomic per counter and CTA at the end
    __shared__ unsigned int sctr[SC_COUNT];
    if (threadIdx.x < SC_COUNT) sctr[threadIdx.x] = 0;
    __syncthreads();
#define SCTR(k, v) atomicAdd_block(&sctr[k], (unsigned)(v))

    // per-lane Newton state (one job at a time)
    bool active = false, exhausted = false, init = false, count = false, parked = false;
    uint32_t n_rays = 0;
    uint32_t job = 0;
    int dsel = 0;
    V3 p1{0, 0, 0}, p2{0, 0, 0}, spos{0, 0, 0}, cpos{0, 0, 0};
    int stri = 0, ctri = 0;
    bool cn_rec = true;  // current point's normal = the record's pn
    // tangent frames are per-triangle lookups (FrameView::tframe): the start
    // point's is tframe[stri], the current point's tframe[ctri]
    StartTerms stt;
    // velocity gates: the endpoint velocities are re-evaluated per trial from
    // their objects (velocity_at, the same inputs: the same values) instead of
    // held as six doubles per lane
    int vobj1 = -1, vobj2 = -1;
    double delta = 0, tol = 0, fnorm = 0, scale = 1;
    V2 step{0, 0};
    int iter = 0, bt = 0;
    bool pdl_fired = false;
#if TOFR_SOLVE_PROFILE
    long long prof_t0 = 0;
    unsigned prof_rounds = 0, prof_rays0 = 0;
#endif

    // small batches: busy lanes per warp if the jobs are spread over every warp
    const uint32_t n_warps = gridDim.x * (blockDim.x >> 5);
    const uint32_t share = j1 > j0 ? (j1 - j0 + n_warps - 1) / n_warps : 1u;
    const bool spread = TOFR_SHARE && share < 32;
    for (;;) {
        // ---- refill: idle lanes take the next jobs (one atomic per warp), but only
        // once at least TOFR_REFILL lanes are idle (or none is busy), so the
        // divergent setup code runs for many lanes at a time
        bool idle = !active && !exhausted;
        unsigned im = __ballot_sync(0xffffffffu, idle);
        unsigned bm = __ballot_sync(0xffffffffu, active);
        bool need = idle && (__popc(im) >= TOFR_REFILL || bm == 0);
#if TOFR_ESCALATE
        const unsigned slow_m = __ballot_sync(0xffffffffu, active && !init && (bt >= TOFR_ESCALATE || iter >= 2));
        if (slow_m) need = false;  // keep the freed lanes as helpers of the slow chains
#else
        const unsigned slow_m = 0;
#endif
        if (spread) {  // at most `share` busy lanes; the others stay free to help
            unsigned nm0 = __ballot_sync(0xffffffffu, need);
            int room = int(share) - __popc(bm);
            need = need && room > 0 && __popc(nm0 & ((1u << lane) - 1)) < room;
        }
        unsigned m = __ballot_sync(0xffffffffu, need);
        if (m) {
            int leader = __ffs(m) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(wq, (unsigned long long)__popc(m));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (need) {
                unsigned long long kk = j0 + base + __popc(m & ((1u << lane) - 1));
                if (kk >= j1) {
                    exhausted = true;
                } else {
                    // TOFR_SOLVE_REVERSE: take the queue from its end (order A/B;
                    // every job's result is independent of the order)
                    job = TOFR_SOLVE_REVERSE ? uint32_t(j1 - 1 - (kk - j0)) : uint32_t(kk);
                    Job jb = job_get(q, job);
                    dsel = (jb.meta & JOB_DST1) ? 1 : 0;
                    const FrameView& F = sF[dsel];
                    const ResStore st = res_pin((jb.meta & JOB_REC1) ? st1 : st0, jb.item);
                    count = (jb.meta & JOB_COUNT) != 0;
                    if (count) SCTR(SC_ATTEMPTS, 1);
                    Meta mt = ld_meta(st, jb.item);
                    bool same_frame = ((jb.meta & JOB_SRC1) != 0) == (dsel != 0);
                    bool ok = mt.valid && !(!same_frame && mt.skind == SK_SURFACE && F.geo_motion);
                    Prefix pre;
                    Suffix suf;
                    if (ok) {
                        bool identity = same_frame && jb.spx == jb.dpx && jb.spy == jb.dpy;
                        pre = job_prefix(F, dsel ? g1 : g0, jb, identity, st, mt, q, job, VEL);
                        ok = pre.ok;
                    }
                    if (ok) {
                        suf = job_suffix(F, st, jb.item, mt.skind, VEL);
                        ok = suf.ok;
                    }
                    if (!ok) {
                        if (count) SCTR(SC_REPLAY_FAILED, 1);
                        sol_fail(q, job);
                    } else {
                        spos = rec_p(st, jb.item);
                        stri = mt.ptri;
                        const bool shrink = (jb.meta & JOB_SHRINK) != 0;
                        if (!cfg.newton && !shrink) {  // shrink_map always solves
                            sol_put(q, job, spos, stri, 1.0, 3);
                        } else {
                            p1 = pre.p1;
                            p2 = suf.p2;
                            // full-path constraint, local two-segment target (length or velocity)
                            double src_total = VEL ? ld2(st, 22, jb.item).x : ld2(st, 1, jb.item).y;
                            double prefix_part = VEL ? pre.u : pre.len;
                            double suffix_part = VEL ? suf.u : suf.len;
                            double target_local;
                            if (shrink) {  // shrink_map: contract (expand) about the gate centre L0
                                const double L0 = jb.dc, K = cfg.shrink_k;
                                const double target_total =
                                    (jb.meta & JOB_FULL) ? (src_total - L0) / K + L0 : (src_total - L0) * K + L0;
                                target_local = target_total - prefix_part - suffix_part;
                            } else {
                                double gate_delta = jb.dc - jb.sc;
                                target_local = src_total + gate_delta - prefix_part - suffix_part;
                            }
                            if (VEL) {
                                vobj1 = F.tri[pre.tri1].obj;
                                vobj2 = suf.vobj;
                            }
                            tol = 0.01 * jb.dw;
                            if (count) SCTR(SC_SOLVES, 1);
                            // start terms and delta = target - (field at the start
                            // point) come with trial 0 (start_from)
                            delta = target_local;
                            // trial 0 evaluates the start point itself
                            cpos = spos;
                            ctri = stri;
                            cn_rec = true;
                            step = V2{0, 0};
                            scale = 1.0;
                            iter = 0;
                            bt = 0;
                            init = true;
                            active = true;
#if TOFR_SOLVE_PROFILE
                            prof_t0 = clock64();
                            prof_rounds = 0;
                            prof_rays0 = n_rays;
#endif
                        }
                    }
                }
            }
        }
        if (__all_sync(0xffffffffu, exhausted)) {
            work_add(cfg.work, WK_CLOSEST, n_rays);
            break;
        }
        // the queue is drained (every job is in a resident warp's hands): let
        // the dependent finish grid launch (PDL; a no-op without it)
        if (q.done && __any_sync(0xffffffffu, exhausted) && lane == 0 && !pdl_fired) {
            asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
            pdl_fired = true;
        }

        // ---- tail phase: once the queue is drained, idle lanes help the lowest
        // busy lane by evaluating the rest of its halving ladder (scale/2, /4, ...)
        // speculatively in the same round.  The trials of a ladder depend only on
        // the current point and step, so taking the first accepted one in ladder
        // order (and counting the rejections before it) is the sequential
        // newton_solve; the serial critical path of long solves shrinks instead.
        bool tail = false, helper = false, own = false;
        int owner = lane, hk = 0, K = 0;
        unsigned group = 1u << lane;
        {
            const bool free_lane = (TOFR_HELP_IDLE || spread || slow_m) ? !active : exhausted;
            unsigned idle = __ballot_sync(0xffffffffu, free_lane);
            // helpers go to the slow chains first while the queue still has work
            const bool drained = __any_sync(0xffffffffu, exhausted);
            unsigned cand = __ballot_sync(0xffffffffu, active && !init && !parked &&
                                                           (drained || !slow_m || ((slow_m >> lane) & 1u)));
            if (idle && cand) {
                // idle lanes are dealt out in rank order, H to each busy lane
                tail = true;
                const int nc = __popc(cand);
                const int H = min(8, max(1, __popc(idle) / nc));
                const int r = __popc(idle & ((1u << lane) - 1));
                const int j = r / H;
                if (free_lane && j < nc) {
                    unsigned m = cand;
                    #pragma unroll 1
                    for (int q = 0; q < j; ++q) m &= m - 1;
                    owner = __ffs(m) - 1;
                }
                int obt = __shfl_sync(0xffffffffu, bt, owner);
                hk = r % H + 1;
                helper = free_lane && j < nc && hk <= 8 - obt;
                if (!helper) owner = lane, hk = 0;
                group = __match_any_sync(0xffffffffu, owner);
                own = !helper && __popc(group) > 1;
                K = own ? __popc(group) - 1 : 0;
#define TOFR_BORROW(x)                                          \
    {                                                           \
        auto t_ = __shfl_sync(0xffffffffu, (x), owner);         \
        if (helper) (x) = t_;                                   \
    }
#define TOFR_BORROW3(v) TOFR_BORROW(v.x) TOFR_BORROW(v.y) TOFR_BORROW(v.z)
                TOFR_BORROW(dsel) TOFR_BORROW(ctri) TOFR_BORROW(cn_rec) TOFR_BORROW(scale) TOFR_BORROW(delta)
                TOFR_BORROW(fnorm) TOFR_BORROW(step.x) TOFR_BORROW(step.y)
                TOFR_BORROW3(cpos) TOFR_BORROW3(spos) TOFR_BORROW3(p1) TOFR_BORROW3(p2)
                TOFR_BORROW(stri)
                TOFR_BORROW3(stt.g3s) TOFR_BORROW(stt.gs.x) TOFR_BORROW(stt.gs.y) TOFR_BORROW(stt.lvs)
                TOFR_BORROW(stt.Hs.a) TOFR_BORROW(stt.Hs.b) TOFR_BORROW(stt.Hs.c) TOFR_BORROW(stt.Hs.d)
                if (VEL) {
                    TOFR_BORROW(vobj1) TOFR_BORROW(vobj2)
                }
#undef TOFR_BORROW3
#undef TOFR_BORROW
                if (helper) {
                    init = false;
                    #pragma unroll 1
                    for (int k = 0; k < hk; ++k) scale *= 0.5;
                }
            }
        }

        // ---- one Newton trial (trial 0 = the initial evaluation at the start point)
        const FrameView& F = sF[dsel];
        V3 tpos = cpos + to_world(F.tframe[ctri], step * scale);  // plane point
        int ttri = ctri;
        bool tn_rec = cn_rec, have = true;
        if (init) tpos = spos;
        // A plane point outside the current triangle needs re-projection rays
        // (reproject_to_mesh).  Such lanes park until TOFR_RAYBATCH lanes of the
        // warp need rays (or no other lane can proceed) and then trace together;
        // in the tail phase rays are traced at once.
        bool part = (active && !parked) || helper;
        bool need_ray = part && !init && !in_triangle(F, ctri, tpos);
        if (need_ray && !tail && active) parked = true;
        unsigned pm = __ballot_sync(0xffffffffu, parked);
        unsigned rm = __ballot_sync(0xffffffffu, active && !parked);
        bool trace_now = (parked && (tail || __popc(pm) >= TOFR_RAYBATCH || rm == 0)) || (tail && need_ray);
        if (trace_now) {
            if (parked) tpos = cpos + to_world(F.tframe[ctri], step * scale);
            SurfR r = reproject_rays(&F, ctri, tpos, p1);
            n_rays += uint32_t(r.rays);
            have = r.ok;
            if (have) {
                tpos = r.pos;
                ttri = r.tri;
                tn_rec = false;
            }
            parked = false;
        }
        unsigned em = __ballot_sync(0xffffffffu, (active && !parked) || helper);
        if (!((active && !parked) || helper)) continue;
#if TOFR_SOLVE_PROFILE
        if (active) ++prof_rounds;
#endif
        __syncwarp(em);
        const Frame2 Jt = F.tframe[ttri];
        const Frame2 Js = F.tframe[stri];
        VelField vf{{0, 0, 0}, {0, 0, 0}};
        if (VEL) vf = VelField{velocity_at(F, vobj1, p1), velocity_at(F, vobj2, p2)};
        LcEval ev = field_eval<VEL>(F, F.tri[ttri].obj, vf, p1, p2, tpos, Jt, cfg.gauge != GAUGE_FIXED);
        if (init) {
            start_from(ev, Js, stt);
            delta = delta - stt.lvs;  // field value at the start point
        }
        TrialEval et = trial_from(ev, spos, Js, stt, tpos, Jt, delta, cfg.gauge);
        double fn = hypot(et.F.x, et.F.y);
        bool accept = have && (init || fn < fnorm);
        if (tail) {
            // each owner takes the first accepted trial of its ladder
            unsigned hm = __ballot_sync(em, helper && accept);
            int src = (own && (group & hm)) ? __ffs(group & hm) - 1 : lane;
#define TOFR_TAKE(x)                                \
    {                                               \
        auto t_ = __shfl_sync(em, (x), src);        \
        if (take) (x) = t_;                         \
    }
#define TOFR_TAKE3(v) TOFR_TAKE(v.x) TOFR_TAKE(v.y) TOFR_TAKE(v.z)
            bool take = own && !accept && (group & hm) != 0;
            TOFR_TAKE3(tpos) TOFR_TAKE(ttri) TOFR_TAKE(tn_rec)
            TOFR_TAKE(et.F.x) TOFR_TAKE(et.F.y) TOFR_TAKE(et.dFp.a) TOFR_TAKE(et.dFp.b) TOFR_TAKE(et.dFp.c)
            TOFR_TAKE(et.dFp.d) TOFR_TAKE(et.det_dF) TOFR_TAKE(et.ngrad) TOFR_TAKE(fn)
#undef TOFR_TAKE3
#undef TOFR_TAKE
            if (own && !accept) {
                if (group & hm) {
                    accept = true;  // helper ladder trial accepted (bt is reset below)
                } else {
                    bt += K;  // K more rejected halvings; the owner's own rejection follows
                    #pragma unroll 1
                    for (int k = 0; k < K; ++k) scale *= 0.5;
                }
            }
            if (helper) continue;  // helpers only evaluate
        }
        bool fin = false, conv = false;
        double jac = 0;
        if (accept) {
            if (!init) ++iter;
            init = false;
            cpos = tpos;
            cn_rec = tn_rec;
            ctri = ttri;
            fnorm = fn;
            if (fabs(et.F.x) <= tol && fabs(et.F.y) <= tol) {
                double dc = det(et.dFp);
                double j = dc == 0 ? 0 : et.det_dF / dc;
                fin = true;
                conv = (j > 0) && isfinite(j);
                jac = j;
            } else if (iter >= 5 || et.ngrad < 1e-8 * F.diag || !solve2x2(et.dFp, -et.F, step)) {
                fin = true;
            } else {
                bt = 0;
                scale = 1.0;
            }
        } else if (++bt > 8) {
            fin = true;  // no halving accepted
        } else {
            scale *= 0.5;
        }
        if (fin) {
#if TOFR_SOLVE_PROFILE
            {
                unsigned k = atomicAdd(&g_solve_prof_n, 1u);
                if (k < kSolveProfCap) {
                    long long now = clock64();
                    unsigned long long gt;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
                    g_solve_prof[k][0] = (unsigned long long)(now - prof_t0);
                    g_solve_prof[k][1] = (unsigned long long)prof_rounds | ((unsigned long long)iter << 32) |
                                         ((unsigned long long)(n_rays - prof_rays0) << 40);
                    g_solve_prof[k][2] = gt;
                }
            }
#endif
            if (cfg.row_cost)  // the job's destination row: Newton iterations + setup and finish
                atomicAdd(&cfg.row_cost[job_get(q, job).dpy], (unsigned long long)(iter) + 4ull);
            if (count) SCTR(SC_ITERATIONS, iter);
            if (conv && !F.mats[F.tri[ctri].mat].reconnectable) {
                if (count) {
                    SCTR(SC_NEWTON_OK, 1);
                    SCTR(SC_NEWTON_FAILED, 1);
                }
                sol_fail(q, job);
            } else if (conv) {
                if (count) SCTR(SC_NEWTON_OK, 1);
                sol_put(q, job, cpos, ctri, jac, cn_rec ? 3 : 1);
            } else {
                if (count) SCTR(SC_NEWTON_FAILED, 1);
                sol_fail(q, job);
            }
            active = false;
        }
    }
    __syncthreads();
    if (ctr_out && threadIdx.x < SC_COUNT && sctr[threadIdx.x])
        atomicAdd(&ctr_out[threadIdx.x], (unsigned long long)sctr[threadIdx.x]);
#undef SCTR
}

// ---------------------------------------------------------------------------
// finish: occlusion, Jacobian, rebuild (shift_sample tail + rebuild_sample,
// shiftmap.hpp:579-654, :740-783), output

// Bvh::occluded, counting the rays it traces
__device__ __forceinline__ bool occluded_n(const FrameView& F, const V3& a, const V3& b, uint32_t& nr) {
    V3 dd = b - a;
    double dist = norm(dd);
    if (dist <= 2 * F.eps_ray) return false;
    ++nr;
    V3 d = dd / dist;
    return trace_any(F, a, d, F.eps_ray, dist - F.eps_ray);
}

__device__ __forceinline__ void out_fail(const ShiftQueue& q, uint32_t k) { st2(q.out, 0, k, 0.0, 0.0); }

template <bool VEL, bool SP>
__global__ void __launch_bounds__(128, TOFR_FINISH_MINB)
    k_shift_finish(FrameView F0, FrameView F1, const GHit* g0, const GHit* g1, ResStore st0, ResStore st1,
                   ShiftQueue q, PathCfg cfg, unsigned long long* ctr_out, unsigned long long* wq) {
    if (!SP) st0.slot = st1.slot = nullptr;
    q.out.slot = nullptr;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ FrameView sF[2];
    stage_two(F0, F1, sF, smem);
    const uint32_t j0 = q.ctl[0];
    uint32_t j1 = q.ctl[1];
    if (j1 > q.cap) j1 = uint32_t(q.cap);
    size_t njobs = j1 > j0 ? j1 - j0 : 0;
    Ctr ctr;
#pragma unroll
    for (int k = 0; k < SC_COUNT; ++k) ctr.v[k] = 0;
    uint32_t n_any = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0 && cfg.work && njobs) atomicAdd(&cfg.work[WK_JOBS], (unsigned long long)njobs);
    TOFR_FOR_ITEMS(i, njobs, wq) {
        uint32_t k = j0 + uint32_t(i);
        sol_wait(q, k);
        double2 c6 = jld(q, 6, k);
        int2 ts;
        memcpy(&ts, &c6.y, 8);
        if (!(ts.y & 1)) {
            out_fail(q, k);
            continue;
        }
        Job jb = job_get(q, k);
        int dsel = (jb.meta & JOB_DST1) ? 1 : 0;
        const FrameView& F = sF[dsel];
        const ResStore st = res_pin((jb.meta & JOB_REC1) ? st1 : st0, jb.item);
        bool count = (jb.meta & JOB_COUNT) != 0;
        Meta mt = ld_meta(st, jb.item);
        bool same_frame = ((jb.meta & JOB_SRC1) != 0) == (dsel != 0);
        bool identity = same_frame && jb.spx == jb.dpx && jb.spy == jb.dpy;
        Prefix pre = job_prefix(F, dsel ? g1 : g0, jb, identity, st, mt, q, k, VEL);
        Suffix suf = job_suffix(F, st, jb.item, mt.skind, VEL);
        double2 c4 = jld(q, 4, k), c5 = jld(q, 5, k);
        V3 ppos{c4.x, c4.y, c5.x};
        int ptri = ts.x;
        V3 pnrm = (ts.y & 2) ? rec_pn(st, jb.item) : F.tri[ptri].n;
        double j_newton = c5.y;
        // the two occlusion tests of shift_sample (shiftmap.hpp:765-767) as one
        // loop around a single traversal site, so lanes stay converged
        bool occ = false;
        for (int r = 0; r < 2 && !occ; ++r) {
            V3 a = r == 0 ? pre.p1 : ppos, bpt = r == 0 ? ppos : suf.p2;
            V3 dd = bpt - a;
            double dist = norm(dd);
            if (dist <= 2 * F.eps_ray) continue;  // Bvh::occluded: nothing between
            ++n_any;
            V3 dir = dd / dist;
            occ = trace_ray_impl(F.nodes, F.tri_isect, a, dir, F.eps_ray, dist - F.eps_ray, true).slot >= 0;
        }
        if (occ) {
            if (count) ctr.v[SC_OCCLUDED]++;
            out_fail(q, k);
            continue;
        }
        double rec_prefix_pdf = st.compact ? res_prefix_derived(st, jb.item).pdf : ld2(st, 5, jb.item).x;
        double jac = (rec_prefix_pdf / pre.pdf) * j_newton;
        if (!isfinite(jac) || jac < cfg.jac_min || jac > cfg.jac_max) {
            if (count) ctr.v[SC_JAC_CLAMPED]++;
            out_fail(q, k);
            continue;
        }
        const bool shrink = (jb.meta & JOB_SHRINK) != 0;
        if (shrink) jac = jac * ((jb.meta & JOB_FULL) ? 1.0 / cfg.shrink_k : cfg.shrink_k);
        // rebuild_sample
        V3 d1 = ppos - pre.p1;
        double l1 = norm(d1);
        V3 d2 = suf.p2 - ppos;
        double l2 = norm(d2);
        bool ok = !(l1 <= 2 * F.eps_ray) && !(l2 <= 2 * F.eps_ray);
        V3 f = splat(0);
        int m2 = -1;
        double u_total = 0;
        if (ok) {
            V3 u1 = d1 / l1;
            V3 u2 = d2 / l2;
            V3 pvel = splat(0);
            if (VEL) {
                pvel = velocity_at(F, F.tri[ptri].obj, ppos);
                u_total = pre.u + dot(velocity_at(F, F.tri[pre.tri1].obj, pre.p1) - pvel, u1);
            }
            const GMat& m1 = F.mats[pre.m1];
            f = pre.fw * eval_bsdf(m1, pre.n1, pre.wi1, u1) * geom_term(pre.p1, pre.n1, ppos, pnrm);
            const GMat& mp = F.mats[F.tri[ptri].mat];
            f = f * eval_bsdf(mp, pnrm, -u1, u2);
            if (mt.skind == SK_SURFACE) {
                V3 sf = rec_suffix_f(st, jb.item, m2);
                V3 n2 = suf.n2, p2 = suf.p2;
                const GMat& mm2 = F.mats[m2];
                V3 f2 = mm2.kind == MAT_MIRROR ? splat(0) : eval_bsdf(mm2, n2, -u2, rec_wo2(st, jb.item));
                f = f * (geom_term(ppos, pnrm, p2, n2) * f2 * sf);
            } else if (mt.skind == SK_LIGHT) {
                LightSample ls;
                if (!light_sample(F.light, ppos, ls)) {
                    f = splat(0);
                } else {
                    f = f * (fabs(dot(pnrm, u2)) * ls.value);
                }
            } else {
                V3 fs = eval_bsdf(F.mats[F.lsub.mat], F.lsub.n, -u2, F.lsub.wo_light);
                f = f * (geom_term(ppos, pnrm, F.lsub.pos, F.lsub.n) * fs * F.lsub.power);
            }
            if (VEL) u_total += dot(pvel - suf.v2, u2) + suf.u;
            ok = finite3(f);
        }
        if (!ok) {
            if (count) ctr.v[SC_REPLAY_FAILED]++;
            out_fail(q, k);
            continue;
        }
        double len = pre.len + l1 + l2 + suf.len;
        double gv = gate_value(VEL, len, u_total);
        if (count && gate_w(jb.dc, jb.dw, gv) > 0 && luminance(f) > 0) ctr.v[SC_SUCCESS]++;
        if (!(jb.meta & JOB_FULL)) {  // inverse shift: p-hat of the source gate times |J|
            const double sw = shrink ? jb.dw * cfg.shrink_k : jb.dw;  // shrink: the wide gate
            st2(q.out, 0, k, luminance(f) * gate_w(jb.dc, sw, gv) * jac, 1.0);
            continue;
        }
        // mapped record (rebuild_sample's record update, stored as res_store would)
        const ResStore& o = q.out;
        st2(o, 0, k, jac, 1.0);
        st2(o, 1, k, 0.0, len);
        st2(o, 2, k, f.x, f.y);
        double suffix_len = mt.skind == SK_LIGHTSUB ? F.lsub.chain_len : ld2(st, 3, jb.item).y;
        st2(o, 3, k, f.z, suffix_len);
        {
            Meta om = mt;
            om.has = 1;
            om.pad0 = om.pad1 = 0;
            om.tri1 = pre.tri1;
            om.ptri = ptri;
            double2 v;
            memcpy(&v, &om, 16);
            st2(o, 4, k, v.x, v.y);
        }
        st2(o, 5, k, pre.pdf, pre.len);
        st2(o, 6, k, pre.fw.x, pre.fw.y);
        st2(o, 7, k, pre.fw.z, pre.p1.x);
        st2(o, 8, k, pre.p1.y, pre.p1.z);
        st2(o, 9, k, pre.wi1.x, pre.wi1.y);
        st2(o, 10, k, pre.wi1.z, ppos.x);
        st2(o, 11, k, ppos.y, ppos.z);
        st2(o, 12, k, pnrm.x, pnrm.y);
        V3 p2o = mt.skind == SK_LIGHTSUB ? F.lsub.pos : (mt.skind == SK_LIGHT ? F.light.pos : suf.p2);
        st2(o, 13, k, pnrm.z, p2o.x);
        st2(o, 14, k, p2o.y, p2o.z);
        double2 c15 = ld2(st, 15, jb.item), c16 = ld2(st, 16, jb.item);
        if (mt.skind == SK_LIGHTSUB) {
            c15 = make_double2(F.lsub.n.x, F.lsub.n.y);
            c16.x = F.lsub.n.z;
        }
        st2r(o, 15, k, c15);
        st2r(o, 16, k, c16);
        {
            const size_t sr = res_row(st, jb.item);
            for (int c = 17; c < (mt.nl > 0 ? 22 : 20); ++c) st2r(o, c, k, ld2r(st, c, sr));
        }
        if (VEL) {
            st2(o, 22, k, u_total, pre.u);
            st2(o, 23, k, mt.skind == SK_LIGHTSUB ? suf.u : ld2(st, 23, jb.item).x, 0.0);
        }
    }
    work_add(cfg.work, WK_ANY, n_any);
    ctr_flush(ctr, ctr_out);
}

// ---------------------------------------------------------------------------
// merge-side helpers

// chunks [from, 24) of the record at row ri -> row rj, without the replay
// lanes (20-21) unless the record has lanes
__device__ __forceinline__ void copy_chunks_r(const ResStore& src, size_t ri, const ResStore& dst, size_t rj,
                                              int from, int n_lanes, bool vel) {
    for (int c = from; c < (vel ? kResChunks : 22); ++c) {
        if ((c == 20 || c == 21) && n_lanes <= 0) continue;
        st2r(dst, c, rj, ld2r(src, c, ri));
    }
}

// Selected mapped record (job k) -> reservoir `it` with the merge's W, M, p-hat.
// (Rows looked up once: every slot-map read is a separate volatile load.)
__device__ __forceinline__ void put_mapped(const ResStore& o, uint32_t k, const ResStore& dst, size_t it, double W,
                                           double M, double phat, bool vel) {
    st2(dst, 0, it, W, M);
    const size_t ro = res_row(o, k), rj = res_row_w(dst, it);
    st2r(dst, 1, rj, make_double2(phat, ld2r(o, 1, ro).y));
    double2 c4 = ld2r(o, 4, ro);
    Meta mt;
    memcpy(&mt, &c4, 16);
    copy_chunks_r(o, ro, dst, rj, 2, mt.nl, vel);
}

// Reservoir copy src[it] -> dst[it] with a new W, M (sample and p-hat kept).
__device__ __forceinline__ void copy_res(const ResStore& src, const ResStore& dst, size_t it, double W, double M,
                                         bool vel) {
    st2(dst, 0, it, W, M);
    const size_t ri = res_row(src, it), rj = res_row_w(dst, it);
    double2 c4 = ld2r(src, 4, ri);
    Meta mt;
    memcpy(&mt, &c4, 16);
    copy_chunks_r(src, ri, dst, rj, 1, mt.nl, vel);
}

// header (W, M, has, p-hat) of a reservoir
__device__ __forceinline__ void res_head_phat(const ResStore& s, size_t i, Res& r) {
    res_load_head(s, i, r);
    if (r.has) r.phat = ld2(s, 1, i).x;
}

// forward-shift output of job k: ok, Jacobian, mapped f and gate value
// (length, or path velocity for Doppler gates)
__device__ __forceinline__ void fwd_output(const ShiftQueue& q, uint32_t k, int gate_vel, MergeShift& ms,
                                           Sample& mapped, double& gv) {
    if (k == kNoJob) return;
    double2 o0 = ld2(q.out, 0, k);
    if (!(o0.y > 0)) return;
    ms.valid = 1;
    ms.jac = o0.x;
    double2 o2 = ld2(q.out, 2, k), o3 = ld2(q.out, 3, k);
    gv = gate_vel ? ld2(q.out, 22, k).x : ld2(q.out, 1, k).y;
    mapped.f = V3{o2.x, o2.y, o3.x};
}

__device__ __forceinline__ double inv_output(const ShiftQueue& q, uint32_t k) {
    if (k == kNoJob) return 0.0;
    double2 o0 = ld2(q.out, 0, k);
    return o0.y > 0 ? o0.x : 0.0;
}

// ---------------------------------------------------------------------------
// temporal reuse (stage::temporal_reuse, pipeline.hpp:209-229)

// ws.tsrc holds, per pixel of the band, the reprojected source pixel qy * W + qx
// (or ~0: no primary hit, off-screen, or outside the rows the band holds);
// job maps are written only for items that have the job (the apply kernel
// reads them under the same non-emptiness tests).
// Reprojection of each band pixel's primary hit into the previous camera
// (temporal_reuse, pipeline.hpp:213-219): ws.tsrc[pixel] = source pixel or ~0.
__global__ void k_temporal_reproject(FrameView Fc, Band bd, const GHit* gc, FrameView Fp, WaveScratch ws) {
    int W = Fc.cam.w;
    size_t n = size_t(bd.y1 - bd.y0) * W;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        int p = bd.y0 * W + int(i);
        int px = p % W, py = p / W;
        uint64_t src_pix = ~uint64_t(0);
        GHit g = gc[p];
        int qx, qy;
        if (g.tri >= 0) {
            V3 d0 = primary_dir(Fc.cam, px, py);
            V3 hp = Fc.cam.pos + d0 * g.t;
            if (project(Fp.cam, hp, qx, qy)) {
                if (qy < bd.t0 || qy >= bd.t1)  // reprojection left the rows this band holds
                    atomicAdd(bd.err, 1ull);
                else
                    src_pix = uint64_t(qy) * W + qx;
            }
        }
        ws.tsrc[i] = src_pix;
    }
}

// TOFR_PREP_ITEMS items per thread and block append: every item's loads
// (reprojected source pixel, both headers) are issued before the append's
// barriers, so a thread keeps several dependent-load chains in flight and the
// block waits at its barriers once per TOFR_PREP_ITEMS x 256 items
// (stages of at least kPrepItemsMin items: the transient grids; smaller
// stages -- gated frames -- keep one item per thread, measured faster there:
// their grids need every thread the machine holds, profiles/r02/ab_prep_items.txt)
#ifndef TOFR_PREP_ITEMS
#define TOFR_PREP_ITEMS 4
#endif
constexpr size_t kPrepItemsMin = size_t(1) << 22;
template <int KP>
__global__ void __launch_bounds__(256, KP > 1 ? 4 : 1)
    k_temporal_prep(FrameView Fc, Band bd, const GHit* gc, FrameView Fp, GateGrid cg, GateGrid pg, PathCfg cfg,
                    ResStore cur, ResStore prev, WaveScratch ws) {
    int W = Fc.cam.w, B = cg.transient ? cg.h.bins : 1;
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    const size_t tile = size_t(blockDim.x) * KP;
    const size_t n_round = (n + tile - 1) / tile * tile;  // block-uniform trip count
    __shared__ uint32_t sh[33];
    for (size_t t0 = blockIdx.x * tile; t0 < n_round; t0 += size_t(gridDim.x) * tile) {
        // item k of this thread: t0 + k * blockDim.x + threadIdx.x (coalesced per k)
        uint64_t sp[KP];
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            const size_t i = t0 + size_t(k) * blockDim.x + threadIdx.x;
            sp[k] = ~uint64_t(0);
            if (i < n) sp[k] = ws.tsrc[size_t((base + i) / B) - size_t(bd.y0) * W];
        }
        double2 s0[KP], c0[KP];
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            const size_t i = t0 + size_t(k) * blockDim.x + threadIdx.x;
            s0[k] = make_double2(0.0, 0.0);
            c0[k] = make_double2(0.0, 0.0);
            if (sp[k] != ~uint64_t(0)) {
                const size_t it = base + i;
                s0[k] = ld2(prev, 0, size_t(sp[k]) * B + it % B);
                c0[k] = ld2(cur, 0, it);
            }
        }
        uint32_t fm = 0, im = 0, mm = 0;  // per-item bits: forward job, inverse job, merge
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            if (sp[k] == ~uint64_t(0) || !(s0[k].y > 0)) continue;
            const bool fwd = s0[k].x > 0, inv = c0[k].x > 0;
            if (fwd) fm |= 1u << k;
            if (inv) im |= 1u << k;
            if (fwd || inv) {
                mm |= 1u << k;
            } else {  // both empty: the merge only adds the confidences (no RNG draw)
                const size_t i = t0 + size_t(k) * blockDim.x + threadIdx.x;
                res_store_w(cur, base + i, 0.0, dmin(c0[k].y + s0[k].y, cfg.m_cap));
            }
        }
        // the items' jobs (forward, then inverse, in item order) and merge-list
        // entries in one block-wide append
        uint32_t mfirst = 0;
        uint32_t kj = block_append_jobs_n(ws, uint32_t(__popc(fm) + __popc(im)), uint32_t(__popc(mm)), &mfirst,
                                          bd.err, cfg.work, sh);
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            const size_t i = t0 + size_t(k) * blockDim.x + threadIdx.x;
            if ((mm >> k) & 1u) ws.mlist[mfirst++] = uint32_t(i);
            const bool fwd = (fm >> k) & 1u, inv = (im >> k) & 1u;
            if (!(fwd || inv) || kj == kNoJob) continue;
            const size_t it = base + i;
            const int p = int(it / B), b = int(it % B);
            const int px = p % W, py = p / W;
            const int qx = int(sp[k] % W), qy = int(sp[k] / W);
            const size_t src_i = size_t(sp[k]) * B + b;
            double dc, dw, sc, sw;
            gate_of(cg, b, dc, dw);
            gate_of(pg, b, sc, sw);
            if (fwd) {
                job_put(ws.q, kj, src_i, JOB_REC1 | JOB_SRC1 | JOB_FULL | JOB_COUNT, qx, qy, px, py, sc, dc, dw);
                ws.map_a[i] = kj++;
            }
            if (inv) {
                job_put(ws.q, kj, it, JOB_DST1, px, py, qx, qy, dc, sc, sw);
                ws.map_b[i] = kj++;
            }
        }
    }
}

// merge kernels: chains of dependent gathers (merge list -> source pixel ->
// slot map -> pool row -> chunks), latency-bound; TOFR_APPLY_MINB resident
// 256-thread CTAs per SM trade registers for loads in flight
#ifndef TOFR_APPLY_MINB
#define TOFR_APPLY_MINB 5
#endif
__global__ void __launch_bounds__(256, TOFR_APPLY_MINB)
    k_temporal_apply(Band bd, int W, GateGrid cg, PathCfg cfg, int frame_idx, ResStore cur,
                                 ResStore prev, WaveScratch ws) {
    int B = cg.transient ? cg.h.bins : 1;
    size_t base = size_t(bd.y0) * W * B;
    uint32_t cnt = ws.q.ctl[3];
    for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < cnt; l += gridDim.x * blockDim.x) {
        size_t i = ws.mlist[l], it = base + i;
        int p = int(it / B), b = int(it % B);
        size_t src_i = size_t(ws.tsrc[size_t(p) - size_t(bd.y0) * W]) * B + b;
        Res dst, src;
        res_load_head(prev, src_i, src);
        res_load_head(cur, it, dst);
        if (dst.has) dst.phat = ld2(cur, 1, it).x;
        if (src.has) src.phat = ld2(prev, 1, src_i).x;
        int px = p % W, py = p / W;
        double dc, dw;
        gate_of(cg, b, dc, dw);
        MergeShift ms{0, 1.0, 0.0};
        Sample mapped;
        double mgv = 0;
        uint32_t kf = src.has ? ws.map_a[i] : kNoJob;
        fwd_output(ws.q, kf, cfg.gate_vel, ms, mapped, mgv);
        ms.phat_src_of_dst = inv_output(ws.q, dst.has ? ws.map_b[i] : kNoJob);
        uint64_t pix = uint64_t(py) * W + px;
        Rng rng = rng_make(cfg.seed, uint64_t(frame_idx), pix, uint64_t(b), 8);
        int which = gris_merge(dst, src, ms, mapped, mgv, dc, dw, cfg.m_cap, rng);
        if (which == 2)
            put_mapped(ws.q.out, kf, cur, it, dst.W, dst.M, dst.phat, cfg.gate_vel);
        else  // in place: the kept sample and its p-hat are already stored
            res_store_w(cur, it, dst.W, dst.M);
    }
}

// ---------------------------------------------------------------------------
// spatial reuse (stage::spatial_reuse, pipeline.hpp:232-269): forward shifts of
// every (neighbour j, item) pair first, then per neighbour the inverse shifts
// of the running output and the merge (the running output and the lane-10 RNG
// position stay in HBM between neighbours; same draws in the same order).

// neighbor_offset (pipeline.hpp:232-239) of every band pixel and neighbour for
// this pass: the offsets depend on the pixel alone, so the prep and merge
// kernels of every item (and every bin) read them instead of re-evaluating
// the rotation hash and sin / cos
__global__ void k_spatial_offsets(Band bd, int W, PathCfg cfg, SpatialParams sp, int pass, int frame_idx,
                                  WaveScratch ws) {
    size_t npx = size_t(bd.y1 - bd.y0) * W;
    for (size_t lp = blockIdx.x * size_t(blockDim.x) + threadIdx.x; lp < npx; lp += size_t(gridDim.x) * blockDim.x) {
        size_t p = size_t(bd.y0) * W + lp;
        uint64_t rk = spatial_rot_key(uint64_t(p), pass, cfg.seed, frame_idx);
        for (int j = 0; j < sp.neighbors; ++j) {
            int dx, dy;
            neighbor_offset(j, sp.neighbors, sp.radius, rk, dx, dy);
            ws.nbr[size_t(j) * npx + lp] = pack_offset(dx, dy);
        }
    }
}

// The spatial prep kernels take TOFR_PREP_ITEMS items per thread per block
// append, like k_temporal_prep: the neighbour lookups and header gathers of
// all of them are in flight before the append's barriers.
template <int KP>
__global__ void __launch_bounds__(256, KP > 1 ? 4 : 1)
    k_spatial_prep_fwd(FrameView F, Band bd, PathCfg cfg, GateGrid gate, SpatialParams sp, int pass, int frame_idx,
                       ResStore src_grid, WaveScratch ws) {
    int W = F.cam.w, H = F.cam.h, B = gate.transient ? gate.h.bins : 1;
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    const size_t npx = size_t(bd.y1 - bd.y0) * W;
    const size_t tile = size_t(blockDim.x) * KP;
    const size_t n_round = (n + tile - 1) / tile * tile;  // block-uniform trip count
    __shared__ uint32_t sh[33];
    for (size_t t0 = blockIdx.x * tile; t0 < n_round; t0 += size_t(gridDim.x) * tile) {
        for (int j = 0; j < sp.neighbors; ++j) {
            int nx[KP], ny[KP];
            size_t si[KP];
            uint32_t wm = 0;
            // every non-empty neighbour is a forward shift attempt (counted even
            // when its record has no reconnection vertex, as the reference does)
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                const size_t i = t0 + size_t(k) * blockDim.x + threadIdx.x;
                nx[k] = ny[k] = 0;
                si[k] = 0;
                if (i < n) {
                    const size_t it = base + i;
                    const int p = int(it / B), b = int(it % B);
                    const size_t lp = size_t(p) - size_t(bd.y0) * W;
                    if (spatial_neighbor_at(bd, W, H, B, p % W, p / W, b, ws.nbr[size_t(j) * npx + lp], src_grid,
                                            nx[k], ny[k], si[k]) &&
                        ld2(src_grid, 0, si[k]).x > 0)
                        wm |= 1u << k;
                }
            }
            uint32_t mfirst = 0;
            uint32_t kj = block_append_jobs_n(ws, uint32_t(__popc(wm)), 0u, &mfirst, bd.err, nullptr, sh);
#pragma unroll
            for (int k = 0; k < KP; ++k) {
                const size_t i = t0 + size_t(k) * blockDim.x + threadIdx.x;
                if (i >= n) continue;
                uint32_t slot = kNoJob;
                if (((wm >> k) & 1u) && kj != kNoJob) {
                    const size_t it = base + i;
                    const int p = int(it / B), b = int(it % B);
                    double dc, dw;
                    gate_of(gate, b, dc, dw);
                    slot = kj++;
                    job_put(ws.q, slot, si[k], JOB_FULL | JOB_COUNT, nx[k], ny[k], p % W, p / W, dc, dc, dw);
                }
                ws.map_a[size_t(j) * n + i] = slot;
            }
        }
    }
}

template <int KP>
__global__ void __launch_bounds__(256, KP > 1 ? 4 : 1)
    k_spatial_prep_inv(FrameView F, Band bd, PathCfg cfg, GateGrid gate, SpatialParams sp, int pass, int j,
                       int frame_idx, ResStore src_grid, ResStore dst_grid, WaveScratch ws) {
    int W = F.cam.w, H = F.cam.h, B = gate.transient ? gate.h.bins : 1;
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    const size_t npx = size_t(bd.y1 - bd.y0) * W;
    const size_t tile = size_t(blockDim.x) * KP;
    const size_t n_round = (n + tile - 1) / tile * tile;  // block-uniform trip count
    __shared__ uint32_t sh[33];
    const ResStore& out_grid = j == 0 ? src_grid : dst_grid;
    for (size_t t0 = blockIdx.x * tile; t0 < n_round; t0 += size_t(gridDim.x) * tile) {
        int nx[KP], ny[KP];
        size_t si[KP];
        double2 o0[KP], s0[KP];
        uint32_t nb = 0;  // items whose neighbour j exists
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            const size_t i = t0 + size_t(k) * blockDim.x + threadIdx.x;
            nx[k] = ny[k] = 0;
            si[k] = 0;
            o0[k] = s0[k] = make_double2(0.0, 0.0);
            if (i >= n) continue;
            const size_t it = base + i;
            const int p = int(it / B), b = int(it % B);
            const size_t lp = size_t(p) - size_t(bd.y0) * W;
            if (spatial_neighbor_at(bd, W, H, B, p % W, p / W, b, ws.nbr[size_t(j) * npx + lp], src_grid, nx[k],
                                    ny[k], si[k])) {
                nb |= 1u << k;
                o0[k] = ld2(out_grid, 0, it);
                s0[k] = ld2(src_grid, 0, si[k]);
            } else if (j == 0) {
                o0[k] = ld2(src_grid, 0, it);  // the pass input's header (copied below)
            }
        }
        uint32_t wm = 0, mm = 0;  // inverse job, merge
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            const size_t i = t0 + size_t(k) * blockDim.x + threadIdx.x;
            if (i >= n) continue;
            const size_t it = base + i;
            if (!((nb >> k) & 1u)) {
                if (j == 0) {  // the output starts as the pass input
                    if (o0[k].x > 0)
                        copy_res(src_grid, dst_grid, it, o0[k].x, o0[k].y, cfg.gate_vel);
                    else
                        res_store_w(dst_grid, it, 0.0, o0[k].y);
                    if (j + 1 < sp.neighbors) ws.rng_ctr[i] = 0;
                }
                continue;
            }
            const bool want = o0[k].x > 0, merge = want || s0[k].x > 0;
            if (want) wm |= 1u << k;
            if (merge) {
                mm |= 1u << k;
            } else {  // both empty: the merge only adds the confidences (no RNG draw)
                res_store_w(dst_grid, it, 0.0, dmin(o0[k].y + s0[k].y, cfg.m_cap));
                if (j == 0 && j + 1 < sp.neighbors) ws.rng_ctr[i] = 0;
            }
        }
        uint32_t mfirst = 0;
        uint32_t kj = block_append_jobs_n(ws, uint32_t(__popc(wm)), uint32_t(__popc(mm)), &mfirst, bd.err, cfg.work,
                                          sh);
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            const size_t i = t0 + size_t(k) * blockDim.x + threadIdx.x;
            if ((mm >> k) & 1u) ws.mlist[mfirst++] = uint32_t(i);
            if (!((wm >> k) & 1u) || kj == kNoJob) continue;
            const size_t it = base + i;
            const int p = int(it / B), b = int(it % B);
            double dc, dw;
            gate_of(gate, b, dc, dw);
            job_put(ws.q, kj, it, j == 0 ? 0u : JOB_REC1, p % W, p / W, nx[k], ny[k], dc, dc, dw);
            ws.map_b[i] = kj++;
        }
    }
}

__global__ void __launch_bounds__(256, TOFR_APPLY_MINB) k_spatial_apply(FrameView F, Band bd, PathCfg cfg, GateGrid gate, SpatialParams sp, int pass, int j,
                                int frame_idx, ResStore src_grid, ResStore dst_grid, WaveScratch ws) {
    int W = F.cam.w, H = F.cam.h, B = gate.transient ? gate.h.bins : 1;
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    uint32_t cnt = ws.q.ctl[3];
    for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < cnt; l += gridDim.x * blockDim.x) {
        size_t i = ws.mlist[l], it = base + i;
        int p = int(it / B), b = int(it % B);
        int px = p % W, py = p / W;
        uint64_t pix = uint64_t(py) * W + px;
        int nx, ny;
        size_t si = 0;
        const size_t npx = size_t(bd.y1 - bd.y0) * W, lp = size_t(p) - size_t(bd.y0) * W;
        spatial_neighbor_at(bd, W, H, B, px, py, b, ws.nbr[size_t(j) * npx + lp], src_grid, nx, ny, si);
        Res out, src;
        res_load_head(j == 0 ? src_grid : dst_grid, it, out);
        res_load_head(src_grid, si, src);
        if (out.has) out.phat = ld2(j == 0 ? src_grid : dst_grid, 1, it).x;
        if (src.has) src.phat = ld2(src_grid, 1, si).x;
        double dc, dw;
        gate_of(gate, b, dc, dw);
        MergeShift ms{0, 1.0, 0.0};
        Sample mapped;
        double mgv = 0;
        uint32_t kf = src.has ? ws.map_a[size_t(j) * n + i] : kNoJob;
        fwd_output(ws.q, kf, cfg.gate_vel, ms, mapped, mgv);
        ms.phat_src_of_dst = inv_output(ws.q, out.has ? ws.map_b[i] : kNoJob);
        Rng rng = rng_make(cfg.seed, uint64_t(frame_idx), pix, uint64_t(pass * 131 + b), 10);
        if (j > 0) rng.ctr = ws.rng_ctr[i];
        int which = gris_merge(out, src, ms, mapped, mgv, dc, dw, cfg.m_cap, rng);
        if (which == 2)
            put_mapped(ws.q.out, kf, dst_grid, it, out.W, out.M, out.phat, cfg.gate_vel);
        else if (which == 1 && j == 0)
            copy_res(src_grid, dst_grid, it, out.W, out.M, cfg.gate_vel);
        else  // kept in place (j > 0) or empty
            res_store_w(dst_grid, it, out.W, out.M);
        if (j + 1 < sp.neighbors) ws.rng_ctr[i] = rng.ctr;
    }
}

// ---------------------------------------------------------------------------
// bin reuse (stage::bin_reuse, pipeline.hpp:273-299): every pixel-bin merges
// bins b - 1 and b + 1 of its own pixel, in that order, on the spatial pass's
// scheme -- the forward shifts of both neighbours in one batch, then per
// neighbour j the inverse shift of the current output, the shifts, the merge.
// A shift between bins keeps the pixel (stored prefix) and moves the path
// length by the bin pitch (the Newton target's gate delta).

// neighbour j (0: b - 1, 1: b + 1) of item p * B + b; false when outside the
// bins or empty of confidence (bin_reuse skips src.M <= 0)
__device__ __forceinline__ bool bin_neighbor(int B, size_t p, int b, int j, const ResStore& src, int& nb,
                                             size_t& si) {
    nb = j == 0 ? b - 1 : b + 1;
    if (nb < 0 || nb >= B) return false;
    si = p * size_t(B) + size_t(nb);
    return ld2(src, 0, si).y > 0;
}

__global__ void k_bin_prep_fwd(Band bd, int W, GateGrid gate, ResStore src_grid, WaveScratch ws) {
    const int B = gate.h.bins;
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t n_round = (n + blockDim.x - 1) / blockDim.x * blockDim.x;  // block-uniform trip count
    __shared__ uint32_t sh[33];
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n_round; i += stride) {
        bool live = i < n;
        size_t it = base + (live ? i : 0);
        size_t p = it / B;
        int b = int(it % B);
        int px = int(p % W), py = int(p / W);
        double dc, dw;
        gate_of(gate, b, dc, dw);
        for (int j = 0; j < 2; ++j) {
            int nb = 0;
            size_t si = 0;
            // a forward shift attempt per non-empty neighbour bin (counted)
            bool want = live && bin_neighbor(B, p, b, j, src_grid, nb, si) && ld2(src_grid, 0, si).x > 0;
            uint32_t k = block_queue_append(ws.q, want, bd.err, sh);
            if (k != kNoJob) {
                double sc, sw;
                gate_of(gate, nb, sc, sw);
                job_put(ws.q, k, si, JOB_FULL | JOB_COUNT, px, py, px, py, sc, dc, dw);
            }
            if (live) ws.map_a[size_t(j) * n + i] = k;
        }
    }
}

__global__ void k_bin_prep_inv(Band bd, int W, PathCfg cfg, GateGrid gate, int j, ResStore src_grid,
                               ResStore dst_grid, WaveScratch ws) {
    const int B = gate.h.bins;
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t n_round = (n + blockDim.x - 1) / blockDim.x * blockDim.x;  // block-uniform trip count
    __shared__ uint32_t sh[33];
    const ResStore& out_grid = j == 0 ? src_grid : dst_grid;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n_round; i += stride) {
        bool live = i < n;
        size_t it = base + (live ? i : 0);
        size_t p = it / B;
        int b = int(it % B);
        int px = int(p % W), py = int(p / W);
        int nb = 0;
        size_t si = 0;
        bool want = false, merge = false;
        if (live) {
            if (!bin_neighbor(B, p, b, j, src_grid, nb, si)) {
                if (j == 0) {  // the output starts as the stage input
                    double2 c0 = ld2(src_grid, 0, it);
                    if (c0.x > 0)
                        copy_res(src_grid, dst_grid, it, c0.x, c0.y, false);
                    else
                        res_store_w(dst_grid, it, 0.0, c0.y);
                    ws.rng_ctr[i] = 0;
                }
            } else {
                double2 o0 = ld2(out_grid, 0, it), s0 = ld2(src_grid, 0, si);
                want = o0.x > 0;
                merge = want || s0.x > 0;
                if (!merge) {  // both empty: the merge only adds the confidences (no RNG draw)
                    res_store_w(dst_grid, it, 0.0, dmin(o0.y + s0.y, cfg.m_cap));
                    if (j == 0) ws.rng_ctr[i] = 0;
                }
            }
        }
        uint32_t k = block_append_jobs(ws, uint32_t(want), merge, uint32_t(i), bd.err, cfg.work, sh);
        if (k != kNoJob) {
            double dc, dw, sc, sw;
            gate_of(gate, b, dc, dw);
            gate_of(gate, nb, sc, sw);
            job_put(ws.q, k, it, j == 0 ? 0u : JOB_REC1, px, py, px, py, dc, sc, dw);
            ws.map_b[i] = k;
        }
    }
}

__global__ void __launch_bounds__(256, TOFR_APPLY_MINB)
    k_bin_apply(Band bd, int W, PathCfg cfg, GateGrid gate, int j, int frame_idx, ResStore src_grid,
                ResStore dst_grid, WaveScratch ws) {
    const int B = gate.h.bins;
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    uint32_t cnt = ws.q.ctl[3];
    for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < cnt; l += gridDim.x * blockDim.x) {
        size_t i = ws.mlist[l], it = base + i;
        size_t p = it / B;
        int b = int(it % B);
        int nb = 0;
        size_t si = 0;
        bin_neighbor(B, p, b, j, src_grid, nb, si);
        Res out, src;
        res_head_phat(j == 0 ? src_grid : dst_grid, it, out);
        res_head_phat(src_grid, si, src);
        double dc, dw;
        gate_of(gate, b, dc, dw);
        MergeShift ms{0, 1.0, 0.0};
        Sample mapped;
        double mgv = 0;
        uint32_t kf = src.has ? ws.map_a[size_t(j) * n + i] : kNoJob;
        fwd_output(ws.q, kf, 0, ms, mapped, mgv);
        ms.phat_src_of_dst = inv_output(ws.q, out.has ? ws.map_b[i] : kNoJob);
        Rng rng = rng_make(cfg.seed, uint64_t(frame_idx), uint64_t(p), uint64_t(b), 12);
        if (j > 0) rng.ctr = ws.rng_ctr[i];
        int which = gris_merge(out, src, ms, mapped, mgv, dc, dw, cfg.m_cap, rng);
        if (which == 2)
            put_mapped(ws.q.out, kf, dst_grid, it, out.W, out.M, out.phat, false);
        else if (which == 1 && j == 0)
            copy_res(src_grid, dst_grid, it, out.W, out.M, false);
        else  // kept in place (j > 0) or empty
            res_store_w(dst_grid, it, out.W, out.M);
        if (j == 0) ws.rng_ctr[i] = rng.ctr;
    }
}

// ---------------------------------------------------------------------------
// shrink initialiser (initial_sampling's shrink branch, pipeline.hpp:137-183):
// the rough (wide-gate) and fine RIS reservoirs come from two k_trace runs that
// share the pixel's pick stream; here the rough winner's forward shrink_map and
// the fine winner's inverse one run as shift jobs, then one merge per pixel.

__global__ void k_shrink_prep(Band bd, int W, double center, double width, int m_fine, ResStore rough,
                              ResStore fine, WaveScratch ws, unsigned long long* work) {
    size_t base = size_t(bd.y0) * W, n = size_t(bd.y1 - bd.y0) * W;
    size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t n_round = (n + blockDim.x - 1) / blockDim.x * blockDim.x;  // block-uniform trip count
    __shared__ uint32_t sh[33];
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n_round; i += stride) {
        bool live = i < n;
        size_t it = base + (live ? i : 0);
        int px = int(it % W), py = int(it / W);
        const bool fwd = live && ld2(rough, 0, it).x > 0;
        const bool inv = fwd && m_fine > 0 && ld2(fine, 0, it).x > 0;
        uint32_t k = block_append_jobs(ws, uint32_t(fwd) + uint32_t(inv), false, uint32_t(i), bd.err, work, sh);
        if (k != kNoJob) {
            job_put(ws.q, k, it, JOB_FULL | JOB_SHRINK, px, py, px, py, center, center, width);
            ws.map_a[i] = k;
            if (inv) {
                job_put(ws.q, k + 1, it, JOB_SHRINK | JOB_REC1, px, py, px, py, center, center, width);
                ws.map_b[i] = k + 1;
            }
        }
    }
}

__global__ void k_shrink_merge(Band bd, int W, PathCfg cfg, double center, double width, int m_fine, int frame_idx,
                               ResStore rough, ResStore fine, WaveScratch ws, const uint64_t* pick_ctr) {
    size_t base = size_t(bd.y0) * W, n = size_t(bd.y1 - bd.y0) * W;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        size_t it = base + i;
        Res r, out;
        res_head_phat(rough, it, r);
        if (!r.has) {  // rough empty: the fine reservoir (M = 1) is the result
            if (m_fine == 0) res_store_w(fine, it, 0.0, 1.0);
            continue;
        }
        Rng pick = rng_make(cfg.seed, uint64_t(frame_idx), uint64_t(it), 0, 9);
        pick.ctr = pick_ctr[i];
        MergeShift ms{0, 1.0, 0.0};
        Sample mapped;
        double mgv = 0;
        const uint32_t kf = ws.map_a[i];
        fwd_output(ws.q, kf, 0, ms, mapped, mgv);
        if (m_fine == 0) {  // every tree on the wide gate: one candidate, the mapped winner
            double w_sum = 0, ph = 0;
            int has = 0;
            if (ms.valid) {
                double pyv = luminance(mapped.f) * gate_w(center, width, mgv);
                double w = pyv * r.W * ms.jac;
                if (isfinite(w) && w > 0) {
                    w_sum += w;
                    if (rng_next(pick) * w_sum < w) {
                        has = 1;
                        ph = pyv;
                    }
                }
            }
            const double Wv = (has && ph > 0) ? w_sum / ph : 0;
            if (has)
                put_mapped(ws.q.out, kf, fine, it, Wv, 1.0, ph, false);
            else
                res_store_w(fine, it, Wv, 1.0);
            continue;
        }
        res_head_phat(fine, it, out);
        ms.phat_src_of_dst = inv_output(ws.q, out.has ? ws.map_b[i] : kNoJob);
        int which = gris_merge(out, r, ms, mapped, mgv, center, width, cfg.m_cap, pick);
        if (which == 2)  // the rough winner, contracted onto the fine gate
            put_mapped(ws.q.out, kf, fine, it, out.W, out.M, out.phat, false);
        else  // the fine winner kept in place, or empty
            res_store_w(fine, it, out.W, out.M);
    }
}

// ---------------------------------------------------------------------------
// queue control and launchers

// op 0: empty queue; op 1: mark the end (the next batch starts after it);
// op 2: rewind to the mark; op 3: mark the end, the current batch continues.
__global__ void k_queue_ctl(uint32_t* ctl, int op) {
    if (op == 0) {
        ctl[0] = ctl[1] = ctl[2] = 0;
    } else if (op == 1) {
        ctl[2] = ctl[1];
        ctl[0] = ctl[1];
    } else if (op == 2) {
        ctl[0] = ctl[2];
        ctl[1] = ctl[2];
    } else {
        ctl[2] = ctl[1];
    }
    ctl[3] = 0;  // merge list of the batch
}

static int grid_n(size_t n, int block) {
    size_t g = (n + block - 1) / block;
    if (g > 148 * 32) g = 148 * 32;
    if (g < 1) g = 1;
    return int(g);
}

static void run_shifts(const FrameView& F0, const FrameView& F1, const GHit* g0, const GHit* g1, ResStore st0,
                       ResStore st1, ShiftQueue q, const ShiftOverlap& ov, const PathCfg& cfg,
                       unsigned long long* ctr, unsigned long long* wq, cudaStream_t s) {
    bool same = F1.nodes == F0.nodes && F1.tri_isect == F0.tri_isect;
    size_t sm = frame_smem_bytes(F0) + (same ? 0 : frame_smem_bytes(F1));
    size_t cap_jobs = q.cap;
    if (cfg.replay) {
        cudaMemsetAsync(wq, 0, sizeof(unsigned long long), s);
        {
            KScope ks("k_shift_replay", s);
            k_shift_replay<<<persistent_grid(reinterpret_cast<const void*>(k_shift_replay), 128, sm, cap_jobs), 128, sm,
                             s>>>(F0, F1, g0, g1, st0, st1, q, cfg, wq);
        }
    }
    // length-gate and velocity-gate (Doppler) instantiations
    // velocity gates are gated-only (dense grids)
    const bool sp = st0.slot != nullptr || st1.slot != nullptr;
    auto solve = cfg.gate_vel ? k_shift_solve<true, false> : (sp ? k_shift_solve<false, true> : k_shift_solve<false, false>);
    auto finish = cfg.gate_vel ? k_shift_finish<true, false>
                               : (sp ? k_shift_finish<false, true> : k_shift_finish<false, false>);
    // Overlap (programmatic dependent launch): every solve CTA triggers the
    // finish launch once its warps find the job queue drained, so the finish
    // grid starts with the solve's tail and fills the SMs it leaves idle (its
    // CTAs start as solve CTAs retire).  The finish does not wait for the solve
    // grid: it takes each job once the solve has published that job's hand-off
    // (ShiftQueue::done, release / acquire).  Every job has been handed to a
    // resident solve warp before the finish can launch: no deadlock.
    const bool overlap = ov.fin_ctr && q.done;
    if (overlap)
        q.epoch = ++*ov.epoch;
    else
        q.done = nullptr;
    unsigned long long* fq = overlap ? ov.fin_ctr : wq;
    cudaMemsetAsync(wq, 0, sizeof(unsigned long long), s);
    if (overlap) cudaMemsetAsync(fq, 0, sizeof(unsigned long long), s);
    {
        KScope ks("k_shift_solve", s);
        solve<<<persistent_grid(reinterpret_cast<const void*>(solve), TOFR_SOLVE_BLOCK, sm, cap_jobs), TOFR_SOLVE_BLOCK,
                sm, s>>>(
            F0, F1, g0, g1, st0, st1, q, cfg, ctr, wq);
    }
    if (!overlap) cudaMemsetAsync(fq, 0, sizeof(unsigned long long), s);
    {
        KScope ks("k_shift_finish", s);
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(unsigned(persistent_grid(reinterpret_cast<const void*>(finish), 128, sm, cap_jobs)));
        lc.blockDim = dim3(128);
        lc.dynamicSmemBytes = sm;
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = overlap ? 1 : 0;
        lc.attrs = at;
        lc.numAttrs = 1;
        cudaLaunchKernelEx(&lc, finish, F0, F1, g0, g1, st0, st1, q, cfg, ctr, fq);
    }
}

// an out-of-range item of a 4-item dense grid: traps in a TOFR_CHECK build
// (res_row of a dense grid touches no memory, so the product build just
// returns the index)
__global__ void k_check_selftest(ResStore st, unsigned long long* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = res_row(st, 5);
}
int launch_check_selftest(unsigned long long* out, cudaStream_t s) {
    ResStore st{nullptr, 4};
    st.ilo = 0;
    st.ihi = 4;
    k_check_selftest<<<1, 32, 0, s>>>(st, out);
    return TOFR_CHECK;
}

// solve profile of a TOFR_SOLVE_PROFILE build: copies min(n, cap) records
// (3 u64 each) and resets; returns false when the build has no profiler
bool debug_solve_profile(unsigned long long* out, size_t cap, size_t* n) {
#if TOFR_SOLVE_PROFILE
    unsigned cnt = 0;
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(&cnt, g_solve_prof_n, sizeof(cnt));
    size_t m = cnt < kSolveProfCap ? cnt : kSolveProfCap;
    if (m > cap) m = cap;
    if (out && m) cudaMemcpyFromSymbol(out, g_solve_prof, m * 3 * sizeof(unsigned long long));
    *n = m;
    unsigned zero = 0;
    cudaMemcpyToSymbol(g_solve_prof_n, &zero, sizeof(zero));
    return true;
#else
    (void)out;
    (void)cap;
    *n = 0;
    return false;
#endif
}

// ---------------------------------------------------------------------------
// Adaptive row batches (transient grids): an upper bound of the shift jobs each
// image row of a stage will queue, so the host cuts the band into as few row
// batches as the queue holds (the worst-case sizing, jobs-per-item x items,
// assumes every reservoir non-empty: 8 batches for 1080p x 64 bins where the
// grids are ~40% full).  Counts are summed per warp for each row.

__device__ __forceinline__ void row_count_add(unsigned long long* rows, int row, unsigned v) {
    const unsigned grp = __match_any_sync(0xffffffffu, row);
    const unsigned sum = __reduce_add_sync(grp, v);
    if ((threadIdx.x & 31) == __ffs(grp) - 1 && sum) atomicAdd(&rows[row], (unsigned long long)sum);
}

// temporal (k_temporal_prep): forward job if the reprojected source is
// non-empty, inverse job if the destination is, both only when the source has M > 0
__global__ void k_count_temporal(Band bd, int W, GateGrid cg, ResStore cur, ResStore prev, const uint64_t* tsrc,
                                 unsigned long long* rows) {
    int B = cg.transient ? cg.h.bins : 1;
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    size_t n_round = (n + 31) / 32 * 32;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n_round; i += size_t(gridDim.x) * blockDim.x) {
        bool live = i < n;
        size_t it = base + (live ? i : 0);
        int p = int(it / B), b = int(it % B);
        unsigned jobs = 0;
        if (live) {
            uint64_t src_pix = tsrc[size_t(p) - size_t(bd.y0) * W];
            if (src_pix != ~uint64_t(0)) {
                double2 s0 = ld2(prev, 0, size_t(src_pix) * B + b);
                if (s0.y > 0) jobs = unsigned(s0.x > 0) + unsigned(ld2(cur, 0, it).x > 0);
            }
        }
        row_count_add(rows, p / W - bd.y0, jobs);
    }
}

// spatial pass (k_spatial_prep_fwd / _inv): the forward jobs of every non-empty
// neighbour, plus at most one inverse job per item at a time (an inverse batch
// replaces the previous one), only when the item or a neighbour is non-empty
__global__ void k_count_spatial(Band bd, int W, int H, GateGrid gate, PathCfg cfg, SpatialParams sp, int pass,
                                int frame_idx, ResStore src_grid, unsigned long long* rows) {
    int B = gate.transient ? gate.h.bins : 1;
    size_t base = size_t(bd.y0) * W * B, n = size_t(bd.y1 - bd.y0) * W * B;
    size_t n_round = (n + 31) / 32 * 32;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n_round; i += size_t(gridDim.x) * blockDim.x) {
        bool live = i < n;
        size_t it = base + (live ? i : 0);
        int p = int(it / B), b = int(it % B);
        int px = p % W, py = p / W;
        unsigned fwd = 0;
        bool self = false;
        if (live) {
            uint64_t rk = spatial_rot_key(uint64_t(p), pass, cfg.seed, frame_idx);
            for (int j = 0; j < sp.neighbors; ++j) {
                int nx, ny;
                size_t si;
                if (spatial_neighbor(bd, W, H, B, px, py, b, sp, rk, j, src_grid, nx, ny, si) &&
                    ld2(src_grid, 0, si).x > 0)
                    ++fwd;
            }
            self = ld2(src_grid, 0, it).x > 0;
        }
        row_count_add(rows, p / W - bd.y0, fwd + unsigned(self || fwd > 0));
    }
}

void launch_count_temporal(const FrameView& Fc, const Band& bd, const GHit* gc, const FrameView& Fp,
                           const GateGrid& cg, ResStore cur, ResStore prev, const WaveScratch& ws,
                           unsigned long long* rows, cudaStream_t s) {
    size_t npx = size_t(bd.y1 - bd.y0) * Fc.cam.w, n = npx * (cg.transient ? cg.h.bins : 1);
    if (!n) return;
    cudaMemsetAsync(rows, 0, size_t(bd.y1 - bd.y0) * sizeof(unsigned long long), s);
    {
        KScope ks("k_temporal_reproject", s);
        k_temporal_reproject<<<grid_n(npx, 256), 256, 0, s>>>(Fc, bd, gc, Fp, ws);
    }
    KScope ks("k_count_temporal", s);
    k_count_temporal<<<grid_n(n, 256), 256, 0, s>>>(bd, Fc.cam.w, cg, cur, prev, ws.tsrc, rows);
}

void launch_count_spatial(const FrameView& F, const Band& bd, const PathCfg& cfg, const GateGrid& gg,
                          const SpatialParams& sp, int pass, int frame_idx, ResStore src, unsigned long long* rows,
                          cudaStream_t s) {
    size_t n = size_t(bd.y1 - bd.y0) * F.cam.w * (gg.transient ? gg.h.bins : 1);
    if (!n) return;
    cudaMemsetAsync(rows, 0, size_t(bd.y1 - bd.y0) * sizeof(unsigned long long), s);
    KScope ks("k_count_spatial", s);
    k_count_spatial<<<grid_n(n, 256), 256, 0, s>>>(bd, F.cam.w, F.cam.h, gg, cfg, sp, pass, frame_idx, src, rows);
}

void launch_temporal_wave(const FrameView& Fc, const Band& bd, const GHit* gc, const FrameView& Fp, const GHit* gp,
                          const PathCfg& cfg, const GateGrid& cg, const GateGrid& pg, int frame_idx, ResStore cur,
                          ResStore prev, const WaveScratch& ws, unsigned long long* ctr, unsigned long long* q,
                          cudaStream_t s) {
    size_t n = size_t(bd.y1 - bd.y0) * Fc.cam.w * (cg.transient ? cg.h.bins : 1);
    if (!n) return;
    {
        KScope ks("k_queue_ctl", s);
        k_queue_ctl<<<1, 1, 0, s>>>(ws.q.ctl, 0);
    }
    {
        KScope ks("k_temporal_reproject", s);
        size_t npx = size_t(bd.y1 - bd.y0) * Fc.cam.w;
        k_temporal_reproject<<<grid_n(npx, 256), 256, 0, s>>>(Fc, bd, gc, Fp, ws);
    }
    {
        KScope ks("k_temporal_prep", s);
        if (n >= kPrepItemsMin)
            k_temporal_prep<TOFR_PREP_ITEMS><<<grid_n((n + TOFR_PREP_ITEMS - 1) / TOFR_PREP_ITEMS, 256), 256, 0, s>>>(
                Fc, bd, gc, Fp, cg, pg, cfg, cur, prev, ws);
        else
            k_temporal_prep<1><<<grid_n(n, 256), 256, 0, s>>>(Fc, bd, gc, Fp, cg, pg, cfg, cur, prev, ws);
    }
    run_shifts(Fc, Fp, gc, gp, cur, prev, ws.q, ws.ov, cfg, ctr, q, s);
    {
        KScope ks("k_temporal_apply", s);
        k_temporal_apply<<<grid_n(n, 256), 256, 0, s>>>(bd, Fc.cam.w, cg, cfg, frame_idx, cur, prev, ws);
    }
}

void launch_spatial_wave(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, const GateGrid& gg,
                         const SpatialParams& sp, int pass, int frame_idx, ResStore src, ResStore dst,
                         const WaveScratch& ws, unsigned long long* ctr, unsigned long long* q, cudaStream_t s) {
    size_t n = size_t(bd.y1 - bd.y0) * F.cam.w * (gg.transient ? gg.h.bins : 1);
    if (!n) return;
    {
        KScope ks("k_queue_ctl", s);
        k_queue_ctl<<<1, 1, 0, s>>>(ws.q.ctl, 0);
    }
    // The forward shifts of every neighbour and the inverse shifts of neighbour 0
    // (from the pass input) are independent: one shift batch.  Inverse shifts
    // of neighbour j > 0 need merge j - 1 and replace the previous inverse batch.
    {
        KScope ks("k_spatial_offsets", s);
        size_t npx = size_t(bd.y1 - bd.y0) * F.cam.w;
        k_spatial_offsets<<<grid_n(npx, 256), 256, 0, s>>>(bd, F.cam.w, cfg, sp, pass, frame_idx, ws);
    }
    {
        KScope ks("k_spatial_prep_fwd", s);
        if (n >= kPrepItemsMin)
            k_spatial_prep_fwd<TOFR_PREP_ITEMS><<<grid_n((n + TOFR_PREP_ITEMS - 1) / TOFR_PREP_ITEMS, 256), 256, 0, s>>>(
                F, bd, cfg, gg, sp, pass, frame_idx, src, ws);
        else
            k_spatial_prep_fwd<1><<<grid_n(n, 256), 256, 0, s>>>(F, bd, cfg, gg, sp, pass, frame_idx, src, ws);
    }
    {
        KScope ks("k_queue_ctl", s);
        k_queue_ctl<<<1, 1, 0, s>>>(ws.q.ctl, 3);
    }
    for (int j = 0; j < sp.neighbors; ++j) {
        if (j > 0) {
            KScope ks("k_queue_ctl", s);
            k_queue_ctl<<<1, 1, 0, s>>>(ws.q.ctl, 2);
        }
        {
            KScope ks("k_spatial_prep_inv", s);
            if (n >= kPrepItemsMin)
                k_spatial_prep_inv<TOFR_PREP_ITEMS><<<grid_n((n + TOFR_PREP_ITEMS - 1) / TOFR_PREP_ITEMS, 256), 256, 0,
                                                      s>>>(F, bd, cfg, gg, sp, pass, j, frame_idx, src, dst, ws);
            else
                k_spatial_prep_inv<1><<<grid_n(n, 256), 256, 0, s>>>(F, bd, cfg, gg, sp, pass, j, frame_idx, src, dst, ws);
        }
        run_shifts(F, F, g, g, src, dst, ws.q, ws.ov, cfg, ctr, q, s);
        {
            KScope ks("k_spatial_apply", s);
            k_spatial_apply<<<grid_n(n, 256), 256, 0, s>>>(F, bd, cfg, gg, sp, pass, j, frame_idx, src, dst, ws);
        }
    }
}

void launch_binreuse_wave(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, const GateGrid& gg,
                          int frame_idx, ResStore src, ResStore dst, const WaveScratch& ws, unsigned long long* ctr,
                          unsigned long long* q, cudaStream_t s) {
    const int W = F.cam.w;
    size_t n = size_t(bd.y1 - bd.y0) * W * gg.h.bins;
    if (!n) return;
    {
        KScope ks("k_queue_ctl", s);
        k_queue_ctl<<<1, 1, 0, s>>>(ws.q.ctl, 0);
    }
    {
        KScope ks("k_bin_prep_fwd", s);
        k_bin_prep_fwd<<<grid_n(n, 256), 256, 0, s>>>(bd, W, gg, src, ws);
    }
    {
        KScope ks("k_queue_ctl", s);
        k_queue_ctl<<<1, 1, 0, s>>>(ws.q.ctl, 3);
    }
    for (int j = 0; j < 2; ++j) {
        if (j > 0) {
            KScope ks("k_queue_ctl", s);
            k_queue_ctl<<<1, 1, 0, s>>>(ws.q.ctl, 2);
        }
        {
            KScope ks("k_bin_prep_inv", s);
            k_bin_prep_inv<<<grid_n(n, 256), 256, 0, s>>>(bd, W, cfg, gg, j, src, dst, ws);
        }
        run_shifts(F, F, g, g, src, dst, ws.q, ws.ov, cfg, ctr, q, s);
        {
            KScope ks("k_bin_apply", s);
            k_bin_apply<<<grid_n(n, 256), 256, 0, s>>>(bd, W, cfg, gg, j, frame_idx, src, dst, ws);
        }
    }
}

void launch_shrink_wave(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, double center,
                        double width, int m_fine, int frame_idx, ResStore rough, ResStore fine,
                        const uint64_t* pick_ctr, const WaveScratch& ws, unsigned long long* ctr,
                        unsigned long long* q, cudaStream_t s) {
    const int W = F.cam.w;
    size_t n = size_t(bd.y1 - bd.y0) * W;
    if (!n) return;
    {
        KScope ks("k_queue_ctl", s);
        k_queue_ctl<<<1, 1, 0, s>>>(ws.q.ctl, 0);
    }
    {
        KScope ks("k_shrink_prep", s);
        k_shrink_prep<<<grid_n(n, 256), 256, 0, s>>>(bd, W, center, width, m_fine, rough, fine, ws, nullptr);
    }
    run_shifts(F, F, g, g, rough, fine, ws.q, ws.ov, cfg, ctr, q, s);
    {
        KScope ks("k_shrink_merge", s);
        k_shrink_merge<<<grid_n(n, 256), 256, 0, s>>>(bd, W, cfg, center, width, m_fine, frame_idx, rough, fine, ws,
                                                       pick_ctr);
    }
}

}  // namespace tofr_b200
