// tofr_store.cuh -- reservoir grids in HBM.
//
// A reservoir is 24 x 16 B chunks (384 B).  Grids are chunk-major: chunk c of
// item i lives at base[c * stride + i], so when a warp touches 32 consecutive
// items every 128-bit load/store instruction moves 512 contiguous bytes
// (fully coalesced).  Readers that only need the header (confidence M,
// emptiness) touch chunks 0 and 4 only; the replay lanes (chunks 20-21) are
// read only when a record has k > 2.
//
//   0: W, M                     8: p1.y, p1.z         16: n2.z, wo2.x
//   1: phat, len                9: wi1.x, wi1.y       17: wo2.y, wo2.z
//   2: f.x, f.y                10: wi1.z, p.x         18: suffix_f.x, .y
//   3: f.z, suffix_len         11: p.y, p.z           19: suffix_f.z, {m2, -}
//   4: {has,valid,k,nl,skind,depth,-,-}, tri1, ptri     19.y: {m2, obj2}
//   5: prefix_pdf, prefix_len  12: pn.x, pn.y         20: lane_key, ctr[0..3]
//   6: prefix_fw.x, .y         13: pn.z, p2.x         21: ctr[4..9], -
//                                                     22: u, prefix_u
//                                                     23: suffix_u, -
//   7: prefix_fw.z, p1.x       14: p2.y, p2.z
//                              15: n2.x, n2.y
#pragma once

#include <cstdio>

#include "tofr_path.cuh"

namespace tofr_b200 {

constexpr int kResChunks = 24;

// Dense store (gated grids, scratch planes): chunk c of item i at
// base[c * stride + i].
//
// Sparse store (transient grids, TOFR_SPARSE): the header plane (chunk 0:
// W, M) stays dense, base[i], but chunks 1..23 live in a pool of rows that
// only non-empty reservoirs occupy: chunk c of item i at
// pool[c * stride + slot[i]] (stride = pool rows + 2).  A W x H x B transient
// grid is mostly empty reservoirs (92% at C2), so the pool is a fraction of the
// dense grid.  A reservoir gets its row the first time a sample chunk is
// written to it (one atomic on the grid's row counter) and keeps it until the
// grid is recycled for another frame or pass (slot map reset to kNoSlot,
// counter to 0: reset_sparse_store).  Rows stride-1 (all zero: what an
// empty reservoir reads) and stride-2 (where writes go once the pool is full;
// raises kErrPool in the band error word) are never handed out.  One thread
// writes a given item of a grid at a time (every writer owns its items), so a
// row is allocated once.
constexpr uint32_t kNoSlot = 0xffffffffu;
constexpr unsigned long long kErrPool = 1ull << 62;
constexpr unsigned long long kErrHalo = 1ull << 61;  // compacted halo: more non-empty rows than its capacity

struct ResStore {
    double2* base;
    size_t stride;                       // dense: items per chunk plane; sparse: pool rows + 2
    uint32_t* slot = nullptr;            // sparse: item -> pool row (global item index)
    double2* pool = nullptr;             // sparse: chunk planes 1..23 (pool[c * stride + row])
    unsigned int* rows = nullptr;        // sparse: rows handed out
    unsigned long long* err = nullptr;   // sparse: band error word (kErrPool on overflow)
    // chunk planes held (header included): a sparse pool drops the replay-lane
    // and velocity chunks (20-23) when no record can have them (no
    // non-reconnectable material, length gates): 20
    int planes = kResChunks;
    // Compact pool rows (sparse, no replay lanes): every record then has its
    // reconnection vertex at k = 2, so its identity-prefix cache -- chunks 5-9
    // (prefix pdf / length / throughput, p1, wi1) -- is a function of its own
    // pixel's primary hit in the grid's frame (the G-buffer hit and camera:
    // pdf 1, length t, throughput 1, p1 = cam + d0 t, wi1 = -d0, exactly the
    // values the trace and the shift write).  Those planes are not stored
    // (304 -> 224 B per row, SURVEY 8d's record size); readers rebuild them.
    int compact = 0;
    const GHit* gbuf = nullptr;  // the grid's frame: G-buffer (global pixel index) and camera
    GCam cam{};
    int bins = 1;
    // a record pinned by res_pin: its pool row, looked up once (the slot map
    // is read with ld.global.cg, a volatile asm the compiler cannot merge, so
    // every chunk access would otherwise re-read it before its own load)
    size_t pin_item = ~size_t(0), pin_row = 0;
    // global item range the grid holds (checked only in a -DTOFR_CHECK=1 build)
    size_t ilo = 0, ihi = ~size_t(0);
};

#if defined(__CUDACC__)

// Checked build (-DTOFR_CHECK=1, the `check` library variant): every grid,
// pool-row and job-queue index is bounds-checked on the device; a failed check
// prints its site and traps (the launch fails, the host call returns an error).
#ifndef TOFR_CHECK
#define TOFR_CHECK 0
#endif
#if TOFR_CHECK
#define TOFR_CHK(cond)                                                                        \
    do {                                                                                     \
        if (!(cond)) {                                                                       \
            printf("TOFR_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
                   int(blockIdx.x), int(threadIdx.x));                                       \
            __trap();                                                                        \
        }                                                                                    \
    } while (0)
#else
#define TOFR_CHK(cond) ((void)0)
#endif

// pool row of item i for reading chunks >= 1 (the zero row when it has none)
__device__ __forceinline__ size_t res_row(const ResStore& s, size_t i) {
    TOFR_CHK(i >= s.ilo && i < s.ihi);
    if (s.slot == nullptr) return i;
    if (i == s.pin_item) return s.pin_row;
    uint32_t r = __ldcg(&s.slot[i]);
    TOFR_CHK(r == kNoSlot || size_t(r) < s.stride - 2);
    return r == kNoSlot ? s.stride - 1 : size_t(r);
}
// pool row of item i for writing chunks >= 1 (allocated on first use)
__device__ __forceinline__ size_t res_row_w(const ResStore& s, size_t i) {
    TOFR_CHK(i >= s.ilo && i < s.ihi);
    if (s.slot == nullptr) return i;
    uint32_t r = __ldcg(&s.slot[i]);
    if (r == kNoSlot) {
        r = atomicAdd(s.rows, 1u);
        if (size_t(r) >= s.stride - 2) {
            atomicOr(s.err, kErrPool);
            return s.stride - 2;
        }
        __stcg(&s.slot[i], r);
    }
    return r;
}
__device__ __forceinline__ double2* res_planes(const ResStore& s) { return s.slot ? s.pool : s.base; }
// a copy of s with item i's row looked up once, for a kernel that reads (never
// writes) several chunks of that record
__device__ __forceinline__ ResStore res_pin(const ResStore& s, size_t i) {
    ResStore v = s;
    v.pin_row = res_row(s, i);
    v.pin_item = i;
    return v;
}

// chunk c >= 1 at a known row (compact rows: chunks 5-9 are not stored -- they
// read as zero, writes are dropped -- and chunks >= 10 sit 5 planes lower)
__device__ __forceinline__ bool res_derived_chunk(const ResStore& s, int c) { return s.compact && c >= 5 && c <= 9; }
__device__ __forceinline__ int res_plane(const ResStore& s, int c) { return (s.compact && c >= 10) ? c - 5 : c; }
__device__ __forceinline__ void res_chk_row(const ResStore& s, int c, size_t row) {
    TOFR_CHK(c >= 0 && res_plane(s, c) < (s.slot ? s.planes - (s.compact ? 5 : 0) : kResChunks));
    TOFR_CHK(s.slot ? row < s.stride : (row >= s.ilo && row < s.ihi));
    (void)s, (void)c, (void)row;
}
__device__ __forceinline__ double2 ld2r(const ResStore& s, int c, size_t row) {
    res_chk_row(s, c, row);
    if (res_derived_chunk(s, c)) return make_double2(0.0, 0.0);
    return __ldcg(&res_planes(s)[size_t(res_plane(s, c)) * s.stride + row]);
}
__device__ __forceinline__ void st2r(const ResStore& s, int c, size_t row, double2 v) {
    res_chk_row(s, c, row);
    if (res_derived_chunk(s, c)) return;
    __stcg(&res_planes(s)[size_t(res_plane(s, c)) * s.stride + row], v);
}

// identity-prefix cache of the record of item i, rebuilt for a compact row
// (see ResStore::compact): prefix pdf, length, throughput, p1, wi1
struct PrefixCache {
    double pdf, len;
    V3 fw, p1, wi1;
};
__device__ __forceinline__ PrefixCache res_prefix_derived(const ResStore& s, size_t i) {
    const size_t p = i / size_t(s.bins);
    const int px = int(p % size_t(s.cam.w)), py = int(p / size_t(s.cam.w));
    const GHit g = s.gbuf[p];
    const V3 d0 = primary_dir(s.cam, px, py);
    PrefixCache c;
    c.pdf = 1;
    c.len = g.t;
    c.fw = splat(1);
    c.p1 = s.cam.pos + d0 * g.t;
    c.wi1 = -d0;
    return c;
}

__device__ __forceinline__ double2 ld2(const ResStore& s, int c, size_t i) {
    TOFR_CHK(i >= s.ilo && i < s.ihi);
    if (c == 0) return __ldcg(&s.base[i]);
    return ld2r(s, c, res_row(s, i));
}
__device__ __forceinline__ void st2(const ResStore& s, int c, size_t i, double a, double b) {
    TOFR_CHK(i >= s.ilo && i < s.ihi);
    if (c == 0)
        __stcg(&s.base[i], make_double2(a, b));
    else
        st2r(s, c, res_row_w(s, i), make_double2(a, b));
}

struct Meta {
    unsigned char has, valid, k, nl, skind, depth, pad0, pad1;
    int tri1, ptri;
};

__device__ __forceinline__ Meta ld_meta_r(const ResStore& s, size_t row) {
    double2 v = ld2r(s, 4, row);
    Meta m;
    memcpy(&m, &v, 16);
    return m;
}
__device__ __forceinline__ Meta ld_meta(const ResStore& s, size_t i) {
    double2 v = ld2(s, 4, i);
    Meta m;
    static_assert(sizeof(Meta) == 16, "meta chunk");
    memcpy(&m, &v, 16);
    return m;
}

// Emptiness lives in chunk 0 alone: a reservoir holds a sample iff W > 0.
// (has <=> W > 0: ris_finalize and gris_merge set W = w_sum / phat > 0 exactly
// when a candidate was selected, and W = 0 otherwise, ris.hpp:52-56, :101-103.)
// Readers therefore touch chunk 0 first and the sample chunks only for
// non-empty reservoirs, and writers of an empty result store chunk 0 only --
// the sample chunks of an empty reservoir are never read.
__device__ __forceinline__ void res_load_hdr(const ResStore& s, size_t i, double& W, double& M, int& has) {
    double2 c0 = ld2(s, 0, i);
    W = c0.x;
    M = c0.y;
    has = W > 0;
}

// chunk 0 only (W, M, has); the sample is not loaded
__device__ __forceinline__ void res_load_head(const ResStore& s, size_t i, Res& r) {
    double2 c0 = ld2(s, 0, i);
    r.W = c0.x;
    r.M = c0.y;
    r.has = r.W > 0;
    r.phat = 0;
}

// chunks 1-3: phat, len, f, suffix_len (what a merge reads of a candidate)
__device__ __forceinline__ void res_load_value(const ResStore& s, size_t i, Res& r) {
    double2 c;
    const size_t row = res_row(s, i);
    c = ld2r(s, 1, row);
    r.phat = c.x;
    r.y.len = c.y;
    c = ld2r(s, 2, row);
    r.y.f.x = c.x;
    r.y.f.y = c.y;
    c = ld2r(s, 3, row);
    r.y.f.z = c.x;
    r.y.rec.suffix_len = c.y;
}

// chunks 4-21: the reconnection record (+ depth)
// `vel`: also the path-velocity terms (chunks 22-23; Doppler gates only)
__device__ inline void res_load_rec(const ResStore& s, size_t i, Sample& y, bool vel = false) {
    double2 c;
    Rec& q = y.rec;
    const size_t row = res_row(s, i);
    Meta m = ld_meta_r(s, row);
    q.valid = m.valid;
    q.k = m.k == 255 ? -1 : int(m.k);
    q.n_lanes = m.nl;
    q.skind = m.skind;
    y.depth = m.depth;
    q.tri1 = m.tri1;
    q.ptri = m.ptri;
    c = ld2r(s, 5, row);
    q.prefix_pdf = c.x;
    q.prefix_len = c.y;
    c = ld2r(s, 6, row);
    q.prefix_fw.x = c.x;
    q.prefix_fw.y = c.y;
    c = ld2r(s, 7, row);
    q.prefix_fw.z = c.x;
    q.p1.x = c.y;
    c = ld2r(s, 8, row);
    q.p1.y = c.x;
    q.p1.z = c.y;
    c = ld2r(s, 9, row);
    q.wi1.x = c.x;
    q.wi1.y = c.y;
    c = ld2r(s, 10, row);
    q.wi1.z = c.x;
    q.p.x = c.y;
    c = ld2r(s, 11, row);
    q.p.y = c.x;
    q.p.z = c.y;
    c = ld2r(s, 12, row);
    q.pn.x = c.x;
    q.pn.y = c.y;
    c = ld2r(s, 13, row);
    q.pn.z = c.x;
    q.p2.x = c.y;
    c = ld2r(s, 14, row);
    q.p2.y = c.x;
    q.p2.z = c.y;
    c = ld2r(s, 15, row);
    q.n2.x = c.x;
    q.n2.y = c.y;
    c = ld2r(s, 16, row);
    q.n2.z = c.x;
    q.wo2.x = c.y;
    c = ld2r(s, 17, row);
    q.wo2.y = c.x;
    q.wo2.z = c.y;
    c = ld2r(s, 18, row);
    q.suffix_f.x = c.x;
    q.suffix_f.y = c.y;
    c = ld2r(s, 19, row);
    q.suffix_f.z = c.x;
    {
        int2 mi;
        memcpy(&mi, &c.y, 8);
        q.m2 = mi.x;
        q.obj2 = mi.y;
    }
    if (s.compact) {
        const PrefixCache pc = res_prefix_derived(s, i);
        q.prefix_pdf = pc.pdf;
        q.prefix_len = pc.len;
        q.prefix_fw = pc.fw;
        q.p1 = pc.p1;
        q.wi1 = pc.wi1;
    }
    if (vel) {
        c = ld2r(s, 22, row);
        y.u = c.x;
        q.prefix_u = c.y;
        q.suffix_u = ld2r(s, 23, row).x;
    } else {
        y.u = 0;
        q.prefix_u = q.suffix_u = 0;
    }
    if (q.n_lanes > 0) {
        c = ld2r(s, 20, row);
        memcpy(&q.lane_key, &c.x, 8);
        memcpy(&q.lane_ctr[0], &c.y, 8);
        c = ld2r(s, 21, row);
        memcpy(&q.lane_ctr[4], &c, 12);
    } else {
        q.lane_key = 0;
        for (int j = 0; j < kMaxLanes; ++j) q.lane_ctr[j] = 0;
    }
}

// Header first; the sample only when the reservoir is non-empty.
__device__ __forceinline__ void res_load(const ResStore& s, size_t i, Res& r) {
    res_load_head(s, i, r);
    if (r.has) {
        res_load_value(s, i, r);
        res_load_rec(s, i, r.y);
    }
}

// Every chunk, whatever the header says (scratch planes).
__device__ __forceinline__ void res_load_all(const ResStore& s, size_t i, Res& r) {
    res_load_head(s, i, r);
    res_load_value(s, i, r);
    res_load_rec(s, i, r.y);
}

__device__ __forceinline__ void st_meta_r(const ResStore& s, size_t row, const Res& r) {
    Meta m;
    const Rec& q = r.y.rec;
    m.has = (unsigned char)(r.has ? 1 : 0);
    m.valid = (unsigned char)q.valid;
    m.k = q.k < 0 ? 255 : (unsigned char)q.k;
    m.nl = (unsigned char)q.n_lanes;
    m.skind = (unsigned char)q.skind;
    m.depth = (unsigned char)r.y.depth;
    m.pad0 = m.pad1 = 0;
    m.tri1 = q.tri1;
    m.ptri = q.ptri;
    double2 v;
    memcpy(&v, &m, 16);
    st2r(s, 4, row, v);
}
__device__ __forceinline__ void st_meta(const ResStore& s, size_t i, const Res& r) { st_meta_r(s, res_row_w(s, i), r); }

__device__ inline void res_store(const ResStore& s, size_t i, const Res& r, bool vel = false) {
    const Rec& q = r.y.rec;
    st2(s, 0, i, r.W, r.M);
    const size_t row = res_row_w(s, i);
    st2r(s, 1, row, make_double2(r.phat, r.y.len));
    st2r(s, 2, row, make_double2(r.y.f.x, r.y.f.y));
    st2r(s, 3, row, make_double2(r.y.f.z, q.suffix_len));
    st_meta_r(s, row, r);
    st2r(s, 5, row, make_double2(q.prefix_pdf, q.prefix_len));
    st2r(s, 6, row, make_double2(q.prefix_fw.x, q.prefix_fw.y));
    st2r(s, 7, row, make_double2(q.prefix_fw.z, q.p1.x));
    st2r(s, 8, row, make_double2(q.p1.y, q.p1.z));
    st2r(s, 9, row, make_double2(q.wi1.x, q.wi1.y));
    st2r(s, 10, row, make_double2(q.wi1.z, q.p.x));
    st2r(s, 11, row, make_double2(q.p.y, q.p.z));
    st2r(s, 12, row, make_double2(q.pn.x, q.pn.y));
    st2r(s, 13, row, make_double2(q.pn.z, q.p2.x));
    st2r(s, 14, row, make_double2(q.p2.y, q.p2.z));
    st2r(s, 15, row, make_double2(q.n2.x, q.n2.y));
    st2r(s, 16, row, make_double2(q.n2.z, q.wo2.x));
    st2r(s, 17, row, make_double2(q.wo2.y, q.wo2.z));
    st2r(s, 18, row, make_double2(q.suffix_f.x, q.suffix_f.y));
    double m2d;
    int2 mi = make_int2(q.m2, q.obj2);
    memcpy(&m2d, &mi, 8);
    st2r(s, 19, row, make_double2(q.suffix_f.z, m2d));
    if (vel) {
        st2r(s, 22, row, make_double2(r.y.u, q.prefix_u));
        st2r(s, 23, row, make_double2(q.suffix_u, 0.0));
    }
    if (q.n_lanes > 0) {
        double a, b;
        memcpy(&a, &q.lane_key, 8);
        memcpy(&b, &q.lane_ctr[0], 8);
        st2r(s, 20, row, make_double2(a, b));
        double2 t = make_double2(0, 0);
        memcpy(&t, &q.lane_ctr[4], 12);
        st2r(s, 21, row, t);
    }
}

// Chunk-0 write: an empty reservoir (W = 0), or a reservoir whose sample and
// p-hat are already in place and only W and M changed.
__device__ __forceinline__ void res_store_w(const ResStore& s, size_t i, double W, double M) { st2(s, 0, i, W, M); }

// Store of a merge/RIS result: the full record when it is non-empty, else the
// header.
__device__ __forceinline__ void res_store_result(const ResStore& s, size_t i, const Res& r) {
    if (r.W > 0)
        res_store(s, i, r);
    else
        res_store_w(s, i, 0.0, r.M);
}

#endif  // __CUDACC__

}  // namespace tofr_b200
