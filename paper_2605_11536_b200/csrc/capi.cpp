// capi.cpp -- host runtime behind include/tofr_gpu.h: contexts, scenes,
// frame upload, the per-frame stage sequence of render_gated /
// render_transient / render_transient_plain, and the parity probes.
//
// Frame loop (pipeline.hpp:323-392, 396-528), per frame f:
//   host : build_frame(def, frame0 + f)  -> SAH BVH, camera, beam   (µs for
//          the bundled scenes) -> one packed blob -> one H2D copy
//   GPU  : k_gbuffer -> k_init_* -> [k_temporal] -> [k_binreuse] ->
//          k_spatial x P -> k_shade_*   (one stream, no host sync inside)
// Reservoir grids rotate between three device buffers (cur / prev / spare);
// the spatial snapshot of the reference (a full copy, pipeline.hpp:363) is a
// pointer swap here.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tofr_gpu.h"
#include "bvh_build.h"
#include "halo_transport.h"
#include "host_scene.h"
#include "ktime.h"
#include "tofr_kernels.h"

using namespace tofr_b200;

namespace {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ScopeError : std::runtime_error {
    int code;
    ScopeError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (e == cudaErrorMemoryAllocation)
            throw ScopeError(TOFR_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
    }
}

struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void ensure(size_t bytes) {
        if (bytes <= n) return;
        release();
        ck(cudaMalloc(&p, bytes), "cudaMalloc");
        n = bytes;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// 32-point Gauss-Legendre rule, built the way ellipsoid.hpp:88-121 does
// (Newton on P_32 from the Chebyshev-like guess) so nodes are bit-identical.
void gauss_rule32(double* x, double* w) {
    constexpr int n = 32;
    for (int i = 0; i < n / 2; ++i) {
        double t = std::cos(kPi * (i + 0.75) / (n + 0.5));
        double p0 = 0, p1 = 0;
        for (int it = 0; it < 100; ++it) {
            p0 = 1.0;
            p1 = 0.0;
            for (int j = 0; j < n; ++j) {
                double p2 = p1;
                p1 = p0;
                p0 = ((2.0 * j + 1.0) * t * p1 - j * p2) / (j + 1);
            }
            double dp = n * (t * p0 - p1) / (t * t - 1.0);
            double dt = p0 / dp;
            t -= dt;
            if (std::abs(dt) < 1e-15) break;
        }
        p0 = 1.0;
        p1 = 0.0;
        for (int j = 0; j < n; ++j) {
            double p2 = p1;
            p1 = p0;
            p0 = ((2.0 * j + 1.0) * t * p1 - j * p2) / (j + 1);
        }
        double dp = n * (t * p0 - p1) / (t * t - 1.0);
        x[i] = -t;
        x[n - 1 - i] = t;
        w[i] = w[n - 1 - i] = 2.0 / ((1.0 - t * t) * dp * dp);
    }
}

void set_err(char* err, size_t errlen, const std::string& m) {
    if (err && errlen) {
        std::snprintf(err, errlen, "%s", m.c_str());
    }
}

}  // namespace

struct tofr_gpu {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    // sessions keep their context alive: tofr_gpu_destroy with live sessions
    // only marks it, the last session destructor releases it (garbage
    // collectors finalise handles in arbitrary order)
    int live_sessions = 0;
    bool closing = false;
    const void* l2_owner = nullptr;  // session holding the stream's persisting L2 window
};

namespace {
void release_ctx(tofr_gpu* ctx) {
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}
}  // namespace

struct tofr_scene {
    HScene s;
};

// pinned host staging buffer (frame snapshot uploads)
struct PinnedBuf {
    void* p = nullptr;
    size_t n = 0;
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
    void ensure(size_t bytes) {
        if (bytes <= n) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
        ck(cudaMallocHost(&p, bytes), "cudaMallocHost");
        n = bytes;
    }
};

// one uploaded frame snapshot
struct FrameSlot {
    DevBuf blob;
    PinnedBuf staging;
    PackedFrame pk;
    FrameView view;
    DevBuf gbuf;  // rows [r0, r1)
    bool cached = false;  // static scene: blob holds the (frame-invariant) snapshot
};

struct tofr_session {
    tofr_gpu* ctx = nullptr;
    HScene scene;
    tofr_render_config cfg;
    int W = 0, H = 0, B = 1;
    bool transient = false, plain = false;
    // row band: compute rows [y0, y1), store rows [r0, r1)
    int y0 = 0, y1 = 0, r0 = 0, r1 = 0;
    bool cam_moves = false;
    bool static_frames = false;  // frame-invariant snapshot: built and uploaded once per slot
    // the frame's BVH built on the device (large animated meshes; wide light)
    bool device_bvh = false;
    std::unique_ptr<DeviceBvh> dbvh;
    FrameSlot slot[3];
    DevBuf res[4];
    int cur = 0, prev = 1, spare = 2;
    // three-deep frame pipeline (gated sessions, see `side`): a fourth grid
    // (index xg, -1 = none) and a third frame slot (nslots)
    int xg = -1, nslots = 2;
    // sparse transient grids (tofr_store.cuh): slot map per grid, pool rows
    // handed out per grid ([3] u32), pool rows per grid (+2 reserved rows)
    bool sparse = false;
    size_t pool_rows = 0;
    int pool_planes = kResChunks;  // chunk planes of a sparse grid (header included)
    bool compact_rows = false;     // sparse rows without the k = 2 prefix cache (ResStore::compact)
    // solve / finish overlap (ShiftQueue::done, ShiftOverlap; opt-in TOFR_OVERLAP=1)
    DevBuf wv_done, wv_fin_ctr, wv_nbr;
    uint32_t ov_epoch = 0;
    DevBuf row_cost;               // per image row shift cost (u64), counted while row_cost_on
    bool row_cost_on = false;
    // res_rows block (32 B): u32 rows handed out per grid [3], pad, u64 sticky
    // pool-overflow word (kErrPool; never reset: frames in flight share the
    // per-frame error word, and a full pool is fatal); occ_host: pinned copy of
    // the block per frame set [2][8 u32]
    unsigned int* occ_host = nullptr;
    size_t occ_seen = 0;               // largest of them over the frames flushed so far
    DevBuf res_slot[4], res_rows;
    DevBuf image, accum, hist;  // owned rows only (plain sessions: accum = wide-band image accumulator)
    DevBuf ctr;                             // [3 stages][SC_COUNT] u64 + band error flag + work counter
    DevBuf send_lo, send_hi, recv_lo, recv_hi;
    DevBuf wo_cls, wo_counts, wo_perm;  // cost-ordered reuse (TOFR_ORDER=0 disables)
    DevBuf sp_mapped, sp_ok, sp_rng, sp_list, sp_count;  // phased spatial pass (TOFR_SPATIAL=mono disables)
    bool phased = false;
    bool order = true;
    // wavefront reuse (tofr_wave.cu; TOFR_REUSE=legacy selects the per-item kernels)
    bool wave = false;
    DevBuf wv_jobs, wv_out, wv_ctl, wv_map_a, wv_map_b, wv_tsrc, wv_rng, wv_mlist;
    // shrink initialiser on the wavefront engine: the rough (wide-gate) grid and
    // the pick stream's counter per pixel between the RIS runs and the merge
    bool shrink_wave = false;
    DevBuf shrink_rough, shrink_pick;
    size_t wv_cap = 0;
    DevBuf row_jobs;          // per-row shift-job bounds of a stage (adaptive row batches)
    size_t batches_seen = 0;  // most row batches one stage took
    tofr_halo_exchange_fn xfn = nullptr;  // host callback transport (gloo / tests)
    void* xuser = nullptr;
    std::unique_ptr<HaloTransport> xport;   // native transport (NCCL or in-process peer copies)
    DevBuf ell_jobs, ell_res, ell_st, ell_ctr, ell_list, ell_count;  // wavefront ellipsoidal sampler
    EllScratch ell{};
    bool ell_ready = false;
    std::shared_ptr<PeerEndpoint> peer;
    uint64_t halo_exchanges = 0;
    // per-frame stage events, two frames in flight
    cudaEvent_t ev[2][7] = {};
    // Frame pipelining (ReSTIR sessions): frame f's upload, camera stage and
    // initial sampling run on `side` as soon as frame f-1's temporal stage is
    // done -- concurrently with frame f-1's spatial pass and shading on the
    // main stream.  They touch only the buffers frame f-1 no longer reads after
    // its temporal stage: the frame slot / G-buffer of frame f-2 and the grid
    // that held frame f-2's final reservoirs.  Gated sessions keep one frame
    // more (a fourth grid, a third slot): frame f's side work then waits for
    // frame f-2's temporal stage only, so it can also fill the SMs frame f-1's
    // temporal shift batch leaves idle while its slowest Newton chains finish
    // (TOFR_PIPE_DEPTH=2: the two-frame pipeline).
    cudaStream_t side = nullptr;
    cudaEvent_t ev_temporal[2] = {}, ev_init[2] = {};
    bool pending[2] = {false, false};
    unsigned long long* err_host = nullptr;  // pinned [2]
    cudaEvent_t read_ev[2] = {};             // asynchronous image read-backs (on copy_stream)
    // read-back slots: the frame's image is staged on the device (a D2D copy, or
    // the transient histogram sum written there directly) on the session stream,
    // then copied to the host on copy_stream, overlapping the next frames' kernels
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t staged_ev[2] = {};
    DevBuf read_stage[2];
    int f = 0;
    double prev_center = 0, prev_width = 0;
    double stage_ms[6] = {0, 0, 0, 0, 0, 0};
    double stage_tot[6] = {0, 0, 0, 0, 0, 0};
    int64_t tot_frames = 0;
    uint64_t camera_rays = 0;  // G-buffer rays (host count; the kernel has no counters)
    size_t last_h2d = 0;  // bytes uploaded by the last step (frame snapshot)
    int has_temporal = 0, has_bin = 0, has_spatial = 0;

    size_t items_stored() const { return size_t(r1 - r0) * W * B; }
    size_t owned_pixels() const { return size_t(y1 - y0) * W; }

    ~tofr_session() {
        if (ctx) {
            cudaSetDevice(ctx->device);
            if (side) cudaStreamSynchronize(side);
            if (ctx->stream) cudaStreamSynchronize(ctx->stream);
        }
        for (auto* e : {&ev_temporal[0], &ev_temporal[1], &ev_init[0], &ev_init[1]})
            if (*e) cudaEventDestroy(*e);
        if (side) cudaStreamDestroy(side);
        for (auto& set : ev)
            for (auto& e : set)
                if (e) cudaEventDestroy(e);
        for (auto& e : read_ev)
            if (e) cudaEventDestroy(e);
        for (auto& e : staged_ev)
            if (e) cudaEventDestroy(e);

        if (copy_stream) {
            cudaStreamSynchronize(copy_stream);
            cudaStreamDestroy(copy_stream);
        }
        if (err_host) cudaFreeHost(err_host);
        if (occ_host) cudaFreeHost(occ_host);
        if (ctx && ctx->l2_owner == this) {  // drop the persisting L2 window over our buffer
            cudaStreamAttrValue a;
            std::memset(&a, 0, sizeof(a));
            cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &a);
            cudaCtxResetPersistingL2Cache();
            cudaGetLastError();
            ctx->l2_owner = nullptr;
        }
        release_buffers();
        if (ctx && --ctx->live_sessions == 0 && ctx->closing) release_ctx(ctx);
    }
    void release_buffers() {
        for (auto& sl : slot) {
            sl.blob.release();
            sl.gbuf.release();
        }
        for (auto& r : res) r.release();
        for (auto& r : res_slot) r.release();
        res_rows.release();
        for (DevBuf* b : {&wv_done, &wv_fin_ctr, &wv_nbr, &row_cost, &read_stage[0], &read_stage[1], &image, &accum, &hist, &ctr, &send_lo, &send_hi, &recv_lo, &recv_hi, &wo_cls,
                          &wo_counts, &wo_perm, &sp_mapped, &sp_ok, &sp_rng, &sp_list, &sp_count, &wv_jobs, &wv_out,
                          &wv_ctl, &wv_map_a, &wv_map_b, &wv_tsrc, &wv_rng, &wv_mlist, &row_jobs})
            b->release();
    }
};

namespace {

template <class T>
const T* rows_base_c(const DevBuf& b, int row0, size_t per_row) {
    return b.as<T>() - ptrdiff_t(size_t(row0) * per_row);
}

// Global-indexed views of band-local buffers (see Band in tofr_kernels.h).
// `frame_slot`: the frame slot whose G-buffer and camera the grid's records
// belong to (compact pool rows rebuild their prefix cache from them).
ResStore store_of(const tofr_session* s, const DevBuf& b, int frame_slot = -1) {
    size_t items = s->items_stored();
    ptrdiff_t off = ptrdiff_t(size_t(s->r0) * s->W * s->B);
    if (!s->sparse) {
        ResStore st{b.as<double2>() - off, items};
        st.ilo = size_t(off);
        st.ihi = size_t(off) + items;
        return st;
    }
    int k = int(&b - &s->res[0]);
    ResStore st{b.as<double2>() - off, s->pool_rows + 2};
    st.ilo = size_t(off);
    st.ihi = size_t(off) + items;
    st.slot = s->res_slot[k].as<uint32_t>() - off;
    // chunk planes 1..23 follow the header plane; plane c at pool + c * stride
    st.pool = b.as<double2>() + items - ptrdiff_t(st.stride);
    st.rows = s->res_rows.as<unsigned int>() + k;
    st.err = reinterpret_cast<unsigned long long*>(s->res_rows.as<unsigned char>() + 16);
    st.planes = s->pool_planes;
    if (s->compact_rows) {
        if (frame_slot < 0) throw ScopeError(TOFR_ERR_INVALID, "compact reservoir rows need their frame");
        st.compact = 1;
        st.gbuf = rows_base_c<GHit>(s->slot[frame_slot].gbuf, s->r0, s->W);
        st.cam = s->slot[frame_slot].view.cam;
        st.bins = s->B;
    }
    return st;
}

// a sparse grid about to be rewritten (new frame's init, spatial / bin-reuse
// output): every reservoir loses its pool row
// Row batches of a wavefront reuse stage: the shift queue holds wv_cap jobs and
// a stage makes at most `per` jobs per item, so batches of at most
// wv_cap / per items can never overflow it (exact, no occupancy estimate; a
// transient grid whose worst case exceeds the queue pays one queue fill per
// batch).
int wave_batches(const tofr_session* s, size_t per) {
    size_t items = s->owned_pixels() * s->B;
    size_t rows = size_t(s->y1 - s->y0);
    size_t per_row = items / std::max<size_t>(1, rows);
    size_t rows_fit = s->wv_cap / std::max<size_t>(1, per * per_row);
    if (rows_fit == 0) throw ScopeError(TOFR_ERR_OOM, "reuse shift queue smaller than one image row (raise TOFR_WAVE_CAP)");
    return int((rows + rows_fit - 1) / rows_fit);
}
// Row cuts of a wavefront stage.  One batch when the worst case fits the queue;
// otherwise uniform row batches sized for the worst case, or -- opt-in,
// TOFR_ADAPTIVE_BATCHES=1, transient grids -- cuts from per-row upper bounds of
// the stage's jobs counted on the device (k_count_temporal / k_count_spatial:
// exact forward jobs, at most one inverse job per item that can have one; one
// host sync per stage).  Measured: 8 -> 2 batches at 1080p x 64 bins, 119 -> 17
// solve launches per C4 band frame, but the transient stages are throughput-
// bound, so the saved tails (solve 6.85 -> 6.76 ms) do not pay for the count
// pass (0.8-3.2 ms): 21.5 -> 20.9 frames/s, C4 band 3.80 -> 3.82 (r02s).
template <class Count>
std::vector<int> stage_cuts(tofr_session* s, const Band& bd, size_t per, cudaStream_t st, Count&& count) {
    const int nb = wave_batches(s, per);
    std::vector<int> cuts{bd.y0};
    const char* ad = std::getenv("TOFR_ADAPTIVE_BATCHES");
    if (nb > 1 && s->transient && ad && ad[0] == '1') {
        const int rows = bd.y1 - bd.y0;
        s->row_jobs.ensure(size_t(rows) * 8);
        std::vector<unsigned long long> h(static_cast<size_t>(rows), 0ull);
        count(s->row_jobs.as<unsigned long long>());
        ck(cudaMemcpyAsync(h.data(), s->row_jobs.p, size_t(rows) * 8, cudaMemcpyDeviceToHost, st), "row jobs");
        ck(cudaStreamSynchronize(st), "row jobs");
        unsigned long long acc = 0;
        for (int r = 0; r < rows; ++r) {
            if (acc + h[r] > s->wv_cap && acc > 0) {
                cuts.push_back(bd.y0 + r);
                acc = 0;
            }
            acc += h[r];  // <= wv_cap: a row's worst case fits (wave_batches)
        }
    } else {
        const int step = (bd.y1 - bd.y0 + nb - 1) / nb;  // <= rows_fit of wave_batches
        for (int y = bd.y0 + step; y < bd.y1; y += step) cuts.push_back(y);
    }
    cuts.push_back(bd.y1);
    s->batches_seen = std::max<size_t>(s->batches_seen, cuts.size() - 1);
    return cuts;
}
template <class Fn>
void for_row_cuts(const Band& bd, const std::vector<int>& cuts, Fn&& fn) {
    for (size_t k = 0; k + 1 < cuts.size(); ++k) {
        Band sb = bd;
        sb.y0 = cuts[k];
        sb.y1 = cuts[k + 1];
        fn(sb);
    }
}
template <class Fn>
void for_row_batches(const Band& bd, int nb, Fn&& fn) {
    int rows = (bd.y1 - bd.y0 + nb - 1) / nb;  // <= rows_fit of wave_batches
    for (int y = bd.y0; y < bd.y1; y += rows) {
        Band sb = bd;
        sb.y0 = y;
        sb.y1 = std::min(bd.y1, y + rows);
        fn(sb);
    }
}

// payload rows a compacted (sparse) halo of n items carries.  The sender's
// send buffer and the receiver's recv buffer must agree on the layout (the
// payload offsets depend on cap), so cap is a function of n alone -- never of
// a rank's own pool size, which depends on its free memory and band height.
// TOFR_HALO_FRAC (default 0.5: C4 bands peak at ~36% non-empty) must be the
// same on every rank; a halo with more non-empty reservoirs raises "pool full".
size_t halo_cap(const tofr_session* s, size_t n) {
    if (!s->sparse || !n) return 0;
    double frac = 0.5;
    if (const char* hf = std::getenv("TOFR_HALO_FRAC")) frac = std::atof(hf);
    if (!(frac > 0)) frac = 0.5;
    size_t cap = size_t(double(n) * frac) + 4096;
    return std::min(n, cap);
}

void reset_store(tofr_session* s, int k, cudaStream_t st) {
    if (!s->sparse) return;
    ck(cudaMemsetAsync(s->res_slot[k].p, 0xff, s->items_stored() * sizeof(uint32_t), st), "memset");
    ck(cudaMemsetAsync(s->res_rows.as<unsigned int>() + k, 0, sizeof(unsigned int), st), "memset");
}
template <class T>
T* rows_base(const DevBuf& b, int row0, size_t per_row) {
    return b.as<T>() - ptrdiff_t(size_t(row0) * per_row);
}

Band band_of(tofr_session* s, bool prev_halo_valid) {
    Band bd;
    bd.y0 = s->y0;
    bd.y1 = s->y1;
    bd.r0 = s->r0;
    bd.r1 = s->r1;
    bd.t0 = prev_halo_valid ? s->r0 : s->y0;
    bd.t1 = prev_halo_valid ? s->r1 : s->y1;
    bd.err = s->ctr.as<unsigned long long>() + 3 * SC_COUNT;
    return bd;
}

PathCfg path_cfg(const tofr_render_config& c, double center, double width, const HScene& sc) {
    PathCfg p;
    std::memset(&p, 0, sizeof(p));
    p.max_depth = c.max_depth;
    p.use_rr = c.use_rr;
    p.ellipsoidal = (c.init_mode == TOFR_INIT_ELLIPSOIDAL && c.gate_kind == TOFR_GATE_LENGTH) ? 1 : 0;
    p.ell_center = center;
    p.ell_width = width;
    p.gauge = c.gauge;
    p.newton = c.newton;
    p.jac_min = 1.0 / 50.0;
    p.jac_max = 50.0;
    p.m_cap = c.m_cap;
    p.seed = c.seed;
    p.replay = 0;
    {
        const char* wc = std::getenv("TOFR_WALK_CUTOFF");
        p.walk_cutoff = (wc && wc[0] == '0') ? 0 : 1;
    }
    p.shrink_k = c.shrink_k;
    p.work = nullptr;
    for (const HMaterial& m : sc.materials)
        if (!m.reconnectable()) p.replay = 1;
    return p;
}

// Static scenes (no animated object, no camera track): build_frame
// (scene.hpp:479-548) returns the same snapshot for every frame -- same
// world-space triangles, same SAH tree, same camera and beam -- so each slot
// builds and uploads it once (a 10^5-triangle mesh costs ~0.1 s of host SAH
// build per frame otherwise, the reference's per-frame rebuild, scene.hpp:503).
bool static_scene(const HScene& sc) {
    for (const HObject& o : sc.objects)
        if (o.track.animated()) return false;
    return sc.camera.track.size() <= 1;
}

void upload_frame(tofr_session* s, int which, double frame, int frame_id, cudaStream_t st) {
    FrameSlot& sl = s->slot[which];
    sl.gbuf.ensure(size_t(s->r1 - s->r0) * s->W * sizeof(GHit));
    if (sl.cached) {
        sl.pk.view.frame_id = frame_id;
        sl.view = rebase_view(sl.pk, static_cast<const unsigned char*>(sl.blob.p));
        s->last_h2d = 0;
        return;
    }
    if (s->device_bvh) {  // the tree built on the device (bvh_build.cu), packed in place
        HFrame hf = build_frame(s->scene, frame, false);
        if (!s->dbvh) s->dbvh = std::make_unique<DeviceBvh>();
        const int nt = int(hf.tris.size());
        sl.staging.ensure(size_t(nt) * sizeof(HTri));
        std::memcpy(sl.staging.p, hf.tris.data(), size_t(nt) * sizeof(HTri));
        const int nn = s->dbvh->build(sl.staging.p, nt, st);
        if (s->dbvh->depth > 60) throw ScopeError(TOFR_ERR_SCENE, "bvh deeper than supported");
        sl.pk = pack_frame_shell(s->scene, hf, nn, frame_id);
        sl.blob.ensure(sl.pk.blob.size());
        // the shell's host part: materials and velocity fields
        unsigned char* dst = static_cast<unsigned char*>(sl.blob.p);
        const size_t small = sl.pk.off_tframe - sl.pk.off_mats;
        ck(cudaMemcpyAsync(dst + sl.pk.off_mats, sl.pk.blob.data() + sl.pk.off_mats, small, cudaMemcpyHostToDevice, st),
           "frame upload");
        s->dbvh->pack(dst, sl.pk, st);
        ck(cudaStreamSynchronize(st), "frame upload");  // the staging buffer is reused by the next frame
        sl.view = rebase_view(sl.pk, dst);
        s->last_h2d = size_t(nt) * sizeof(HTri) + small;
        sl.cached = s->static_frames;
        return;
    }
    HFrame hf = build_frame(s->scene, frame);
    if (hf.max_depth > 60) throw ScopeError(TOFR_ERR_SCENE, "bvh deeper than supported");
    sl.pk = pack_frame(s->scene, hf, frame_id);
    size_t nb = sl.pk.blob.size();
    // the staging buffer of this slot was last copied two frames ago; that
    // frame's events were synchronised before this call (flush_set)
    sl.staging.ensure(nb);
    std::memcpy(sl.staging.p, sl.pk.blob.data(), nb);
    sl.blob.ensure(nb);
    ck(cudaMemcpyAsync(sl.blob.p, sl.staging.p, nb, cudaMemcpyHostToDevice, st), "frame upload");
    sl.view = rebase_view(sl.pk, static_cast<const unsigned char*>(sl.blob.p));
    s->last_h2d = nb;
    sl.cached = s->static_frames;
}

void check_config(const tofr_render_config* c) {
    if (!c) throw ScopeError(TOFR_ERR_INVALID, "null config");
    if (c->max_depth < 1 || c->max_depth > 64) throw ScopeError(TOFR_ERR_INVALID, "max_depth out of range");
    if (c->frames < 0) throw ScopeError(TOFR_ERR_INVALID, "frames < 0");
    if (c->gate_kind == TOFR_GATE_VELOCITY) {
        // Doppler gates (render_doppler, pipeline.hpp:573-578): the gated image
        // pipeline on the path velocity; built on the wavefront kernels
        if (c->mode == TOFR_MODE_TRANSIENT)
            throw ScopeError(TOFR_ERR_UNSUPPORTED, "velocity gates apply to gated rendering only");
        if (!(c->gate_f0 != 0)) throw ScopeError(TOFR_ERR_INVALID, "velocity gate needs a carrier f0");
        for (const char* var : {"TOFR_REUSE", "TOFR_TRACE"}) {
            const char* e = std::getenv(var);
            if (e && std::strcmp(e, "legacy") == 0)
                throw ScopeError(TOFR_ERR_UNSUPPORTED, "velocity gates need the wavefront kernels (unset TOFR_REUSE / TOFR_TRACE)");
        }
    } else if (c->gate_kind != TOFR_GATE_LENGTH) {
        throw ScopeError(TOFR_ERR_INVALID, "unknown gate kind");
    }
}

enum SessionKind { KIND_RESTIR = 0, KIND_PLAIN = 1, KIND_BARE = 2 };

// Persisting L2 access-policy window on the context stream over [p, p + bytes),
// owned by session `owner` (its destructor clears it).
void set_l2_window(tofr_gpu* ctx, const void* owner, void* p, size_t bytes) {
    int dev = 0, max_persist = 0, max_win = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    if (max_persist <= 0 || max_win <= 0) return;
    cudaStreamAttrValue a;
    std::memset(&a, 0, sizeof(a));
    if (bytes) {
        size_t win = std::min(bytes, size_t(max_win));
        size_t keep = std::min(win, size_t(max_persist));
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, keep);
        a.accessPolicyWindow.base_ptr = p;
        a.accessPolicyWindow.num_bytes = win;
        a.accessPolicyWindow.hitRatio = float(double(keep) / double(win));
        a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    }
    cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &a);
    cudaGetLastError();  // best effort: no window is not an error
    ctx->l2_owner = owner;
}

tofr_session* make_session(tofr_gpu* ctx, const tofr_scene* sc, const tofr_render_config* cfg, int kind,
                           int y0 = 0, int y1 = -1, int halo = 0) {
    check_config(cfg);
    auto s = std::make_unique<tofr_session>();
    s->ctx = ctx;
    ctx->live_sessions++;
    s->scene = sc->s;
    s->cfg = *cfg;
    s->W = sc->s.camera.width;
    s->H = sc->s.camera.height;
    if (s->W <= 0 || s->H <= 0) throw ScopeError(TOFR_ERR_INVALID, "empty image");
    if (y1 < 0) y1 = s->H;
    if (y0 < 0 || y1 > s->H || y0 >= y1 || halo < 0) throw ScopeError(TOFR_ERR_INVALID, "bad row band");
    s->y0 = y0;
    s->y1 = y1;
    s->r0 = std::max(0, y0 - halo);
    s->r1 = std::min(s->H, y1 + halo);
    if ((y0 - s->r0) > (y1 - y0) || (s->r1 - y1) > (y1 - y0))
        throw ScopeError(TOFR_ERR_INVALID, "row band thinner than its halo (use fewer ranks)");
    s->cam_moves = !sc->s.camera.track.empty();
    const char* sf = std::getenv("TOFR_STATIC_FRAMES");
    s->static_frames = static_scene(sc->s) && !(sf && sf[0] == '0');
    {
        // TOFR_DEVICE_BVH=1: always (wide-light scenes), 0: never; default: when a
        // non-static frame has >= 4096 triangles (the host SAH build then costs
        // more than the device build's per-level syncs)
        size_t ntri = 0;
        for (const HObject& o : sc->s.objects) ntri += o.local.size();
        const char* db = std::getenv("TOFR_DEVICE_BVH");
        const bool wide = sc->s.light.regime == LIGHT_WIDE;
        if (db && db[0] == '1')
            s->device_bvh = wide;
        else if (!(db && db[0] == '0'))
            s->device_bvh = wide && !s->static_frames && ntri >= 4096;
    }
    if (kind == KIND_RESTIR && cfg && cfg->temporal && s->cam_moves && halo == 0 && (y0 > 0 || y1 < s->H))
        throw ScopeError(TOFR_ERR_INVALID,
                         "row band of a moving camera with temporal reuse needs a reprojection halo (halo > 0)");
    for (auto& set : s->ev)
        for (auto& e : set) ck(cudaEventCreate(&e), "event");
    for (auto& e : s->read_ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    for (auto& e : s->staged_ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    ck(cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking), "stream");
    ck(cudaMallocHost(reinterpret_cast<void**>(&s->err_host), 2 * sizeof(unsigned long long)), "pinned");
    s->err_host[0] = s->err_host[1] = 0;
    // [3 stages x SC_COUNT][band error][work counter q][WK_COUNT device work][side-stream work counter]
    s->ctr.ensure((3 * SC_COUNT + 3 + WK_COUNT) * sizeof(unsigned long long));
    ck(cudaMemsetAsync(s->ctr.p, 0, (3 * SC_COUNT + 3 + WK_COUNT) * sizeof(unsigned long long), ctx->stream),
       "memset");
    if (kind == KIND_BARE) return s.release();
    bool plain = kind == KIND_PLAIN;
    s->plain = plain;
    // on by default (TOFR_PIPELINE=0: off): +0.2-3.5% frames/s, bit-identical
    // (test_pipelined_frames_equal_serial); the per-kernel event times of a
    // pipelined run overlap
    const char* pipe_env = std::getenv("TOFR_PIPELINE");
    if (!plain && !(pipe_env && pipe_env[0] == '0')) {
        ck(cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking), "stream");
        for (auto* e : {&s->ev_temporal[0], &s->ev_temporal[1], &s->ev_init[0], &s->ev_init[1]})
            ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    }
    s->transient = plain || cfg->mode == TOFR_MODE_TRANSIENT;
    s->B = s->transient ? cfg->bins : 1;
    if (s->transient && (cfg->bins < 1 || !(cfg->hist_bin_width > 0)))
        throw ScopeError(TOFR_ERR_INVALID, "transient needs bins >= 1 and hist_bin_width > 0");
    if (!s->transient && cfg->m_init < 0) throw ScopeError(TOFR_ERR_INVALID, "m_init < 0");
    size_t own = s->owned_pixels() * s->B;
    if (plain) {
        // 32 B bin records {r, g, b, count} (hist_deposit) + the wide-band image accumulator
        s->hist.ensure(own * 4 * sizeof(double));
        ck(cudaMemsetAsync(s->hist.p, 0, own * 4 * sizeof(double), ctx->stream), "memset");
        s->accum.ensure(s->owned_pixels() * 3 * sizeof(double));
        ck(cudaMemsetAsync(s->accum.p, 0, s->owned_pixels() * 3 * sizeof(double), ctx->stream), "memset");
        // the image accumulator is read-modify-written by every frame's deposits:
        // keep it in a persisting L2 window (50 MB at 1080p) so the streaming
        // histogram sectors (evict-first reductions) do not push it to HBM
        const char* l2p = std::getenv("TOFR_L2_PERSIST");
        if (!(l2p && l2p[0] == '0')) set_l2_window(ctx, s.get(), s->accum.p, s->owned_pixels() * 3 * sizeof(double));
    } else {
        s->has_temporal = cfg->temporal ? 1 : 0;
        s->has_bin = (s->transient && cfg->bin_reuse) ? 1 : 0;
        s->has_spatial = cfg->spatial_passes > 0 ? 1 : 0;
        size_t items = s->items_stored();
        size_t rb = items * kResChunks * 16;
        // three-frame buffers (see `side`): only for frames staged in shared
        // memory -- a snapshot traversed from L2 (the 10^5-triangle mesh)
        // measured 6% slower with a third frame's copy competing for the cache
        // (profiles/r02/ab_pipe.txt); transient grids: below
        size_t n_tris = 0;
        for (const HObject& o : s->scene.objects) n_tris += o.local.size();
        const bool staged = n_tris * (2 * sizeof(GNode) + sizeof(GTriIsect)) <= kSmemStageLimit;
        const char* pdepth = std::getenv("TOFR_PIPE_DEPTH");
        bool deep = s->side && staged && !(pdepth && pdepth[0] == '2');
        {
            // transient grids are mostly empty reservoirs: header plane + a pool
            // of sample rows (TOFR_SPARSE=0: dense).  Pool rows per grid: one per
            // item while the three pools fit in 55% of the free memory, else what
            // fits (TOFR_POOL_FRAC: that fraction of the items instead).
            const char* sp = std::getenv("TOFR_SPARSE");
            s->sparse = s->transient && !(sp && sp[0] == '0');
            // three-frame buffers for sparse grids only where the fourth grid takes
            // the place of the spare one a temporal-only session does not use
            deep = deep && (!s->transient || (s->sparse && !s->has_bin && !s->has_spatial));
            if (s->sparse) {
                // records of scenes without non-reconnectable materials never carry
                // replay lanes (k = 2), and transient gates are length gates: the
                // pool holds chunks 1-19 only
                bool lanes = false;
                for (const HMaterial& m : sc->s.materials)
                    if (!m.reconnectable()) lanes = true;
                s->pool_planes = lanes ? kResChunks : 20;
                // ... and without replay lanes every record reconnects at k = 2, so its
                // prefix cache (chunks 5-9) is rebuilt from the G-buffer: 224 B rows
                // (TOFR_COMPACT_ROWS=0: 304 B)
                const char* cr = std::getenv("TOFR_COMPACT_ROWS");
                s->compact_rows = !lanes && !(cr && cr[0] == '0');
                const size_t row_bytes = size_t(s->pool_planes - 1 - (s->compact_rows ? 5 : 0)) * 16;
                size_t rows = items;
                size_t fr = 0, tot = 0;
                if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
                    auto fit_rows = [&](size_t ngrid) {
                        size_t fit = size_t(double(fr) * 0.55) / ngrid;
                        fit = fit > items * 20 ? (fit - items * 20) / row_bytes : 0;
                        return std::min(rows, std::max<size_t>(fit, 1024));
                    };
                    const size_t ngrid = (s->has_bin || s->has_spatial) ? 3 : 2;
                    // the fourth grid only while the pools still hold half the grid
                    // (1080p x 256 bins: 187 M rows per pool with two, 109 M with three
                    // -- 94 M in use by frame 45 -- so it keeps two frames)
                    if (deep && fit_rows(ngrid + 1) < items / 2) deep = false;
                    rows = fit_rows(deep ? ngrid + 1 : ngrid);
                }
                if (const char* pf = std::getenv("TOFR_POOL_FRAC")) rows = size_t(double(items) * std::atof(pf)) + 1;
                if (rows > items) rows = items;
                if (const char* pr = std::getenv("TOFR_POOL_ROWS")) rows = size_t(std::strtoull(pr, nullptr, 10));
                if (rows > 0xfffffff0ull) rows = 0xfffffff0ull;
                s->pool_rows = rows;
                rb = items * 16 + row_bytes * (rows + 2);
                for (int k = 0; k < 4; ++k)
                    if (k < 2 || ((s->has_bin || s->has_spatial) && k == 2) || (deep && k == 3)) {
                        s->res_slot[k].ensure(items * sizeof(uint32_t));
                        ck(cudaMemsetAsync(s->res_slot[k].p, 0xff, items * sizeof(uint32_t), ctx->stream), "memset");
                    }
                ck(cudaMallocHost(reinterpret_cast<void**>(&s->occ_host), 16 * sizeof(unsigned int)), "pinned");
                std::memset(s->occ_host, 0, 16 * sizeof(unsigned int));
                s->res_rows.ensure(32);
                ck(cudaMemsetAsync(s->res_rows.p, 0, 32, ctx->stream), "memset");
            }
        }
        s->res[0].ensure(rb);
        s->res[1].ensure(rb);
        if (s->has_bin || s->has_spatial) s->res[2].ensure(rb);
        // a never-written grid must read as empty (M = 0) for temporal reuse
        ck(cudaMemsetAsync(s->res[0].p, 0, rb, ctx->stream), "memset");
        ck(cudaMemsetAsync(s->res[1].p, 0, rb, ctx->stream), "memset");
        if (s->res[2].p) ck(cudaMemsetAsync(s->res[2].p, 0, rb, ctx->stream), "memset");
        if (deep) {
            s->res[3].ensure(rb);
            ck(cudaMemsetAsync(s->res[3].p, 0, rb, ctx->stream), "memset");
            s->xg = 3;
            s->nslots = 3;
        }
        {
            // wavefront reuse: job queue of (N + 1) jobs per item for the spatial
            // pass (2 for temporal), bounded for the transient grids, whose
            // non-empty reservoirs are a small fraction of W x H x B
            const char* rv = std::getenv("TOFR_REUSE");
            size_t own_items = s->owned_pixels() * s->B;
            size_t nj = size_t(std::max(0, cfg->spatial_neighbors));
            const char* tv = std::getenv("TOFR_TRACE");
            const bool shrink = !s->transient && cfg->init_mode == TOFR_INIT_SHRINK &&
                                cfg->gate_kind == TOFR_GATE_LENGTH && !(tv && std::strcmp(tv, "legacy") == 0);
            s->wave = (s->has_temporal || s->has_spatial || s->has_bin || shrink) &&
                      !(rv && std::strcmp(rv, "legacy") == 0);
            s->shrink_wave = shrink && s->wave && !s->sparse;
            if (s->wave) {
                size_t per = wave_jobs_per_item(s->has_spatial ? cfg->spatial_neighbors : 0);
                if (s->has_bin) per = std::max<size_t>(per, 3);  // bin reuse: 2 forward + 1 inverse
                size_t cap = per * own_items;
                // 64 M jobs (38 GB) when a quarter of the free memory holds them, else 32 M;
                // larger stages run in row batches (wave_batches)
                size_t limit = size_t(32) << 20;
                {
                    size_t fr = 0, tot = 0;
                    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess &&
                        fr / 4 > (size_t(64) << 20) * (kJobChunks + kResChunks) * 16)
                        limit = size_t(64) << 20;
                }
                if (const char* cl = std::getenv("TOFR_WAVE_CAP")) limit = size_t(std::strtoull(cl, nullptr, 10));
                if (cap > limit) cap = limit;
                if (cap > 0xfffffff0ull) cap = 0xfffffff0ull;
                s->wv_cap = cap;
                s->wv_jobs.ensure(cap * kJobChunks * 16);
                s->wv_out.ensure(cap * kResChunks * 16);
                s->wv_ctl.ensure(16);
                s->wv_map_a.ensure(std::max<size_t>(s->has_bin ? 2 : 1, nj) * own_items * sizeof(uint32_t));
                s->wv_map_b.ensure(own_items * sizeof(uint32_t));
                s->wv_tsrc.ensure(own_items * sizeof(uint64_t));
                s->wv_rng.ensure(own_items * sizeof(uint64_t));
                s->wv_mlist.ensure(own_items * sizeof(uint32_t));
                s->wv_nbr.ensure(std::max<size_t>(1, nj) * s->owned_pixels() * sizeof(uint32_t));
                if (s->shrink_wave) {
                    s->shrink_rough.ensure(rb);
                    s->shrink_pick.ensure(s->owned_pixels() * sizeof(uint64_t));
                }
                // opt-in (TOFR_OVERLAP=1): measured 2-7% slower -- the finish warps
                // take issue slots from the tail's serial Newton chains
                const char* ovs = std::getenv("TOFR_OVERLAP");
                if (ovs && ovs[0] == '1') {
                    s->wv_done.ensure(cap * sizeof(uint32_t));
                    ck(cudaMemsetAsync(s->wv_done.p, 0, cap * sizeof(uint32_t), ctx->stream), "memset");
                    s->wv_fin_ctr.ensure(16);
                }
            }
        }
        const char* ord = std::getenv("TOFR_ORDER");
        s->order = !(ord && ord[0] == '0');
        {
            // phased spatial pass: N planes of forward-shifted samples; only when
            // they fit comfortably (gated frames; transient grids use k_spatial)
            const char* sm = std::getenv("TOFR_SPATIAL");
            size_t own_items = s->owned_pixels() * s->B;
            size_t nj = size_t(std::max(0, cfg->spatial_neighbors));
            size_t need = nj * own_items * kResChunks * 16;
            s->phased = !s->wave && s->has_spatial && nj > 0 && cfg->spatial_radius > 0 &&
                        !(sm && std::strcmp(sm, "mono") == 0) && need <= (size_t(16) << 30);
            if (s->phased) {
                s->sp_mapped.ensure(need);
                s->sp_ok.ensure(nj * own_items);
                s->sp_rng.ensure(own_items * sizeof(uint64_t));
                s->sp_list.ensure(nj * own_items * sizeof(uint32_t));
                s->sp_count.ensure(16);
            }
        }
        if (s->order && !s->wave) {
            size_t own_items = s->owned_pixels() * s->B;
            s->wo_cls.ensure(own_items);
            s->wo_perm.ensure(own_items * sizeof(uint32_t));
            s->wo_counts.ensure(64 * sizeof(uint32_t));
        }
        if (s->transient) {
            s->hist.ensure(own * 3 * sizeof(double));
            ck(cudaMemsetAsync(s->hist.p, 0, own * 3 * sizeof(double), ctx->stream), "memset");
        } else {
            size_t npix = s->owned_pixels();
            s->image.ensure(npix * 3 * sizeof(double));
            s->accum.ensure(npix * 3 * sizeof(double));
            ck(cudaMemsetAsync(s->accum.p, 0, npix * 3 * sizeof(double), ctx->stream), "memset");
            ck(cudaMemsetAsync(s->image.p, 0, npix * 3 * sizeof(double), ctx->stream), "memset");
        }
        // read-back staging (tofr_gpu_session_read_image_async) allocated with the
        // session: a cudaMalloc at the first read-backs of a frame loop would
        // synchronise the device in the middle of it
        for (auto& rs : s->read_stage) rs.ensure(s->owned_pixels() * 24);
        size_t per_row_items = size_t(s->W) * s->B;
        size_t lo = halo_bytes(size_t(s->y0 - s->r0) * per_row_items, halo_cap(s.get(), size_t(s->y0 - s->r0) * per_row_items),
                               s->sparse);
        size_t hi = halo_bytes(size_t(s->r1 - s->y1) * per_row_items, halo_cap(s.get(), size_t(s->r1 - s->y1) * per_row_items),
                               s->sparse);
        if (lo) {
            s->send_lo.ensure(lo);
            s->recv_lo.ensure(lo);
            ck(cudaMemsetAsync(s->recv_lo.p, 0, lo, ctx->stream), "memset");  // empty until received
        }
        if (hi) {
            s->send_hi.ensure(hi);
            s->recv_hi.ensure(hi);
            ck(cudaMemsetAsync(s->recv_hi.p, 0, hi, ctx->stream), "memset");
        }
    }
    return s.release();
}

void fill_counts(tofr_shift_counts& o, const unsigned long long* c) {
    o.attempts = c[SC_ATTEMPTS];
    o.newton_ok = c[SC_NEWTON_OK];
    o.newton_failed = c[SC_NEWTON_FAILED];
    o.occluded = c[SC_OCCLUDED];
    o.jac_clamped = c[SC_JAC_CLAMPED];
    o.replay_failed = c[SC_REPLAY_FAILED];
    o.iterations = c[SC_ITERATIONS];
    o.solves = c[SC_SOLVES];
    o.success = c[SC_SUCCESS];
}

// Waits for the frame recorded in event set `set`, folds its stage times into
// the running totals and checks the band error flag it copied out.
void flush_set(tofr_session* s, int set) {
    if (!s->pending[set]) return;
    ck(cudaEventSynchronize(s->ev[set][6]), "frame");
    s->pending[set] = false;
    if (kt_enabled()) kt_collect();
    float ms[6];
    for (int i = 0; i < 5; ++i) {
        ms[i] = 0;
        cudaEventElapsedTime(&ms[i], s->ev[set][i], s->ev[set][i + 1]);
    }
    ms[5] = 0;
    cudaEventElapsedTime(&ms[5], s->ev[set][0], s->ev[set][6]);
    // stage split: init (incl. camera), temporal, bin, spatial (incl. halo), shade, total
    for (int i = 0; i < 6; ++i) {
        s->stage_ms[i] = ms[i];
        s->stage_tot[i] += ms[i];
    }
    s->tot_frames++;
    if (s->sparse)
        for (int k = 0; k < 4; ++k) s->occ_seen = std::max<size_t>(s->occ_seen, s->occ_host[8 * set + k]);
    unsigned long long pool_err = 0;
    if (s->sparse) std::memcpy(&pool_err, s->occ_host + 8 * set + 4, 8);
    if ((s->err_host[set] | pool_err) & kErrHalo)
        throw ScopeError(TOFR_ERR_OOM,
                         "compacted halo overflow: more non-empty reservoirs in the halo rows than TOFR_HALO_FRAC "
                         "of them (raise it on every rank)");
    if ((s->err_host[set] | pool_err) & kErrPool)
        throw ScopeError(TOFR_ERR_OOM,
                         "transient reservoir pool full: more non-empty reservoirs than TOFR_POOL_FRAC of the grid "
                         "(raise it, or TOFR_SPARSE=0)");
    if (s->err_host[set] >> 32)
        throw ScopeError(TOFR_ERR_OOM,
                         "reuse shift queue overflow: more shifts than TOFR_WAVE_CAP jobs in one stage (raise it, or "
                         "TOFR_REUSE=legacy)");
    if (s->err_host[set])
        throw ScopeError(TOFR_ERR_UNSUPPORTED,
                         "row band read outside its rows (camera motion larger than the halo, or a spatial "
                         "radius larger than the halo)");
}

void flush_all(tofr_session* s) {
    int a = s->f & 1;  // oldest pending first
    flush_set(s, a);
    flush_set(s, a ^ 1);
}

// Halo exchange of a global-indexed grid around the band: pack the edge rows
// the neighbours need, let the caller move them (NCCL / P2P, ordered on the
// session stream), unpack what arrived into the halo rows.
// Scratch of the wavefront ellipsoidal sampler (EllScratch, tofr_ellipsoid.cuh)
// for an ellipsoidal gated initialisation; null: the per-lane sampler
// (TOFR_ELL=legacy, or not enough memory).
const EllScratch* ell_scratch(tofr_session* s, const PathCfg& pc, const InitParams& ip) {
    if (!pc.ellipsoidal || ip.mode != INIT_ELLIPSOIDAL) return nullptr;
    const char* e = std::getenv("TOFR_ELL");
    if (e && std::strcmp(e, "legacy") == 0) return nullptr;
    const int per_pixel = std::max(1, ip.m_init) * std::max(1, s->cfg.max_depth - 2);
    const size_t slots = s->owned_pixels() * size_t(per_pixel);
    if (!s->ell_ready || s->ell.per_pixel != per_pixel) {
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) == cudaSuccess && slots * kEllSlotBytes > fr / 2) return nullptr;
        s->ell_jobs.ensure(slots * sizeof(EllJob));
        s->ell_res.ensure(slots * sizeof(EllRes));
        s->ell_st.ensure(slots);
        s->ell_ctr.ensure(slots * 8);
        s->ell_list.ensure(slots * 4);
        s->ell_count.ensure(16);
        s->ell = EllScratch{s->ell_jobs.as<EllJob>(), s->ell_res.as<EllRes>(), s->ell_st.as<uint8_t>(),
                            s->ell_ctr.as<uint64_t>(), s->ell_list.as<uint32_t>(), s->ell_count.as<unsigned int>(),
                            per_pixel};
        s->ell_ready = true;
    }
    return &s->ell;
}

HaloBufs halo_bufs(const tofr_session* s) {
    HaloBufs b;
    b.send_lo = s->send_lo.p;
    b.recv_lo = s->recv_lo.p;
    b.bytes_lo = s->send_lo.p ? s->send_lo.n : 0;
    b.send_hi = s->send_hi.p;
    b.recv_hi = s->recv_hi.p;
    b.bytes_hi = s->send_hi.p ? s->send_hi.n : 0;
    b.device = s->ctx->device;
    b.stream = s->ctx->stream;
    return b;
}

void exchange_halo(tofr_session* s, ResStore g, int pass) {
    if (s->r0 == s->y0 && s->r1 == s->y1) return;
    if (!s->xport && !s->xfn)
        throw ScopeError(TOFR_ERR_INVALID, "band session with a halo needs a halo transport (NCCL, peer link or "
                                           "exchange callback)");
    cudaStream_t st = s->ctx->stream;
    size_t per_row = size_t(s->W) * s->B;
    size_t lo = size_t(s->y0 - s->r0) * per_row, hi = size_t(s->r1 - s->y1) * per_row;
    const HaloBufs hb = halo_bufs(s);
    if (s->xport) s->xport->before_pack(hb);
    launch_halo_pack(g, size_t(s->y0) * per_row, lo, s->send_lo.as<double2>(), halo_cap(s, lo), st);
    launch_halo_pack(g, size_t(s->y1) * per_row - hi, hi, s->send_hi.as<double2>(), halo_cap(s, hi), st);
    ck(cudaGetLastError(), "halo pack");
    if (s->xport) {
        s->xport->exchange(hb, pass);
    } else {
        int rc = s->xfn(s->xuser, pass);
        if (rc != 0) throw ScopeError(TOFR_ERR_CUDA, "halo exchange callback failed");
    }
    launch_halo_unpack(g, size_t(s->r0) * per_row, lo, s->recv_lo.as<double2>(), halo_cap(s, lo), st);
    launch_halo_unpack(g, size_t(s->y1) * per_row, hi, s->recv_hi.as<double2>(), halo_cap(s, hi), st);
    ck(cudaGetLastError(), "halo unpack");
    s->halo_exchanges++;
}

// One frame of the pipeline (body of the frame loops).  Asynchronous unless
// `st` is requested (then it waits for the frame and reads its counters).
void session_step(tofr_session* s, tofr_frame_stats* st) {
    cudaStream_t stream = s->ctx->stream;
    const tofr_render_config& c = s->cfg;
    int f = s->f;
    int set = f & 1;
    flush_set(s, set);  // frame f-2: frees its event set and its staging buffer
    int sl = f % s->nslots, psl = (f + s->nslots - 1) % s->nslots;
    if (s->side && !s->plain) {
        if (s->nslots == 3) {
            if (f > 1)  // frame f-1 no longer reads frame f-3's slot and grid after frame f-2's temporal stage
                cudaStreamWaitEvent(s->side, s->ev_temporal[set], 0);
        } else if (f > 0) {  // frame f-1 no longer reads frame f-2's slot and grid
            cudaStreamWaitEvent(s->side, s->ev_temporal[set ^ 1], 0);
        }
    }
    upload_frame(s, sl, c.frame0 + f, f, (s->side && !s->plain) ? s->side : stream);
    const FrameView& F = s->slot[sl].view;
    GHit* g_local = s->slot[sl].gbuf.as<GHit>();
    const GHit* g = rows_base<GHit>(s->slot[sl].gbuf, s->r0, s->W);
    // gate of this frame (RenderConfig::gate_at) in constraint units
    // (GateSpec::ccenter / cwidth: Hz / f0 for velocity gates)
    const bool vel = c.gate_kind == TOFR_GATE_VELOCITY;
    double center = c.gate_center + c.gate_step * f;
    double width = c.gate_width;
    if (vel) {
        center = center / c.gate_f0;
        width = width / c.gate_f0;
    }
    PathCfg pc = path_cfg(c, center, width, s->scene);
    pc.gate_vel = vel ? 1 : 0;
    pc.work = s->ctr.as<unsigned long long>() + 3 * SC_COUNT + 2;
    pc.row_cost = s->row_cost_on ? s->row_cost.as<unsigned long long>() : nullptr;
    HistSpec h{s->B, c.hist_t0, c.hist_bin_width};
    unsigned long long* ctr = s->ctr.as<unsigned long long>();
    unsigned long long* q = ctr + 3 * SC_COUNT + 1;  // persistent-kernel work counter (stream-ordered reuse)
    bool halo = !(s->r0 == s->y0 && s->r1 == s->y1);
    bool prev_halo = halo && s->cam_moves;
    Band bd = band_of(s, prev_halo);
    cudaEvent_t* ev = s->ev[set];
    // camera + initial sampling stream (see tofr_session::side)
    const bool piped = s->side != nullptr && !s->plain;
    cudaStream_t fs = piped ? s->side : stream;
    unsigned long long* q_side = piped ? ctr + 3 * SC_COUNT + 2 + WK_COUNT : q;
    WorkOrder wo{nullptr, nullptr, nullptr};
    WaveScratch wv;
    if (s->wave) {
        size_t own_items = s->owned_pixels() * s->B;
        (void)own_items;
        wv.q.jobs = s->wv_jobs.as<double2>();
        wv.q.cap = s->wv_cap;
        wv.q.out = ResStore{s->wv_out.as<double2>(), s->wv_cap};
        wv.q.out.ihi = s->wv_cap;
        // mapped records land in compact grids only: their prefix-cache chunks
        // (5-9) would be dropped by put_mapped, so the job outputs skip them too
        wv.q.out.compact = s->compact_rows ? 1 : 0;
        wv.q.ctl = s->wv_ctl.as<uint32_t>();
        wv.map_a = s->wv_map_a.as<uint32_t>();
        wv.map_b = s->wv_map_b.as<uint32_t>();
        wv.tsrc = s->wv_tsrc.as<uint64_t>();
        wv.rng_ctr = s->wv_rng.as<uint64_t>();
        wv.mlist = s->wv_mlist.as<uint32_t>();
        wv.nbr = s->wv_nbr.as<uint32_t>();
        if (s->wv_done.p) {
            wv.q.done = s->wv_done.as<uint32_t>();
            wv.ov.fin_ctr = s->wv_fin_ctr.as<unsigned long long>();
            wv.ov.epoch = &s->ov_epoch;
        }
    }
    if (s->order && s->wo_perm.p)
        wo = WorkOrder{s->wo_cls.as<uint8_t>(), s->wo_counts.as<uint32_t>(), s->wo_perm.as<uint32_t>()};
    if (!piped) ck(cudaMemsetAsync(ctr, 0, (3 * SC_COUNT + 1) * sizeof(unsigned long long), stream), "memset");

    cudaEventRecord(ev[0], fs);
    launch_gbuffer(F, bd, g_local, fs);
    s->camera_rays += uint64_t(s->r1 - s->r0) * s->W;
    if (s->plain) {
        size_t pr = size_t(s->W) * s->B;
        launch_hist_plain(F, bd, g, pc, h, c.m_init, f, rows_base<double>(s->hist, s->y0, pr * 4),
                          rows_base<double>(s->accum, s->y0, size_t(s->W) * 3), q, stream);
        for (int i = 1; i < 6; ++i) cudaEventRecord(ev[i], stream);
    } else {
        // the ellipsoidal and shrink initializers apply to length gates only; velocity
        // gates fall back to plain RIS (pipeline.hpp:110, :130)
        InitParams ip{vel ? int(INIT_DIRECT) : c.init_mode, c.m_init, center, width, c.shrink_k, c.shrink_r};
        reset_store(s, s->cur, fs);
        ResStore cur = store_of(s, s->res[s->cur], sl);
        // shrink initialiser (pipeline.hpp:137-183) on the wavefront engine: the
        // rough and fine RIS runs here, the shrink_map shifts and the merge on
        // the main stream below (they use the stage shift queue)
        int shrink_fine = -1;
        ResStore rough{};
        if (s->transient) {
            launch_init_transient(F, bd, g, pc, ip, h, f, cur, q_side, fs);
        } else if (s->shrink_wave && ip.mode == INIT_SHRINK) {
            int m_rough = int(std::llround(ip.shrink_r * ip.m_init));
            m_rough = std::min(std::max(m_rough, 0), ip.m_init);
            const int m_fine = ip.m_init - m_rough;
            uint64_t* pick = s->shrink_pick.as<uint64_t>();
            if (m_rough == 0 || !(ip.shrink_k >= 1)) {  // no rough candidates / K < 1: the fine RIS alone
                if (m_rough == 0)
                    launch_trace_gated_ris(F, bd, g, pc, ip.m_init, center, width, f, cur, nullptr, nullptr, q_side, fs);
                else  // shrink_map refuses K < 1: every rough winner fails to map
                    launch_init_gated(F, bd, g, pc, ip, f, cur, q_side, fs, nullptr);
            } else {
                rough = ResStore{s->shrink_rough.as<double2>() - ptrdiff_t(size_t(s->r0) * s->W), s->items_stored()};
                rough.ilo = size_t(s->r0) * s->W;
                rough.ihi = rough.ilo + s->items_stored();
                launch_trace_gated_ris(F, bd, g, pc, m_rough, center, width * ip.shrink_k, f, rough, nullptr, pick,
                                       q_side, fs);
                if (m_fine > 0)
                    launch_trace_gated_ris(F, bd, g, pc, m_fine, center, width, f, cur, pick, pick, q_side, fs);
                shrink_fine = m_fine;
            }
        } else {
            launch_init_gated(F, bd, g, pc, ip, f, cur, q_side, fs, ell_scratch(s, pc, ip));
        }
        cudaEventRecord(ev[1], fs);
        if (piped) {  // the main stream continues once this frame's reservoirs exist
            cudaEventRecord(s->ev_init[set], fs);
            cudaStreamWaitEvent(stream, s->ev_init[set], 0);
            ck(cudaMemsetAsync(ctr, 0, (3 * SC_COUNT + 1) * sizeof(unsigned long long), stream), "memset");
        }
        if (shrink_fine >= 0)
            launch_shrink_wave(F, bd, g, pc, center, width, shrink_fine, f, rough, cur, s->shrink_pick.as<uint64_t>(),
                               wv, ctr + 0 * SC_COUNT, q, stream);
        GateGrid cg{s->transient ? 1 : 0, center, width, h};
        if (c.temporal && f > 0) {
            GateGrid pg{s->transient ? 1 : 0, s->prev_center, s->prev_width, h};
            const GHit* gp = rows_base<GHit>(s->slot[psl].gbuf, s->r0, s->W);
            if (s->wave) {
                ResStore prev_st = store_of(s, s->res[s->prev], psl);
                auto cuts = stage_cuts(s, bd, 2, stream, [&](unsigned long long* rows) {
                    launch_count_temporal(F, bd, g, s->slot[psl].view, cg, cur, prev_st, wv, rows, stream);
                });
                for_row_cuts(bd, cuts, [&](const Band& sb) {
                    launch_temporal_wave(F, sb, g, s->slot[psl].view, gp, pc, cg, pg, f, cur, prev_st, wv,
                                         ctr + 0 * SC_COUNT, q, stream);
                });
            }
            else
                launch_temporal(F, bd, g, s->slot[psl].view, gp, pc, cg, pg, f, cur, store_of(s, s->res[s->prev], psl),
                                wo, ctr + 0 * SC_COUNT, q, stream);
        }
        cudaEventRecord(ev[2], stream);
        if (piped) cudaEventRecord(s->ev_temporal[set], stream);
        if (s->transient && c.bin_reuse) {
            reset_store(s, s->spare, stream);
            if (s->wave) {  // per pixel: no halo; 2 forward + 1 inverse job per item
                for_row_batches(bd, wave_batches(s, 3), [&](const Band& sb) {
                    launch_binreuse_wave(F, sb, g, pc, cg, f, cur, store_of(s, s->res[s->spare], sl), wv,
                                         ctr + 2 * SC_COUNT, q, stream);
                });
            } else {
                launch_binreuse(F, bd, g, pc, h, f, cur, store_of(s, s->res[s->spare], sl), ctr + 2 * SC_COUNT, q,
                                stream);
            }
            std::swap(s->cur, s->spare);
            cur = store_of(s, s->res[s->cur], sl);
        }
        cudaEventRecord(ev[3], stream);
        SpatialParams sp{c.spatial_neighbors, c.spatial_radius};
        // no neighbours or radius 0: spatial_reuse returns its input (pipeline.hpp:246),
        // so the passes are skipped (every rank agrees: same config)
        const int passes = (sp.neighbors > 0 && sp.radius > 0) ? c.spatial_passes : 0;
        for (int pass = 0; pass < passes; ++pass) {
            if (halo) exchange_halo(s, cur, pass);
            reset_store(s, s->spare, stream);
            SpatialScratch scr;
            const SpatialScratch* scp = nullptr;
            if (s->phased) {
                size_t own_items = s->owned_pixels() * s->B;
                scr.mapped = ResStore{s->sp_mapped.as<double2>(), own_items * size_t(c.spatial_neighbors)};
                scr.ok = s->sp_ok.as<uint8_t>();
                scr.rng_ctr = s->sp_rng.as<uint64_t>();
                scr.list = s->sp_list.as<uint32_t>();
                scr.count = s->sp_count.as<uint32_t>();
                scp = &scr;
            }
            if (s->wave && sp.neighbors > 0 && sp.radius > 0) {
                auto cuts = stage_cuts(s, bd, wave_jobs_per_item(sp.neighbors), stream, [&](unsigned long long* rows) {
                    launch_count_spatial(F, bd, pc, cg, sp, pass, f, cur, rows, stream);
                });
                for_row_cuts(bd, cuts, [&](const Band& sb) {
                    launch_spatial_wave(F, sb, g, pc, cg, sp, pass, f, cur, store_of(s, s->res[s->spare], sl), wv,
                                        ctr + 1 * SC_COUNT, q, stream);
                });
            } else
                launch_spatial(F, bd, g, pc, cg, sp, pass, f, cur, store_of(s, s->res[s->spare], sl), wo, scp,
                               ctr + 1 * SC_COUNT, q, stream);
            std::swap(s->cur, s->spare);
            cur = store_of(s, s->res[s->cur], sl);
        }
        cudaEventRecord(ev[4], stream);
        if (s->transient)
            launch_shade_transient(cur, bd, s->W, h, rows_base<double>(s->hist, s->y0, size_t(s->W) * s->B * 3),
                                   stream);
        else
            launch_shade_gated(cur, bd, s->W, center, width, pc.gate_vel, rows_base<double>(s->image, s->y0, size_t(s->W) * 3),
                               rows_base<double>(s->accum, s->y0, size_t(s->W) * 3), stream);
        // a moving camera reprojects across band edges: give the next
        // frame's temporal stage the neighbours' final reservoirs too
        if (prev_halo && c.temporal) exchange_halo(s, cur, -1);
        cudaEventRecord(ev[5], stream);
        if (s->xg >= 0) {  // bufs.flip() with a fourth grid: the next init writes frame f-2's final grid
            const int fin = s->cur;
            s->cur = s->xg;
            s->xg = s->prev;
            s->prev = fin;
        } else {
            std::swap(s->cur, s->prev);  // bufs.flip()
        }
    }
    ck(cudaMemcpyAsync(&s->err_host[set], ctr + 3 * SC_COUNT, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       stream),
       "flag");
    if (s->sparse)
        ck(cudaMemcpyAsync(s->occ_host + 8 * set, s->res_rows.p, 32, cudaMemcpyDeviceToHost,
                           stream),
           "occupancy");
    cudaEventRecord(ev[6], stream);
    ck(cudaGetLastError(), "kernel launch");
    s->pending[set] = true;
    s->prev_center = center;
    s->prev_width = width;
    s->f++;
    if (st) {
        flush_all(s);
        std::memset(st, 0, sizeof(*st));
        st->frame = f;
        unsigned long long hc[3 * SC_COUNT];
        ck(cudaMemcpy(hc, ctr, sizeof(hc), cudaMemcpyDeviceToHost), "counters");
        fill_counts(st->temporal.shift, hc + 0 * SC_COUNT);
        fill_counts(st->spatial.shift, hc + 1 * SC_COUNT);
        fill_counts(st->binwise.shift, hc + 2 * SC_COUNT);
        const double* ms = s->stage_ms;
        st->t_init = ms[0] * 1e-3;
        st->temporal.seconds = (c.temporal && f > 0) ? ms[1] * 1e-3 : 0;
        st->binwise.seconds = (s->transient && c.bin_reuse) ? ms[2] * 1e-3 : 0;
        st->spatial.seconds = ms[3] * 1e-3;
        st->t_shade = ms[4] * 1e-3;
    }
}

template <class F>
int guard(tofr_gpu* ctx, F&& fn) {
    try {
        if (ctx) ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        fn();
        if (ctx) ctx->err.clear();
        return TOFR_OK;
    } catch (const ScopeError& e) {
        if (ctx) ctx->err = e.what();
        return e.code;
    } catch (const CudaError& e) {
        if (ctx) ctx->err = e.what();
        return TOFR_ERR_CUDA;
    } catch (const std::bad_alloc& e) {
        if (ctx) ctx->err = "host allocation failed";
        return TOFR_ERR_OOM;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        return TOFR_ERR_SCENE;
    }
}

// Histogram of a session's owned rows in the reference's layout: rgb (3 f64 per
// bin) and, for plain sessions, the per-bin deposit counts (de-interleaved
// from the 32 B bin records).
void read_hist_records(tofr_session* s, double* rgb, std::vector<int64_t>* count) {
    size_t items = s->owned_pixels() * s->B;
    if (!s->plain) {
        ck(cudaMemcpy(rgb, s->hist.p, items * 24, cudaMemcpyDeviceToHost), "histogram");
        return;
    }
    std::vector<double> rec(items * 4);
    ck(cudaMemcpy(rec.data(), s->hist.p, rec.size() * 8, cudaMemcpyDeviceToHost), "histogram");
    if (count) count->resize(items);
    for (size_t i = 0; i < items; ++i) {
        rgb[3 * i + 0] = rec[4 * i + 0];
        rgb[3 * i + 1] = rec[4 * i + 1];
        rgb[3 * i + 2] = rec[4 * i + 2];
        if (count) {
            uint64_t c;
            std::memcpy(&c, &rec[4 * i + 3], 8);
            (*count)[i] = int64_t(c);
        }
    }
}

// Output of a (full-frame) session in RenderOutput form (pipeline.hpp:384-391,
// :516-527, :563-570).
void read_outputs(tofr_session* s, const tofr_render_config* cfg, tofr_output* out, bool plain) {
    flush_all(s);
    int frames = cfg->frames;
    size_t npix = s->owned_pixels();
    if (!s->transient) {
        std::vector<double> img(npix * 3);
        if (cfg->accumulate && frames > 0) {
            ck(cudaMemcpy(img.data(), s->accum.p, img.size() * 8, cudaMemcpyDeviceToHost), "image");
            double k = 1.0 / frames;
            for (double& v : img) v *= k;
        } else {
            ck(cudaMemcpy(img.data(), s->image.p, img.size() * 8, cudaMemcpyDeviceToHost), "image");
        }
        if (cfg->normalize_gate && cfg->gate_width > 0) {
            double k = 1.0 / cfg->gate_width;
            for (double& v : img) v *= k;
        }
        if (out->image) std::memcpy(out->image, img.data(), img.size() * 8);
        return;
    }
    size_t items = npix * s->B;
    std::vector<double> rgb(items * 3);
    std::vector<int64_t> cnt;
    read_hist_records(s, rgb.data(), plain ? &cnt : nullptr);
    double k = plain ? 1.0 / std::max(1, frames) : (frames > 0 ? 1.0 / double(frames) : 1.0);
    if (plain || frames > 0)
        for (double& v : rgb) v *= k;
    if (out->hist_rgb) std::memcpy(out->hist_rgb, rgb.data(), rgb.size() * 8);
    if (out->hist_count) {
        if (plain)
            std::memcpy(out->hist_count, cnt.data(), items * 8);
        else
            for (size_t i = 0; i < items; ++i) out->hist_count[i] = frames;
    }
    if (out->image) {
        for (size_t p = 0; p < npix; ++p) {
            double sx = 0, sy = 0, sz = 0;
            for (int b = 0; b < s->B; ++b) {
                const double* v = &rgb[3 * (p * s->B + b)];
                sx += v[0];
                sy += v[1];
                sz += v[2];
            }
            out->image[3 * p + 0] = sx;
            out->image[3 * p + 1] = sy;
            out->image[3 * p + 2] = sz;
        }
    }
}

void render_loop(tofr_gpu* ctx, const tofr_scene* sc, const tofr_render_config* cfg, tofr_output* out,
                 bool plain) {
    if (!ctx || !sc) throw ScopeError(TOFR_ERR_INVALID, "null handle");
    std::unique_ptr<tofr_session> s(make_session(ctx, sc, cfg, plain ? KIND_PLAIN : KIND_RESTIR));
    int frames = cfg->frames;
    for (int f = 0; f < frames; ++f) {
        tofr_frame_stats st;
        bool want = out && out->stats && f < out->stats_capacity;
        session_step(s.get(), want ? &st : nullptr);
        if (want) out->stats[f] = st;
    }
    if (!out) {
        flush_all(s.get());
        return;
    }
    read_outputs(s.get(), cfg, out, plain);
}

HScene scene_from_desc(const tofr_scene_desc* d) {
    if (!d) throw ScopeError(TOFR_ERR_INVALID, "null scene desc");
    HScene s;
    s.camera.base.position = {d->cam_position[0], d->cam_position[1], d->cam_position[2]};
    s.camera.base.forward = {d->cam_forward[0], d->cam_forward[1], d->cam_forward[2]};
    s.camera.base.up = {d->cam_up[0], d->cam_up[1], d->cam_up[2]};
    s.camera.fov_y = d->fov_y;
    s.camera.width = d->width;
    s.camera.height = d->height;
    for (int i = 0; i < d->n_cam_keys; ++i) {
        const tofr_camera_key& k = d->cam_keys[i];
        HCamPose p;
        p.position = {k.position[0], k.position[1], k.position[2]};
        p.forward = {k.forward[0], k.forward[1], k.forward[2]};
        p.up = {k.up[0], k.up[1], k.up[2]};
        s.camera.track.emplace_back(k.frame, p);
    }
    for (int i = 0; i < d->n_materials; ++i) {
        HMaterial m;
        m.kind = d->materials[i].kind;
        m.albedo = {d->materials[i].albedo[0], d->materials[i].albedo[1], d->materials[i].albedo[2]};
        m.roughness = d->materials[i].roughness;
        s.materials.push_back(m);
    }
    if (s.materials.empty()) s.materials.push_back(HMaterial{});
    const tofr_light& l = d->light;
    s.light.regime = l.regime;
    s.light.position = {l.position[0], l.position[1], l.position[2]};
    s.light.direction = {l.direction[0], l.direction[1], l.direction[2]};
    s.light.cone_half_angle = l.cone_half_angle;
    s.light.intensity = {l.intensity[0], l.intensity[1], l.intensity[2]};
    for (int i = 0; i < d->n_objects; ++i) {
        const tofr_object_desc& od = d->objects[i];
        HObject o;
        o.name = od.name ? od.name : "";
        for (int t = 0; t < od.n_tris; ++t) {
            const double* v = od.verts + 9 * size_t(t);
            int mat = od.materials ? od.materials[t] : 0;
            if (mat < 0 || mat >= int(s.materials.size())) throw ScopeError(TOFR_ERR_INVALID, "material index");
            o.local.push_back(make_tri({v[0], v[1], v[2]}, {v[3], v[4], v[5]}, {v[6], v[7], v[8]}, mat));
        }
        for (int k = 0; k < od.n_keys; ++k) {
            HPoseKey pk;
            pk.frame = od.keys[k].frame;
            pk.pose.q = {od.keys[k].q[0], od.keys[k].q[1], od.keys[k].q[2], od.keys[k].q[3]};
            pk.pose.t = {od.keys[k].t[0], od.keys[k].t[1], od.keys[k].t[2]};
            o.track.keys.push_back(pk);
        }
        s.objects.push_back(std::move(o));
    }
    s.dt_frame = d->dt_frame;
    return s;
}

}  // namespace

extern "C" {

void tofr_render_config_default(tofr_render_config* c) {
    if (!c) return;
    std::memset(c, 0, sizeof(*c));
    c->mode = TOFR_MODE_GATED;
    c->gate_kind = TOFR_GATE_LENGTH;
    c->gate_center = 0;
    c->gate_width = 1;
    c->gate_f0 = 1;
    c->gate_step = 0;
    c->bins = 1;
    c->hist_t0 = 0;
    c->hist_bin_width = 0;
    c->m_init = 8;
    c->init_mode = TOFR_INIT_DIRECT;
    c->shrink_k = 10;
    c->shrink_r = 1.0;
    c->spatial_passes = 0;
    c->spatial_neighbors = 5;
    c->spatial_radius = 10;
    c->temporal = 0;
    c->bin_reuse = 0;
    c->m_cap = 20;
    c->gauge = TOFR_GAUGE_AVG;
    c->newton = 1;
    c->seed = 1;
    c->frames = 1;
    c->frame0 = 0;
    c->max_depth = 6;
    c->use_rr = 1;
    c->accumulate = 0;
    c->normalize_gate = 0;
}

const char* tofr_gpu_version(void) { return "tofr_b200 0.1 sm_100a"; }

int tofr_gpu_create(const int* devices, int n_devices, tofr_gpu** out) {
    if (!out) return TOFR_ERR_INVALID;
    *out = nullptr;
    auto ctx = std::make_unique<tofr_gpu>();
    int rc = guard(ctx.get(), [&] {
        ctx->device = (devices && n_devices > 0) ? devices[0] : 0;
        ck(cudaSetDevice(ctx->device), "cudaSetDevice");
        {
            // the frame's critical path runs on this stream at the highest
            // priority: when a pipelined session's side stream (next frame's
            // path trees, default priority) competes for SM slots, the block
            // scheduler serves this stream's reuse kernels first
            // (TOFR_STREAM_PRIORITY=0: default priority)
            int least = 0, greatest = 0;
            const char* pe = std::getenv("TOFR_STREAM_PRIORITY");
            bool prio = !(pe && pe[0] == '0') && cudaDeviceGetStreamPriorityRange(&least, &greatest) == cudaSuccess;
            if (prio)
                ck(cudaStreamCreateWithPriority(&ctx->stream, cudaStreamNonBlocking, greatest), "stream");
            else
                ck(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "stream");
        }
        double x[32], w[32];
        gauss_rule32(x, w);
        set_gauss_rule(x, w, ctx->stream);
        ck(cudaStreamSynchronize(ctx->stream), "init");
    });
    if (rc != TOFR_OK) {
        static thread_local std::string last;
        last = ctx->err;
        std::fprintf(stderr, "tofr_gpu_create: %s\n", last.c_str());
        return rc;
    }
    *out = ctx.release();
    return TOFR_OK;
}

void tofr_gpu_destroy(tofr_gpu* ctx) {
    if (!ctx) return;
    if (ctx->live_sessions > 0) {
        ctx->closing = true;
        return;
    }
    release_ctx(ctx);
}

const char* tofr_gpu_last_error(const tofr_gpu* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

static int scene_guard(char* err, size_t errlen, const std::function<void()>& fn);

int tofr_scene_create(const tofr_scene_desc* desc, tofr_scene** out, char* err, size_t errlen) {
    if (!out) return TOFR_ERR_INVALID;
    *out = nullptr;
    return scene_guard(err, errlen, [&] {
        auto s = std::make_unique<tofr_scene>();
        s->s = scene_from_desc(desc);
        if (s->s.objects.empty()) throw ScopeError(TOFR_ERR_INVALID, "scene has no objects");
        *out = s.release();
    });
}

int tofr_scene_parse(const char* text, const char* base_dir, tofr_scene** out, char* err, size_t errlen) {
    if (!out || !text) return TOFR_ERR_INVALID;
    *out = nullptr;
    return scene_guard(err, errlen, [&] {
        auto s = std::make_unique<tofr_scene>();
        s->s = parse_scene_text(text, base_dir ? base_dir : ".");
        *out = s.release();
    });
}

int tofr_scene_load(const char* path, tofr_scene** out, char* err, size_t errlen) {
    if (!out || !path) return TOFR_ERR_INVALID;
    *out = nullptr;
    return scene_guard(err, errlen, [&] {
        auto s = std::make_unique<tofr_scene>();
        s->s = load_scene_file(path);
        *out = s.release();
    });
}

void tofr_scene_destroy(tofr_scene* s) { delete s; }

int tofr_scene_set_resolution(tofr_scene* s, int32_t width, int32_t height) {
    if (!s || width <= 0 || height <= 0) return TOFR_ERR_INVALID;
    s->s.camera.width = width;
    s->s.camera.height = height;
    return TOFR_OK;
}

int tofr_scene_info(const tofr_scene* s, int32_t* width, int32_t* height, int32_t* n_tris, int32_t* n_nodes,
                    double* diag, char* err, size_t errlen) {
    if (!s) return TOFR_ERR_INVALID;
    return scene_guard(err, errlen, [&] {
        HFrame f = build_frame(s->s, 0);
        if (width) *width = s->s.camera.width;
        if (height) *height = s->s.camera.height;
        if (n_tris) *n_tris = int32_t(f.tris.size());
        if (n_nodes) *n_nodes = int32_t(f.nodes.size());
        if (diag) *diag = f.diag;
    });
}

int tofr_scene_probe_rays_host(const tofr_scene* s, double frame, const double* rays, int32_t n, int32_t mode,
                               double* out_t, int32_t* out_tri, char* err, size_t errlen) {
    if (!s || n < 0) return TOFR_ERR_INVALID;
    return scene_guard(err, errlen, [&] {
        HFrame hf = build_frame(s->s, frame);
        PackedFrame pk = pack_frame(s->s, hf, 0);
        FrameView v = rebase_view(pk, pk.blob.data());
        for (int i = 0; i < n; ++i) {
            const double* r = rays + 8 * size_t(i);
            V3 o{r[0], r[1], r[2]}, d{r[3], r[4], r[5]};
            if (mode == 0) {
                Hit h;
                bool ok = trace_closest(v, o, d, r[6], r[7], h);
                out_t[i] = ok ? h.t : kInf;
                out_tri[i] = ok ? h.tri : -1;
            } else {
                out_tri[i] = occluded(v, o, d) ? 1 : 0;
                out_t[i] = 0;
            }
        }
    });
}

int tofr_scene_dump_bvh(const tofr_scene* s, double frame, int32_t cap_nodes, double* nodes, int32_t* node_parent,
                        int32_t* n_nodes, int32_t cap_tris, int32_t* tri_order, int32_t* n_tris, double* diag,
                        char* err, size_t errlen) {
    if (!s) return TOFR_ERR_INVALID;
    return scene_guard(err, errlen, [&] {
        HFrame f = build_frame(s->s, frame);
        if (n_nodes) *n_nodes = int32_t(f.nodes.size());
        if (n_tris) *n_tris = int32_t(f.tris.size());
        if (diag) *diag = f.diag;
        if (nodes && int(f.nodes.size()) <= cap_nodes) {
            for (size_t i = 0; i < f.nodes.size(); ++i) {
                const HNode& h = f.nodes[i];
                double* o = nodes + 11 * i;
                o[0] = h.lo.x;
                o[1] = h.lo.y;
                o[2] = h.lo.z;
                o[3] = h.hi.x;
                o[4] = h.hi.y;
                o[5] = h.hi.z;
                o[6] = h.tri_area;
                o[7] = h.left;
                o[8] = h.right;
                o[9] = h.first;
                o[10] = h.count;
                if (node_parent) node_parent[i] = h.parent;
            }
        }
        if (tri_order && int(f.tri_order.size()) <= cap_tris)
            for (size_t i = 0; i < f.tri_order.size(); ++i) tri_order[i] = f.tri_order[i];
    });
}

int tofr_gpu_dump_bvh_device(tofr_gpu* ctx, const tofr_scene* s, double frame, int32_t cap_nodes, double* nodes,
                             int32_t* node_parent, int32_t* n_nodes, int32_t cap_tris, int32_t* tri_order,
                             int32_t* n_tris, double* diag) {
    return guard(ctx, [&] {
        if (!ctx || !s) throw ScopeError(TOFR_ERR_INVALID, "null handle");
        HFrame f = build_frame(s->s, frame, false);
        DeviceBvh db;
        int nn = db.build(f.tris.data(), int(f.tris.size()), ctx->stream);
        if (n_nodes) *n_nodes = nn;
        if (n_tris) *n_tris = int32_t(f.tris.size());
        if (diag) *diag = f.diag;
        if (nodes && node_parent && tri_order && nn <= cap_nodes && int(f.tris.size()) <= cap_tris)
            db.dump(nodes, node_parent, tri_order, ctx->stream);
    });
}

int tofr_gpu_render_gated(tofr_gpu* ctx, const tofr_scene* s, const tofr_render_config* cfg, tofr_output* out) {
    return guard(ctx, [&] {
        if (cfg && cfg->mode == TOFR_MODE_TRANSIENT)
            throw ScopeError(TOFR_ERR_INVALID, "render_gated called with a transient config");
        render_loop(ctx, s, cfg, out, false);
    });
}

// render_doppler (pipeline.hpp:573-578): render_gated with the velocity gate
int tofr_gpu_render_doppler(tofr_gpu* ctx, const tofr_scene* s, const tofr_render_config* cfg, tofr_output* out) {
    return guard(ctx, [&] {
        if (!cfg) throw ScopeError(TOFR_ERR_INVALID, "null config");
        tofr_render_config c = *cfg;
        c.gate_kind = TOFR_GATE_VELOCITY;
        if (c.mode == TOFR_MODE_TRANSIENT) throw ScopeError(TOFR_ERR_INVALID, "render_doppler is a gated mode");
        render_loop(ctx, s, &c, out, false);
    });
}

int tofr_gpu_render_transient(tofr_gpu* ctx, const tofr_scene* s, const tofr_render_config* cfg,
                              tofr_output* out) {
    return guard(ctx, [&] {
        if (!cfg) throw ScopeError(TOFR_ERR_INVALID, "null config");
        tofr_render_config c = *cfg;
        c.mode = TOFR_MODE_TRANSIENT;
        render_loop(ctx, s, &c, out, false);
    });
}

int tofr_gpu_render_transient_plain(tofr_gpu* ctx, const tofr_scene* s, const tofr_render_config* cfg,
                                    tofr_output* out) {
    return guard(ctx, [&] { render_loop(ctx, s, cfg, out, true); });
}

int tofr_gpu_reference(tofr_gpu* ctx, const tofr_scene* sc, double frame, double gate_center, double gate_width,
                       int32_t spp, uint64_t seed, int32_t max_depth, double* mean, double* se) {
    return guard(ctx, [&] {
        if (!ctx || !sc || spp < 1) throw ScopeError(TOFR_ERR_INVALID, "bad arguments");
        tofr_render_config c;
        tofr_render_config_default(&c);
        c.max_depth = max_depth;
        c.seed = seed;
        std::unique_ptr<tofr_session> s(make_session(ctx, sc, &c, KIND_BARE));
        upload_frame(s.get(), 0, frame, 0, ctx->stream);
        size_t npix = size_t(s->W) * s->H;
        DevBuf dm, ds;
        dm.ensure(npix * 3 * 8);
        ds.ensure(npix * 3 * 8);
        const FrameView& F = s->slot[0].view;
        GHit* g = s->slot[0].gbuf.as<GHit>();
        Band bd = band_of(s.get(), false);
        launch_gbuffer(F, bd, g, ctx->stream);
        PathCfg pc = path_cfg(c, gate_center, gate_width, s->scene);
        pc.ellipsoidal = 0;
        launch_reference(F, bd, g, pc, gate_center, gate_width, spp, uint64_t(frame), dm.as<double>(), ds.as<double>(),
                         s->ctr.as<unsigned long long>() + 3 * SC_COUNT + 1, ctx->stream);
        ck(cudaGetLastError(), "reference launch");
        if (mean) ck(cudaMemcpyAsync(mean, dm.p, npix * 24, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
        if (se) ck(cudaMemcpyAsync(se, ds.p, npix * 24, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
        ck(cudaStreamSynchronize(ctx->stream), "reference");
    });
}

int tofr_gpu_session_create(tofr_gpu* ctx, const tofr_scene* s, const tofr_render_config* cfg,
                            tofr_session** out) {
    return tofr_gpu_session_create_band(ctx, s, cfg, 0, -1, 0, out);
}

int tofr_gpu_session_create_band(tofr_gpu* ctx, const tofr_scene* s, const tofr_render_config* cfg, int32_t y0,
                                 int32_t y1, int32_t halo, tofr_session** out) {
    if (!out) return TOFR_ERR_INVALID;
    *out = nullptr;
    return guard(ctx, [&] {
        if (!ctx || !s) throw ScopeError(TOFR_ERR_INVALID, "null handle");
        if (cfg && cfg->mode == TOFR_MODE_TRANSIENT && cfg->bins < 1)
            throw ScopeError(TOFR_ERR_INVALID, "transient needs bins >= 1");
        *out = make_session(ctx, s, cfg, KIND_RESTIR, y0, y1, halo);
    });
}

int tofr_gpu_session_create_plain(tofr_gpu* ctx, const tofr_scene* s, const tofr_render_config* cfg, int32_t y0,
                                  int32_t y1, tofr_session** out) {
    if (!out) return TOFR_ERR_INVALID;
    *out = nullptr;
    return guard(ctx, [&] {
        if (!ctx || !s) throw ScopeError(TOFR_ERR_INVALID, "null handle");
        *out = make_session(ctx, s, cfg, KIND_PLAIN, y0, y1, 0);
    });
}

int tofr_gpu_session_band(tofr_session* ss, int32_t* y0, int32_t* y1, int32_t* r0, int32_t* r1) {
    if (!ss) return TOFR_ERR_INVALID;
    if (y0) *y0 = ss->y0;
    if (y1) *y1 = ss->y1;
    if (r0) *r0 = ss->r0;
    if (r1) *r1 = ss->r1;
    return TOFR_OK;
}

int tofr_gpu_session_set_halo_exchange(tofr_session* ss, tofr_halo_exchange_fn fn, void* user) {
    if (!ss) return TOFR_ERR_INVALID;
    ss->xfn = fn;
    ss->xuser = user;
    return TOFR_OK;
}

int tofr_gpu_nccl_unique_id(uint8_t* id) {
    if (!id) return TOFR_ERR_INVALID;
    if (!nccl_available()) return TOFR_ERR_UNSUPPORTED;
    try {
        nccl_unique_id(id);
    } catch (const std::exception&) {
        return TOFR_ERR_CUDA;
    }
    return TOFR_OK;
}

int tofr_gpu_session_halo_nccl(tofr_session* ss, const uint8_t* id, int32_t rank, int32_t world) {
    if (!ss || !id) return TOFR_ERR_INVALID;
    return guard(ss->ctx, [&] {
        if (!nccl_available()) throw ScopeError(TOFR_ERR_UNSUPPORTED, "libnccl.so.2 not loadable");
        // rank g's band lies above rank g+1's: a halo side needs a neighbour rank
        if ((ss->r0 < ss->y0 && rank == 0) || (ss->r1 > ss->y1 && rank == world - 1))
            throw ScopeError(TOFR_ERR_INVALID, "halo_nccl: the band keeps a halo on a side without a neighbour rank");
        ss->xport = make_nccl_transport(id, rank, world, ss->ctx->device);
    });
}

int tofr_gpu_session_link_halo(tofr_session* upper, tofr_session* lower) {
    if (!upper || !lower || upper == lower) return TOFR_ERR_INVALID;
    return guard(upper->ctx, [&] {
        if (upper->y1 != lower->y0 || upper->W != lower->W || upper->B != lower->B)
            throw ScopeError(TOFR_ERR_INVALID, "link_halo: the bands are not adjacent (upper.y1 != lower.y0)");
        if ((upper->r1 - upper->y1) != (lower->y0 - lower->r0))
            throw ScopeError(TOFR_ERR_INVALID, "link_halo: the bands keep different halos");
        for (tofr_session* s : {upper, lower})
            if (!s->peer) {
                s->peer = make_peer_endpoint(halo_bufs(s));
                s->xport = make_peer_transport(s->peer);
            }
        peer_link(upper->peer, lower->peer);
    });
}

int tofr_gpu_session_halo_transport(tofr_session* ss, const char** name) {
    if (!ss || !name) return TOFR_ERR_INVALID;
    *name = ss->xport ? ss->xport->name() : (ss->xfn ? "callback" : "none");
    return TOFR_OK;
}

int tofr_gpu_session_halo_buffers(tofr_session* ss, void** send_lo, void** recv_lo, uint64_t* bytes_lo,
                                  void** send_hi, void** recv_hi, uint64_t* bytes_hi) {
    if (!ss) return TOFR_ERR_INVALID;
    if (send_lo) *send_lo = ss->send_lo.p;
    if (recv_lo) *recv_lo = ss->recv_lo.p;
    if (bytes_lo) *bytes_lo = ss->send_lo.n;
    if (send_hi) *send_hi = ss->send_hi.p;
    if (recv_hi) *recv_hi = ss->recv_hi.p;
    if (bytes_hi) *bytes_hi = ss->send_hi.n;
    return TOFR_OK;
}

int tofr_gpu_session_step(tofr_session* ss, tofr_frame_stats* stats) {
    if (!ss) return TOFR_ERR_INVALID;
    return guard(ss->ctx, [&] { session_step(ss, stats); });
}

namespace {
}  // namespace

int tofr_gpu_session_read_image_async(tofr_session* ss, double* pinned_image, int32_t slot) {
    if (!ss || !pinned_image || slot < 0 || slot > 1) return TOFR_ERR_INVALID;
    return guard(ss->ctx, [&] {
        cudaStream_t st = ss->ctx->stream;
        size_t bytes = ss->owned_pixels() * 24;
        DevBuf& stage = ss->read_stage[slot];
        stage.ensure(bytes);
        // the slot's previous host copy must be done before its staging buffer is rewritten
        ck(cudaStreamWaitEvent(st, ss->read_ev[slot], 0), "wait");
        if (ss->plain) {
            // wide-band image accumulated by the deposits, / frames
            double scale = ss->f > 0 ? 1.0 / double(ss->f) : 1.0;
            launch_scale3(ss->accum.as<double>(), ss->owned_pixels(), scale, stage.as<double>(), st);
            ck(cudaGetLastError(), "image scale");
        } else if (ss->transient) {
            // wide-band image of the histogram accumulated so far, / frames
            Band bd = band_of(ss, false);
            double scale = ss->f > 0 ? 1.0 / double(ss->f) : 1.0;
            launch_hist_image(rows_base<double>(ss->hist, ss->y0, size_t(ss->W) * ss->B * 3), bd, ss->W, ss->B,
                              scale, rows_base<double>(stage, ss->y0, size_t(ss->W) * 3), st);
            ck(cudaGetLastError(), "hist image");
        } else {
            launch_copy_f64(ss->image.as<double>(), bytes / 8, stage.as<double>(), st);
            ck(cudaGetLastError(), "image copy");
        }
        ck(cudaEventRecord(ss->staged_ev[slot], st), "event");
        ck(cudaStreamWaitEvent(ss->copy_stream, ss->staged_ev[slot], 0), "wait");
        ck(cudaMemcpyAsync(pinned_image, stage.p, bytes, cudaMemcpyDeviceToHost, ss->copy_stream), "d2h");
        ck(cudaEventRecord(ss->read_ev[slot], ss->copy_stream), "event");
    });
}

int tofr_gpu_session_wait_read(tofr_session* ss, int32_t slot) {
    if (!ss || slot < 0 || slot > 1) return TOFR_ERR_INVALID;
    return guard(ss->ctx, [&] { ck(cudaEventSynchronize(ss->read_ev[slot]), "read-back"); });
}

int tofr_gpu_session_read_image(tofr_session* ss, double* image) {
    if (!ss || !image) return TOFR_ERR_INVALID;
    return guard(ss->ctx, [&] {
        if (ss->plain) {
            size_t npix = ss->owned_pixels();
            ss->image.ensure(npix * 3 * sizeof(double));
            double scale = ss->f > 0 ? 1.0 / double(ss->f) : 1.0;
            launch_scale3(ss->accum.as<double>(), npix, scale, ss->image.as<double>(), ss->ctx->stream);
            ck(cudaGetLastError(), "image scale");
        } else if (ss->transient) {
            // wide-band image of the histogram accumulated so far, / frames
            size_t npix = ss->owned_pixels();
            ss->image.ensure(npix * 3 * sizeof(double));
            Band bd = band_of(ss, false);
            double scale = ss->f > 0 ? 1.0 / double(ss->f) : 1.0;
            launch_hist_image(rows_base<double>(ss->hist, ss->y0, size_t(ss->W) * ss->B * 3), bd, ss->W, ss->B,
                              scale, rows_base<double>(ss->image, ss->y0, size_t(ss->W) * 3), ss->ctx->stream);
            ck(cudaGetLastError(), "hist image");
        }
        ck(cudaMemcpyAsync(image, ss->image.p, ss->owned_pixels() * 24, cudaMemcpyDeviceToHost, ss->ctx->stream),
           "d2h");
        flush_all(ss);
    });
}

int tofr_gpu_session_read_histogram(tofr_session* ss, double* rgb, int64_t* count) {
    if (!ss) return TOFR_ERR_INVALID;
    return guard(ss->ctx, [&] {
        if (!ss->transient) throw ScopeError(TOFR_ERR_UNSUPPORTED, "read_histogram on a gated session");
        flush_all(ss);
        size_t items = ss->owned_pixels() * ss->B;
        double k = ss->f > 0 ? 1.0 / double(ss->f) : 1.0;
        std::vector<double> tmp;
        if (!rgb) tmp.resize(items * 3);
        std::vector<int64_t> cnt;
        read_hist_records(ss, rgb ? rgb : tmp.data(), (count && ss->plain) ? &cnt : nullptr);
        if (rgb)
            for (size_t i = 0; i < items * 3; ++i) rgb[i] *= k;
        if (count) {
            if (ss->plain)
                std::memcpy(count, cnt.data(), items * 8);
            else
                for (size_t i = 0; i < items; ++i) count[i] = ss->f;
        }
    });
}

int tofr_gpu_session_sync(tofr_session* ss) {
    if (!ss) return TOFR_ERR_INVALID;
    return guard(ss->ctx, [&] {
        flush_all(ss);
        ck(cudaStreamSynchronize(ss->ctx->stream), "sync");
    });
}

int tofr_gpu_session_last_ms(tofr_session* ss, double* total_ms, double* stage_ms) {
    if (!ss) return TOFR_ERR_INVALID;
    return guard(ss->ctx, [&] {
        flush_all(ss);
        if (total_ms) *total_ms = ss->stage_ms[5];
        if (stage_ms)
            for (int i = 0; i < 6; ++i) stage_ms[i] = ss->stage_ms[i];
    });
}

int tofr_gpu_session_stage_totals(tofr_session* ss, double* stage_ms, int64_t* frames, uint64_t* halo_exchanges,
                                  int32_t reset) {
    if (!ss) return TOFR_ERR_INVALID;
    return guard(ss->ctx, [&] {
        flush_all(ss);
        if (stage_ms)
            for (int i = 0; i < 6; ++i) stage_ms[i] = ss->stage_tot[i];
        if (frames) *frames = ss->tot_frames;
        if (halo_exchanges) *halo_exchanges = ss->halo_exchanges;
        if (reset) {
            for (double& v : ss->stage_tot) v = 0;
            ss->tot_frames = 0;
            ss->halo_exchanges = 0;
        }
    });
}

int tofr_gpu_session_stream(tofr_session* ss, void** stream) {
    if (!ss || !stream) return TOFR_ERR_INVALID;
    *stream = static_cast<void*>(ss->ctx->stream);
    return TOFR_OK;
}

int tofr_gpu_session_io_bytes(tofr_session* ss, uint64_t* h2d_per_step, uint64_t* d2h_image) {
    if (!ss) return TOFR_ERR_INVALID;
    if (h2d_per_step) *h2d_per_step = ss->last_h2d;
    if (d2h_image) *d2h_image = uint64_t(ss->owned_pixels()) * 3 * sizeof(double);
    return TOFR_OK;
}

int tofr_gpu_session_row_cost(tofr_session* ss, int32_t enable, uint64_t* out) {
    if (!ss) return TOFR_ERR_INVALID;
    return guard(ss->ctx, [&] {
        flush_all(ss);
        size_t H = size_t(ss->H);
        if (out) {
            std::vector<unsigned long long> h(H, 0);
            if (ss->row_cost.p) ck(cudaMemcpy(h.data(), ss->row_cost.p, H * 8, cudaMemcpyDeviceToHost), "row cost");
            for (size_t y = 0; y < H; ++y) out[y] = h[y];
        }
        if (enable) {
            ss->row_cost.ensure(H * 8);
            ck(cudaMemset(ss->row_cost.p, 0, H * 8), "memset");
        }
        ss->row_cost_on = enable != 0;
    });
}

int tofr_gpu_session_pool(tofr_session* ss, uint64_t* rows_used, uint64_t* rows_cap) {
    if (!ss || !rows_used || !rows_cap) return TOFR_ERR_INVALID;
    return guard(ss->ctx, [&] {
        flush_all(ss);
        unsigned int r[3] = {0, 0, 0};
        if (ss->sparse) ck(cudaMemcpy(r, ss->res_rows.p, sizeof(r), cudaMemcpyDeviceToHost), "pool");
        for (int k = 0; k < 3; ++k) rows_used[k] = r[k];
        *rows_cap = ss->sparse ? ss->pool_rows : 0;
    });
}

int tofr_gpu_session_work(tofr_session* ss, uint64_t* out) {
    if (!ss || !out) return TOFR_ERR_INVALID;
    return guard(ss->ctx, [&] {
        flush_all(ss);
        unsigned long long w[WK_COUNT];
        ck(cudaMemcpy(w, ss->ctr.as<unsigned long long>() + 3 * SC_COUNT + 2, sizeof(w), cudaMemcpyDeviceToHost),
           "work");
        out[0] = w[WK_JOBS];
        out[1] = w[WK_CLOSEST] + ss->camera_rays;
        out[2] = w[WK_ANY];
        out[3] = w[WK_DEPOSITS];
        out[4] = w[WK_MERGES];
    });
}

void tofr_gpu_session_destroy(tofr_session* ss) { delete ss; }

int tofr_gpu_kernel_timing(int32_t enable) {
    bool prev = kt_enabled();
    if (!enable) kt_collect();
    kt_set_enabled(enable != 0);
    return prev ? 1 : 0;
}

uint64_t tofr_gpu_kernel_launches(void) { return kt_launches(); }

int tofr_gpu_kernel_times(char* names, int32_t name_len, double* total_ms, uint64_t* launches, int32_t cap) {
    kt_collect();
    return kt_read(names, name_len, total_ms, launches, cap);
}

uint64_t tofr_fnv1a64(const void* data, uint64_t n) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

void tofr_gpu_kernel_times_reset(void) {
    kt_collect();
    kt_reset();
}

int tofr_gpu_selftest_div(tofr_gpu* ctx, uint64_t n, uint64_t seed, uint64_t* mismatches) {
    return guard(ctx, [&] {
        if (!ctx || !mismatches) throw ScopeError(TOFR_ERR_INVALID, "bad arguments");
        DevBuf d;
        d.ensure(8);
        ck(cudaMemsetAsync(d.p, 0, 8, ctx->stream), "memset");
        launch_selftest_div(n, seed, d.as<unsigned long long>(), ctx->stream);
        ck(cudaMemcpyAsync(mismatches, d.p, 8, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
        ck(cudaStreamSynchronize(ctx->stream), "selftest");
    });
}

int tofr_gpu_debug_solve_profile(uint64_t* out, uint64_t cap, uint64_t* n) {
    if (!n) return TOFR_ERR_INVALID;
    size_t m = 0;
    bool ok = debug_solve_profile(reinterpret_cast<unsigned long long*>(out), size_t(cap), &m);
    *n = m;
    return ok ? TOFR_OK : TOFR_ERR_UNSUPPORTED;
}

int tofr_gpu_debug_check_selftest(tofr_gpu* ctx, int32_t* checked) {
    return guard(ctx, [&] {
        if (!ctx || !checked) throw ScopeError(TOFR_ERR_INVALID, "bad arguments");
        DevBuf out;
        out.ensure(sizeof(unsigned long long));
        *checked = launch_check_selftest(out.as<unsigned long long>(), ctx->stream);
        ck(cudaStreamSynchronize(ctx->stream), "check selftest");
        unsigned long long v = 0;
        ck(cudaMemcpy(&v, out.p, sizeof(v), cudaMemcpyDeviceToHost), "check selftest");
        if (v != 5) throw ScopeError(TOFR_ERR_CUDA, "check selftest: unexpected row");
    });
}

int tofr_gpu_fp64_peak(tofr_gpu* ctx, double* gflops) {
    return guard(ctx, [&] {
        if (!ctx || !gflops) throw ScopeError(TOFR_ERR_INVALID, "bad arguments");
        *gflops = measure_fp64_peak_gflops(ctx->stream);
        ck(cudaGetLastError(), "fp64 peak");
    });
}

int tofr_gpu_probe_rays(tofr_gpu* ctx, const tofr_scene* sc, double frame, const double* rays, int32_t n,
                        int32_t mode, double* out_t, int32_t* out_tri) {
    return guard(ctx, [&] {
        if (!ctx || !sc || n < 0) throw ScopeError(TOFR_ERR_INVALID, "bad arguments");
        tofr_render_config c;
        tofr_render_config_default(&c);
        std::unique_ptr<tofr_session> s(make_session(ctx, sc, &c, KIND_BARE));
        upload_frame(s.get(), 0, frame, 0, ctx->stream);
        if (n == 0) {
            ck(cudaStreamSynchronize(ctx->stream), "probe");
            return;
        }
        DevBuf dr, dt, di;
        dr.ensure(size_t(n) * 64);
        dt.ensure(size_t(n) * 8);
        di.ensure(size_t(n) * 4);
        ck(cudaMemcpyAsync(dr.p, rays, size_t(n) * 64, cudaMemcpyHostToDevice, ctx->stream), "h2d");
        launch_probe_rays(s->slot[0].view, dr.as<double>(), n, mode, dt.as<double>(), di.as<int>(), ctx->stream);
        ck(cudaGetLastError(), "probe launch");
        ck(cudaMemcpyAsync(out_t, dt.p, size_t(n) * 8, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
        ck(cudaMemcpyAsync(out_tri, di.p, size_t(n) * 4, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
        ck(cudaStreamSynchronize(ctx->stream), "probe");
    });
}

}  // extern "C"

static int scene_guard(char* err, size_t errlen, const std::function<void()>& fn) {
    try {
        fn();
        set_err(err, errlen, "");
        return TOFR_OK;
    } catch (const tofr_b200::ParseError& e) {
        set_err(err, errlen, std::to_string(e.line) + ":" + std::to_string(e.col) + ": " + e.what());
        return TOFR_ERR_PARSE;
    } catch (const ScopeError& e) {
        set_err(err, errlen, e.what());
        return e.code;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return TOFR_ERR_SCENE;
    }
}
