// tofr_kernels.h -- host-visible launch interface of the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include "tofr_path.cuh"
#include "tofr_store.cuh"

namespace tofr_b200 {

// Per-frame traversal arrays above this size stay in global memory.
constexpr size_t kSmemStageLimit = 20 * 1024;

enum : int { INIT_DIRECT = 0, INIT_ELLIPSOIDAL = 1, INIT_SHRINK = 2 };

// Wavefront ellipsoidal sampling scratch (tofr_ellipsoid.cuh: plan -> arcs ->
// replay).  Per band pixel `per_pixel` slots, slot k = the pixel's k-th
// connection-vertex sampler call.
struct EllJob {
    V2 center, ax1, ax2;
    double r1, r2;
    double t0[6], t1[6];
    double u;     // the arc draw (sample_arc's rng_next)
    double p_dt;  // p_desc * p_tri
    int nseg, tri;
};
struct EllRes {
    V3 pos;
    double pdf_arc;
};
struct EllScratch {
    EllJob* jobs;
    EllRes* res;
    uint8_t* st;      // 1: job recorded (the clip kept a segment), 0: the sampler failed
    uint64_t* ctr;    // ellipsoid RNG counter after the sampler call
    uint32_t* list;   // slots with a job
    unsigned int* count;
    int per_pixel;
};
// bytes of scratch per slot (EllScratch)
constexpr size_t kEllSlotBytes = sizeof(EllJob) + sizeof(EllRes) + 1 + 8 + 4;

struct InitParams {
    int mode;
    int m_init;
    double center, width;  // gate of this frame
    double shrink_k, shrink_r;
};

// Gate per reservoir item: one gate (gated) or the bin gates (transient).
struct GateGrid {
    int transient;
    double center, width;
    HistSpec h;
};

// Row band of a session (parallel.py): the kernels compute rows [y0, y1) of
// the image; reservoir grids and G-buffers store rows [r0, r1) (the band plus
// the spatial halo).  Device pointers handed to the kernels are rebased so
// that they are indexed by GLOBAL pixel / item numbers (RNG keys and
// neighbour arithmetic stay those of the full frame, pipeline.hpp:102).
// Temporal reuse may read the previous grid on rows [t0, t1).  A read outside
// the stored rows raises *err (the host turns it into an error).
struct Band {
    int y0, y1, r0, r1, t0, t1;
    unsigned long long* err;
};

// Cost-ordered processing of the reuse kernels (see k_cost_* in the .cu):
// per-item cost class, bucket counters/cursors [16], the permutation.
// perm == nullptr processes items in storage order.
struct WorkOrder {
    uint8_t* cls;
    uint32_t* counts;
    uint32_t* perm;
};

// Scratch of the phased spatial pass (k_spatial_fwd_list / k_spatial_fwd /
// k_spatial_merge): forward-shifted samples of every (neighbour j, item i)
// job, their usable flags, the running lane-10 RNG position, the job list.
struct SpatialScratch {
    ResStore mapped;    // item j * n + i (jac in the W slot), stride N * n
    uint8_t* ok;        // [N * n]
    uint64_t* rng_ctr;  // [n]
    uint32_t* list;     // [N * n]
    uint32_t* count;    // [1]
};

struct SpatialParams {
    int neighbors;
    double radius;
};

// ---------------------------------------------------------------------------
// Wavefront shift engine (tofr_wave.cu).  A shift job maps the sample stored
// at (store, item) from a source domain (frame, pixel, gate centre) into a
// destination domain (frame, pixel, gate centre and width) -- shift_sample,
// shiftmap.hpp:662-783.  Stages append jobs to a compacted queue; two kernels
// run the shifts (k_shift_solve: record, prefix, suffix and the Newton solve;
// k_shift_finish: occlusion, Jacobian, rebuild); the stage's merge kernel then
// reads the per-job outputs.
constexpr int kJobChunks = 14;
enum : uint32_t {
    JOB_REC1 = 1u,    // source record lives in store 1 (else store 0)
    JOB_SRC1 = 2u,    // source domain is frame 1 (else frame 0)
    JOB_DST1 = 4u,    // destination domain is frame 1
    JOB_FULL = 8u,    // output the mapped record (else only p-hat of the source gate)
    JOB_COUNT = 16u,  // accumulate the shift counters (forward shifts)
    // shrink_map (shiftmap.hpp:789-876) instead of shift_sample: same pixel and
    // frame, Newton target L0 + (len - L0) / K (JOB_FULL: forward) or * K
    // (inverse) with L0 = the job's dc, Jacobian * 1/K or * K after the clamp,
    // inverse p-hat on the K-times wider gate
    JOB_SHRINK = 32u,
};
constexpr uint32_t kNoJob = 0xffffffffu;

struct ShiftQueue {
    double2* jobs;  // chunk-major job records: chunk c of job k at jobs[c * cap + k]
    size_t cap;
    // Per-job output, indexed by job id.  Chunk 0 = (value, ok): value is the
    // Jacobian (JOB_FULL) or p-hat_src(S^-1 y) * |J| (otherwise), ok = 1 when the
    // shift succeeded.  JOB_FULL jobs also get the mapped record in chunks 1-21.
    ResStore out;
    uint32_t* ctl;  // [0] first job of the current batch, [1] end, [2] mark, [3] merge-list length
    // solve -> finish overlap (TOFR_OVERLAP): the solve marks job k done with
    // the batch's epoch after its hand-off is written; the finish, running
    // concurrently on a second stream, waits for the mark (null: no overlap)
    uint32_t* done = nullptr;
    uint32_t epoch = 0;
};

// host side of the solve / finish overlap
struct ShiftOverlap {
    unsigned long long* fin_ctr = nullptr;  // the finish kernel's work counter (null: no overlap)
    uint32_t* epoch = nullptr;              // host counter of shift batches
};

struct WaveScratch {
    ShiftQueue q;
    uint32_t* map_a;    // spatial: forward job of (j, i) [N * n]; temporal: forward job of i [n]
    uint32_t* map_b;    // spatial: inverse job of i [n]; temporal: inverse job of i [n]
    uint64_t* tsrc;     // temporal: reprojected source pixel of each band pixel, or ~0
    uint64_t* rng_ctr;  // spatial: lane-10 RNG position per item
    uint32_t* mlist;    // items whose merge has a non-empty side (count in q.ctl[3])
    uint32_t* nbr;      // spatial: neighbor_offset of (j, band pixel) for the pass [N * pixels]
    ShiftOverlap ov;    // host only
};

// jobs per item a stage can enqueue (capacity planning)
inline size_t wave_jobs_per_item(int neighbors) { return size_t(neighbors > 1 ? neighbors + 1 : 2); }

// per-row upper bounds of a stage's shift jobs (adaptive row batches)
void launch_count_temporal(const FrameView& Fc, const Band& bd, const GHit* gc, const FrameView& Fp,
                           const GateGrid& cg, ResStore cur, ResStore prev, const WaveScratch& ws,
                           unsigned long long* rows, cudaStream_t s);
void launch_count_spatial(const FrameView& F, const Band& bd, const PathCfg& cfg, const GateGrid& gg,
                          const SpatialParams& sp, int pass, int frame_idx, ResStore src, unsigned long long* rows,
                          cudaStream_t s);
void launch_temporal_wave(const FrameView& Fc, const Band& bd, const GHit* gc, const FrameView& Fp, const GHit* gp,
                          const PathCfg& cfg, const GateGrid& cg, const GateGrid& pg, int frame_idx, ResStore cur,
                          ResStore prev, const WaveScratch& ws, unsigned long long* ctr, unsigned long long* q,
                          cudaStream_t s);
void launch_spatial_wave(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, const GateGrid& gg,
                         const SpatialParams& sp, int pass, int frame_idx, ResStore src, ResStore dst,
                         const WaveScratch& ws, unsigned long long* ctr, unsigned long long* q, cudaStream_t s);

// Path-tree tracing as a per-lane state machine (tofr_trace.cu): direct
// initial sampling (gated / transient), plain transient deposits, the brute-
// force reference.  The launchers below route to these unless the ellipsoidal
// or shrink initialiser is selected (or TOFR_TRACE=legacy).
void launch_trace_gated(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, int m_init,
                        double center, double width, int frame_idx, ResStore cur, unsigned long long* q,
                        cudaStream_t s);
void launch_trace_transient(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, int m_init,
                            const HistSpec& h, int frame_idx, ResStore cur, unsigned long long* q, cudaStream_t s);
// plain deposits into 32 B bin records {r, g, b, count} (hist) and the per-pixel
// wide-band accumulator img (3 doubles per pixel; may be null)
void launch_trace_plain(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, const HistSpec& h,
                        int m_init, int frame_idx, double* hist, double* img, unsigned long long* q,
                        cudaStream_t s);
void launch_trace_reference(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, double center,
                            double width, int spp, uint64_t frame_key, double* mean, double* se,
                            unsigned long long* q, cudaStream_t s);

size_t frame_smem_bytes(const FrameView& F);
void set_gauss_rule(const double* x, const double* w, cudaStream_t s);
// g (launch_gbuffer) is the band's local G-buffer (row r0 first); every other
// G-buffer / grid / image pointer is global-indexed (see Band).
void launch_gbuffer(const FrameView& F, const Band& bd, GHit* g, cudaStream_t s);
// The path kernels below are persistent with dynamic work distribution; `q`
// is one device u64 of the caller's (zeroed by the launcher, stream-ordered).
void launch_init_gated(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg,
                       const InitParams& ip, int frame_idx, ResStore cur, unsigned long long* q, cudaStream_t s, const EllScratch* es = nullptr);
void launch_init_transient(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg,
                           const InitParams& ip, const HistSpec& h, int frame_idx, ResStore cur,
                           unsigned long long* q, cudaStream_t s);
void launch_temporal(const FrameView& Fc, const Band& bd, const GHit* gc, const FrameView& Fp, const GHit* gp,
                     const PathCfg& cfg, const GateGrid& cg, const GateGrid& pg, int frame_idx,
                     ResStore cur, ResStore prev, const WorkOrder& wo, unsigned long long* ctr,
                     unsigned long long* q, cudaStream_t s);
void launch_spatial(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, const GateGrid& gg,
                    const SpatialParams& sp, int pass, int frame_idx, ResStore src, ResStore dst,
                    const WorkOrder& wo, const SpatialScratch* sc, unsigned long long* ctr, unsigned long long* q,
                    cudaStream_t s);
// bin reuse on the wavefront shift engine (tofr_wave.cu); src / dst: the stage's
// input and output grids
void launch_binreuse_wave(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, const GateGrid& gg,
                          int frame_idx, ResStore src, ResStore dst, const WaveScratch& ws, unsigned long long* ctr,
                          unsigned long long* q, cudaStream_t s);
// shrink initialiser on the wavefront engine: the two RIS runs (k_trace, the
// pick stream's counter carried in pick_in / pick_out), then the shrink_map
// jobs and the per-pixel merge into `fine` (tofr_wave.cu)
void launch_trace_gated_ris(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, int trees,
                            double center, double width, int frame_idx, ResStore cur, const uint64_t* pick_in,
                            uint64_t* pick_out, unsigned long long* q, cudaStream_t s);
void launch_shrink_wave(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, double center,
                        double width, int m_fine, int frame_idx, ResStore rough, ResStore fine,
                        const uint64_t* pick_ctr, const WaveScratch& ws, unsigned long long* ctr,
                        unsigned long long* q, cudaStream_t s);
void launch_binreuse(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, const HistSpec& h,
                     int frame_idx, ResStore src, ResStore dst, unsigned long long* ctr, unsigned long long* q,
                     cudaStream_t s);
void launch_shade_gated(ResStore cur, const Band& bd, int W, double center, double width, int gate_vel,
                        double* image, double* accum, cudaStream_t s);
void launch_shade_transient(ResStore cur, const Band& bd, int W, const HistSpec& h, double* hist,
                            cudaStream_t s);
void launch_hist_plain(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, const HistSpec& h,
                       int m_init, int frame_idx, double* hist, double* img, unsigned long long* q,
                       cudaStream_t s);
void launch_copy_f64(const double* a, size_t n, double* out, cudaStream_t s);  // 16 B aligned
void launch_scale3(const double* a, size_t n_pixels, double scale, double* out, cudaStream_t s);
void launch_reference(const FrameView& F, const Band& bd, const GHit* g, const PathCfg& cfg, double center,
                      double width, int spp, uint64_t frame_key, double* mean, double* se, unsigned long long* q,
                      cudaStream_t s);
// wide-band image (sum over bins x scale) of a global-indexed histogram
void launch_hist_image(const double* hist, const Band& bd, int W, int B, double scale, double* image,
                       cudaStream_t s);
// halo staging: rows [a, b) of a global-indexed grid <-> a contiguous buffer
// laid out chunk-major ([kResChunks][(b - a) * W * B] x 16 B)
// halo rows of a grid: dense grids as n_items x 24 chunks; sparse grids
// compacted (headers + the non-empty reservoirs' rows, at most `cap` of them)
size_t halo_bytes(size_t n_items, size_t cap, bool sparse);
void launch_halo_pack(ResStore grid, size_t item0, size_t n_items, double2* buf, size_t cap, cudaStream_t s);
void launch_halo_unpack(ResStore grid, size_t item0, size_t n_items, const double2* buf, size_t cap,
                        cudaStream_t s);
void launch_selftest_div(uint64_t n, uint64_t seed, unsigned long long* bad, cudaStream_t s);
// measured FP64 DFMA throughput of this device (GFLOP/s, 2 flops per DFMA)
double measure_fp64_peak_gflops(cudaStream_t s);
bool debug_solve_profile(unsigned long long* out, size_t cap, size_t* n);
// bounds-check self-test (tofr_gpu_debug_check_selftest); returns TOFR_CHECK
int launch_check_selftest(unsigned long long* out, cudaStream_t s);
void launch_probe_rays(const FrameView& F, const double* rays, int n, int mode, double* out_t, int* out_tri,
                       cudaStream_t s);

}  // namespace tofr_b200
