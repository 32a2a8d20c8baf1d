/*
 * tofr_gpu.h -- C ABI of the B200 ToF ReSTIR renderer (libtofr_b200.so).
 *
 * Drop-in boundary for the CPU reference library `tofr`
 * (/root/reference/proj/include/tofr).  The reference has no FFI; its public
 * surface is the C++ API below, and each entry point here replaces one of
 * those functions with plain pointers/sizes (no C++ or torch types):
 *
 *   tofr_scene_create / tofr_scene_parse / tofr_scene_load
 *       <- SceneDef construction, parse_scene, load_scene
 *          (scene.hpp:417-429, scene_io.hpp:136-313)
 *   tofr_gpu_render_gated       <- render_gated           (pipeline.hpp:323-392)
 *   tofr_gpu_render_doppler     <- render_doppler         (pipeline.hpp:574-578)  (velocity gates)
 *   tofr_gpu_render_transient   <- render_transient       (pipeline.hpp:396-528)
 *   tofr_gpu_render_transient_plain <- render_transient_plain (pipeline.hpp:531-571)
 *   tofr_gpu_reference          <- reference_render       (harness.hpp:16-30)
 *   tofr_render_config          <- RenderConfig           (pipeline.hpp:18-61)
 *   tofr_frame_stats            <- FrameStats/StageStats/ShiftCounts
 *                                  (pipeline.hpp:63-72, shiftmap.hpp:398-417)
 *
 * Errors: every call returns 0 (TOFR_OK) or a TOFR_ERR_* code and never
 * throws; the message of the last failure is tofr_gpu_last_error(ctx) (or the
 * err buffer of the scene calls).  The reference's exceptions map as:
 * ParseError(line,col) -> TOFR_ERR_PARSE with "line:col: msg";
 * runtime_error("bvh: empty mesh"/"bvh: degenerate triangle") -> TOFR_ERR_SCENE.
 *
 * Threading: one context per process/device; a context is not re-entrant.
 * Outputs are caller-allocated host buffers filled by the call (the reference
 * returns RenderOutput by value).
 */
#ifndef TOFR_GPU_H
#define TOFR_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TOFR_OK 0
#define TOFR_ERR_INVALID 1
#define TOFR_ERR_PARSE 2
#define TOFR_ERR_SCENE 3
#define TOFR_ERR_CUDA 4
#define TOFR_ERR_OOM 5
#define TOFR_ERR_UNSUPPORTED 6

/* enums keep the reference's enumerator order */
enum { TOFR_MAT_DIFFUSE = 0, TOFR_MAT_GLOSSY = 1, TOFR_MAT_MIRROR = 2 };     /* MatKind */
enum { TOFR_LIGHT_COLLIMATED = 0, TOFR_LIGHT_WIDE = 1 };                     /* LightRegime */
enum { TOFR_MODE_GATED = 0, TOFR_MODE_TRANSIENT = 1, TOFR_MODE_DOPPLER = 2 }; /* RenderMode */
enum { TOFR_INIT_DIRECT = 0, TOFR_INIT_ELLIPSOIDAL = 1, TOFR_INIT_SHRINK = 2 }; /* InitMode */
enum { TOFR_GAUGE_FIXED = 0, TOFR_GAUGE_RAW = 1, TOFR_GAUGE_AVG = 2 };        /* GaugeKind */
enum { TOFR_GATE_LENGTH = 0, TOFR_GATE_VELOCITY = 1 };                       /* GateSpec::Kind */

typedef struct tofr_material {
    int32_t kind;
    double albedo[3];
    double roughness;
} tofr_material;

typedef struct tofr_light {
    int32_t regime;
    double position[3];
    double direction[3]; /* unit */
    double cone_half_angle;
    double intensity[3];
} tofr_light;

typedef struct tofr_camera_key {
    double frame;
    double position[3], forward[3], up[3];
} tofr_camera_key;

typedef struct tofr_pose_key {
    double frame;
    double q[4]; /* w, x, y, z */
    double t[3];
} tofr_pose_key;

typedef struct tofr_object_desc {
    const char* name;
    int32_t n_tris;
    const double* verts;       /* n_tris * 9: object-space v0, v1, v2 (make_triangle) */
    const int32_t* materials;  /* n_tris */
    int32_t n_keys;
    const tofr_pose_key* keys; /* rigid motion track, sorted by frame */
} tofr_object_desc;

typedef struct tofr_scene_desc {
    double cam_position[3], cam_forward[3], cam_up[3];
    double fov_y; /* radians */
    int32_t width, height;
    int32_t n_cam_keys;
    const tofr_camera_key* cam_keys;
    int32_t n_materials;
    const tofr_material* materials;
    tofr_light light;
    int32_t n_objects;
    const tofr_object_desc* objects;
    double dt_frame;
} tofr_scene_desc;

typedef struct tofr_render_config {
    int32_t mode;
    int32_t gate_kind;
    double gate_center, gate_width, gate_f0;
    double gate_step;
    int32_t bins;
    double hist_t0, hist_bin_width;
    int32_t m_init;
    int32_t init_mode;
    double shrink_k, shrink_r;
    int32_t spatial_passes, spatial_neighbors;
    double spatial_radius;
    int32_t temporal, bin_reuse;
    double m_cap;
    int32_t gauge;
    int32_t newton;
    uint64_t seed;
    int32_t frames;
    double frame0;
    int32_t max_depth;
    int32_t use_rr, accumulate, normalize_gate;
} tofr_render_config;

typedef struct tofr_shift_counts {
    uint64_t attempts, newton_ok, newton_failed, occluded, jac_clamped, replay_failed, iterations,
        solves, success;
} tofr_shift_counts;

typedef struct tofr_stage_stats {
    tofr_shift_counts shift;
    double seconds;
} tofr_stage_stats;

typedef struct tofr_frame_stats {
    int32_t frame;
    tofr_stage_stats temporal, spatial, binwise;
    double t_init, t_shade;
} tofr_frame_stats;

/* RenderOutput: image W*H*3 (row-major, rgb), histogram W*H*B(*3) in the
 * reference index order (y*W + x)*B + b.  Any pointer may be NULL. */
typedef struct tofr_output {
    double* image;
    double* hist_rgb;
    int64_t* hist_count;
    tofr_frame_stats* stats;
    int32_t stats_capacity;
} tofr_output;

typedef struct tofr_gpu tofr_gpu;
typedef struct tofr_scene tofr_scene;
typedef struct tofr_session tofr_session;

/* RenderConfig{} defaults (pipeline.hpp:18-61) */
void tofr_render_config_default(tofr_render_config* cfg);

/* context */
int tofr_gpu_create(const int* devices, int n_devices, tofr_gpu** out);
void tofr_gpu_destroy(tofr_gpu* ctx);
const char* tofr_gpu_last_error(const tofr_gpu* ctx);
const char* tofr_gpu_version(void);

/* scenes (host objects; frames are built and uploaded per render) */
int tofr_scene_create(const tofr_scene_desc* desc, tofr_scene** out, char* err, size_t errlen);
int tofr_scene_parse(const char* text, const char* base_dir, tofr_scene** out, char* err, size_t errlen);
int tofr_scene_load(const char* path, tofr_scene** out, char* err, size_t errlen);
void tofr_scene_destroy(tofr_scene* s);
int tofr_scene_set_resolution(tofr_scene* s, int32_t width, int32_t height);
/* info: width, height, n_triangles (frame 0), BVH nodes (frame 0); diag = scene_scale() */
int tofr_scene_info(const tofr_scene* s, int32_t* width, int32_t* height, int32_t* n_tris, int32_t* n_nodes,
                    double* diag, char* err, size_t errlen);

/* render drivers (RenderOutput is written into caller buffers) */
int tofr_gpu_render_gated(tofr_gpu* ctx, const tofr_scene* s, const tofr_render_config* cfg, tofr_output* out);
int tofr_gpu_render_doppler(tofr_gpu* ctx, const tofr_scene* s, const tofr_render_config* cfg, tofr_output* out);
int tofr_gpu_render_transient(tofr_gpu* ctx, const tofr_scene* s, const tofr_render_config* cfg,
                              tofr_output* out);
int tofr_gpu_render_transient_plain(tofr_gpu* ctx, const tofr_scene* s, const tofr_render_config* cfg,
                                    tofr_output* out);
/* reference_render(build_frame(def, frame), gate, spp, seed, max_depth): mean, se are W*H*3 */
int tofr_gpu_reference(tofr_gpu* ctx, const tofr_scene* s, double frame, double gate_center, double gate_width,
                       int32_t spp, uint64_t seed, int32_t max_depth, double* mean, double* se);

/* interactive sessions: the frame loop of render_gated / render_transient
 * one frame per call, reservoirs kept on the device between calls.  Steps are
 * asynchronous (two frames in flight) unless `stats` is non-NULL. */
int tofr_gpu_session_create(tofr_gpu* ctx, const tofr_scene* s, const tofr_render_config* cfg,
                            tofr_session** out);
/* Row-band session (multi-GPU sharding, parallel.hpp:17-36 generalised to
 * processes): computes image rows [y0, y1) and keeps `halo` rows on each side
 * for spatial reuse (pass halo >= ceil(spatial_radius)).  y1 = -1 means H.
 * RNG keys use global pixel indices, so a band is bit-identical to the same
 * rows of a full-frame session. */
int tofr_gpu_session_create_band(tofr_gpu* ctx, const tofr_scene* s, const tofr_render_config* cfg, int32_t y0,
                                 int32_t y1, int32_t halo, tofr_session** out);
/* Trace-only transient session (the frame loop of render_transient_plain):
 * rows [y0, y1) (y1 = -1: all), no reservoirs, no halo. */
int tofr_gpu_session_create_plain(tofr_gpu* ctx, const tofr_scene* s, const tofr_render_config* cfg, int32_t y0,
                                  int32_t y1, tofr_session** out);
int tofr_gpu_session_band(tofr_session* ss, int32_t* y0, int32_t* y1, int32_t* r0, int32_t* r1);
/* Halo exchange: before every spatial pass (pass >= 0) and, for moving
 * cameras, after the final grid of a frame (pass = -1) the library packs the
 * band's first rows into send_lo and last rows into send_hi (device buffers,
 * chunk-major), calls fn(user, pass), then unpacks recv_lo into the rows above
 * the band and recv_hi into the rows below.  fn must enqueue the transfer
 * (e.g. NCCL send/recv with the upper / lower neighbour rank) on the session
 * stream and return 0; a non-zero return aborts the step. */
typedef int (*tofr_halo_exchange_fn)(void* user, int32_t pass);
int tofr_gpu_session_set_halo_exchange(tofr_session* ss, tofr_halo_exchange_fn fn, void* user);
/* Native halo transports (no host callback per exchange):
 *  - NCCL, one process per GPU: every rank calls tofr_gpu_session_halo_nccl
 *    with the same 128-byte ncclUniqueId (rank 0: tofr_gpu_nccl_unique_id,
 *    broadcast by the host), its rank and the world size; rank g's band lies
 *    above rank g+1's.  ncclSend/ncclRecv with g-1 and g+1 run in one group on
 *    the session stream (libnccl.so.2 is loaded at run time:
 *    TOFR_ERR_UNSUPPORTED when it is missing).
 *  - in-process peer copies: tofr_gpu_session_link_halo(upper, lower) joins
 *    two adjacent band sessions of one process (any devices; NVLink P2P when
 *    they differ); each band is stepped from its own host thread.
 * tofr_gpu_session_halo_transport names the active one: "nccl", "peer",
 * "callback" or "none". */
int tofr_gpu_nccl_unique_id(uint8_t* id128);
int tofr_gpu_session_halo_nccl(tofr_session* ss, const uint8_t* id128, int32_t rank, int32_t world);
int tofr_gpu_session_link_halo(tofr_session* upper, tofr_session* lower);
int tofr_gpu_session_halo_transport(tofr_session* ss, const char** name);
int tofr_gpu_session_halo_buffers(tofr_session* ss, void** send_lo, void** recv_lo, uint64_t* bytes_lo,
                                  void** send_hi, void** recv_hi, uint64_t* bytes_hi);
int tofr_gpu_session_step(tofr_session* ss, tofr_frame_stats* stats);
/* image of the band's rows ((y1 - y0) * W * 3 doubles): the last frame's
 * image (gated) or the wide-band sum over bins of the histogram accumulated so
 * far divided by the frame count (transient, pipeline.hpp:521-526) */
int tofr_gpu_session_read_image(tofr_session* ss, double* image);
/* pipelined read-back: enqueue the same image into a caller-owned PINNED
 * buffer on the session stream (slot 0 or 1) and return at once;
 * tofr_gpu_session_wait_read(slot) blocks until that copy has landed */
int tofr_gpu_session_read_image_async(tofr_session* ss, double* pinned_image, int32_t slot);
int tofr_gpu_session_wait_read(tofr_session* ss, int32_t slot);
/* transient histogram accumulated so far / frames, reference index order;
 * count = deposits per bin (plain) or the frame count (reservoir mode) */
int tofr_gpu_session_read_histogram(tofr_session* ss, double* rgb, int64_t* count);
int tofr_gpu_session_sync(tofr_session* ss);
/* device timing of the last finished frame's kernels (ms) and the stage split
 * {init (incl. camera), temporal, bin reuse, spatial (incl. halo), shade, total} */
int tofr_gpu_session_last_ms(tofr_session* ss, double* total_ms, double* stage_ms /* [6] */);
/* running sums of the stage split over all finished frames (+ halo exchanges) */
int tofr_gpu_session_stage_totals(tofr_session* ss, double* stage_ms /* [6] */, int64_t* frames,
                                  uint64_t* halo_exchanges, int32_t reset);
/* the cudaStream_t all of the session's work is ordered on */
int tofr_gpu_session_stream(tofr_session* ss, void** stream);
/* bytes the last step uploaded (frame snapshot: BVH, triangles, camera, beam)
 * and the size of one image read-back */
int tofr_gpu_session_io_bytes(tofr_session* ss, uint64_t* h2d_per_step, uint64_t* d2h_image);
/* device work counted since the session was created: out[0] shift jobs,
 * out[1] closest-hit rays (incl. camera rays), out[2] any-hit (shadow /
 * occlusion) rays, out[3] transient histogram deposits, out[4] GRIS merges
 * with a non-empty side (reuse merge lists) */
int tofr_gpu_session_work(tofr_session* ss, uint64_t* out /* [5] */);
/* sparse transient grids: pool rows currently held by each of the three
 * reservoir grids (rows_used[3]) and the rows per grid (*rows_cap; 0 = the
 * session's grids are dense).  Waits for the frames in flight. */
int tofr_gpu_session_pool(tofr_session* ss, uint64_t* rows_used, uint64_t* rows_cap);
/* per-image-row shift cost (Newton iterations + 4 per shift job, by destination
 * row), for balancing multi-GPU row bands: enable = 1 zeroes the counters and
 * counts the following frames, enable = 0 stops; out (image height entries,
 * may be null) receives the counts so far.  Waits for the frames in flight. */
int tofr_gpu_session_row_cost(tofr_session* ss, int32_t enable, uint64_t* out);
void tofr_gpu_session_destroy(tofr_session* ss);

/* launch accounting of the library's kernels (process-wide): every launch is
 * counted; with timing enabled each launch is bracketed by CUDA events on its
 * stream and the per-kernel totals are read after the work finished */
int tofr_gpu_kernel_timing(int32_t enable); /* returns the previous setting */
uint64_t tofr_gpu_kernel_launches(void);
/* names: cap x name_len chars; returns the number of kernels written */
int tofr_gpu_kernel_times(char* names, int32_t name_len, double* total_ms, uint64_t* launches, int32_t cap);
void tofr_gpu_kernel_times_reset(void);

/* FNV-1a 64 of a byte buffer (image.hpp:90-97; manifest output hashes) */
uint64_t tofr_fnv1a64(const void* data, uint64_t n);

/* self-test of the device's shared-reciprocal FP64 division against the
 * compiler's a / b on n random V3 / scalar quotients: *mismatches = quotients
 * whose bits differ (0 expected) */
int tofr_gpu_selftest_div(tofr_gpu* ctx, uint64_t n, uint64_t seed, uint64_t* mismatches);

/* tofr_scene_dump_bvh of the tree built on the device (bvh_build.cu) for the
 * frame's world-space triangles: the same layout, for node-for-node parity
 * checks against the host builder (wide-light scenes) */
int tofr_gpu_dump_bvh_device(tofr_gpu* ctx, const tofr_scene* s, double frame, int32_t cap_nodes, double* nodes,
                             int32_t* node_parent, int32_t* n_nodes, int32_t cap_tris, int32_t* tri_order,
                             int32_t* n_tris, double* diag);

/* diagnostic (a -DTOFR_SOLVE_PROFILE=1 build only, else TOFR_ERR_UNSUPPORTED):
 * per solved shift job {cycles from refill to finish, trial rounds | Newton
 * iterations << 32 | re-projection rays << 40, global timer (ns) at finish}; copies up
 * to cap records (3 u64 each) and resets the recorder */
int tofr_gpu_debug_solve_profile(uint64_t* out, uint64_t cap, uint64_t* n);

/* bounds-check self-test: one thread asks a 4-item grid for the pool row of
 * item 5.  A checked build (-DTOFR_CHECK=1) traps (returns TOFR_ERR_CUDA and
 * leaves the context unusable: call it in a throw-away process); the product
 * build, which does no checks and touches no memory there, returns TOFR_OK
 * with *checked = 0.  *checked = 1 when the library was built with checks. */
int tofr_gpu_debug_check_selftest(tofr_gpu* ctx, int32_t* checked);

/* measured FP64 throughput of the context's device (DFMA chains; GFLOP/s with
 * 2 flops per DFMA): the FP64 roofline's peak */
int tofr_gpu_fp64_peak(tofr_gpu* ctx, double* gflops);

/* parity probes: rays[i] = {o.xyz, d.xyz, tmin, tmax}; mode 0 = closest hit
 * (Bvh::intersect_min) -> t, tri; mode 1 = occluded(a = o, b = d) -> tri = 0/1 */
int tofr_gpu_probe_rays(tofr_gpu* ctx, const tofr_scene* s, double frame, const double* rays, int32_t n,
                        int32_t mode, double* out_t, int32_t* out_tri);
/* same probe through the host build of the traversal code (no GPU needed) */
int tofr_scene_probe_rays_host(const tofr_scene* s, double frame, const double* rays, int32_t n, int32_t mode,
                               double* out_t, int32_t* out_tri, char* err, size_t errlen);
/* host BVH of one frame in the reference layout (for build parity):
 * nodes: n_nodes * 11 doubles {lo.xyz, hi.xyz, tri_area, left, right, first, count}, parent in
 * node_parent; tri_order n_tris */
int tofr_scene_dump_bvh(const tofr_scene* s, double frame, int32_t cap_nodes, double* nodes,
                        int32_t* node_parent, int32_t* n_nodes, int32_t cap_tris, int32_t* tri_order,
                        int32_t* n_tris, double* diag, char* err, size_t errlen);

#ifdef __cplusplus
}
#endif

#endif /* TOFR_GPU_H */
