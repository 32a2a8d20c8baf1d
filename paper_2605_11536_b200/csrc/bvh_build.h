// bvh_build.h -- the frame's SAH BVH built on the device (bvh_build.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "host_scene.h"
#include "tofr_geom.h"

namespace tofr_b200 {

// Per-session scratch of the device build.  build() uploads the frame's
// world-space triangles (HTri layout) and builds the tree (one host sync per
// level); pack() writes the snapshot's tree and triangle arrays into a device
// blob laid out by pack_frame_shell(..., n_nodes, ...).
struct DeviceBvh {
    void *tris = nullptr, *order = nullptr, *tmp = nullptr, *nodes = nullptr, *bfs = nullptr, *next_lists = nullptr,
         *size = nullptr, *pre = nullptr, *esc = nullptr, *ctr = nullptr, *host_ctr = nullptr;
    // wide (multi-CTA) levels: node accumulators, chunk plan, chunk left
    // counts, tri_area snapshots summed on the side stream
    void *acc = nullptr, *chunks = nullptr, *chunk_left = nullptr, *area_snap = nullptr;
    std::vector<cudaStream_t> side;       // one per snapshot slot
    cudaEvent_t fork = nullptr;           // the level's snapshot is written
    std::vector<cudaEvent_t> slot_done;  // the slot's sums are done
    int cap = 0, nt = 0, n_nodes = 0, depth = 0;
    std::vector<int> level_off, level_n, level_nw, level_nb;  // per level: first task, tasks, wide, big tasks
    ~DeviceBvh();
    void release();
    void ensure(int nt);
    int build(const void* host_tris, int nt, cudaStream_t s);  // -> node count
    void wide_level(const int* tasks, int nw, int wide_levels, cudaStream_t s);
    void pack(unsigned char* blob, const PackedFrame& shell, cudaStream_t s);
    // the host builder's dump layout (tofr_scene_dump_bvh), for parity checks
    void dump(double* nodes_out, int32_t* parent_out, int32_t* order_out, cudaStream_t s);
};

}  // namespace tofr_b200
