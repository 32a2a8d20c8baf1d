// bvh_build.cu -- the binned SAH BVH of a frame built on the device,
// node-for-node the host builder's (SahBuilder, host_scene.cpp), which is the
// reference's Bvh::build_node (geometry.hpp:234-317): 8 bins on the widest
// centroid axis, <= 4 triangles per leaf, stable partition, the same
// fall-backs, node boxes, tri_area sums and depth-first (pre-order) numbering.
//
// Level-synchronous: one CTA per node of the current level computes its box,
// centroid box and binned split (min / max reductions: exact in any order),
// its tri_area (a sequential sum by one thread: the reference's order), and
// stably partitions its range of the triangle order (block-wide scans); nodes
// of <= 64 triangles take one warp each (k_bvh_level_warp); the children form
// the next level.  Nodes of more than kWideNode triangles (the
// top levels, where one CTA per node would leave the GPU idle) are split over
// many CTAs (k_wide_*).  After the last level the nodes are
// renumbered in the reference's depth-first order (subtree sizes bottom-up,
// pre-order indices top-down) and packed into the frame snapshot layout
// (pack_frame: threaded hit / miss links, leaf-order triangles, per-triangle
// info and tangent frames) in place, in the slot's device blob.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>
#include <vector>

#include "bvh_build.h"
#include "ktime.h"

namespace tofr_b200 {

namespace {

struct BNode {  // a node in build (creation) order
    V3 lo, hi;
    double tri_area;
    int left, right, first, count, parent, pad;
};

struct BTri {  // == HTri (host_scene.h): v0, v1, v2, n, material, object, area
    V3 v0, v1, v2, n;
    int material, object;
    double area;
};

constexpr int kBinsDev = 8;
constexpr int kBuildThreads = 256;

__device__ __forceinline__ double centroid_axis(const BTri& t, int a) {
    return (comp(t.v0, a) + comp(t.v1, a) + comp(t.v2, a)) / 3.0;
}
__device__ __forceinline__ double box_area(const V3& lo, const V3& hi) {  // Box::area
    V3 e = hi - lo;
    if (e.x < 0) return 0;
    return 2.0 * (e.x * e.y + e.y * e.z + e.z * e.x);
}

// block-wide min / max of one double (every thread gets the result)
__device__ double block_min(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v = dmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = sh[0];
    for (int i = 1; i < int(blockDim.x >> 5); ++i) r = dmin(r, sh[i]);
    return r;
}
__device__ double block_max(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v = dmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = sh[0];
    for (int i = 1; i < int(blockDim.x >> 5); ++i) r = dmax(r, sh[i]);
    return r;
}
__device__ int block_sum(int v, int* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    int r = 0;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) r += sh[i];
    return r;
}
// block-wide min (k < nmin) / max (k >= nmin) of N doubles per thread, written to
// out[N] in shared memory: one shuffle tree per value, one barrier pair
template <int N>
__device__ void block_minmax(double (&v)[N], int nmin, double (*wsh)[N], double* out) {
#pragma unroll
    for (int k = 0; k < N; ++k)
        for (int o = 16; o > 0; o >>= 1) {
            double w = __shfl_xor_sync(0xffffffffu, v[k], o);
            v[k] = k < nmin ? dmin(v[k], w) : dmax(v[k], w);
        }
    const int wid = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0)
#pragma unroll
        for (int k = 0; k < N; ++k) wsh[wid][k] = v[k];
    __syncthreads();
    if (threadIdx.x < N) {
        const int k = threadIdx.x;
        double r = wsh[0][k];
        for (int i = 1; i < int(blockDim.x >> 5); ++i) r = k < nmin ? dmin(r, wsh[i][k]) : dmax(r, wsh[i][k]);
        out[k] = r;
    }
    __syncthreads();
}

// exclusive block scan of a small count per thread; *total = the block sum
__device__ int block_scan_count(int c, int* sh, int* total) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    int incl = c;
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (l >= o) incl += t;
    }
    __syncthreads();
    if (l == 31) sh[w] = incl;
    __syncthreads();
    int before = 0, all = 0;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) {
        if (i < w) before += sh[i];
        all += sh[i];
    }
    *total = all;
    return before + incl - c;
}

// exclusive block scan of a 0/1 flag; returns the prefix, *total the block sum
__device__ int block_scan(int f, int* sh, int* total) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const unsigned m = __ballot_sync(0xffffffffu, f);
    const int in_warp = __popc(m & ((1u << l) - 1));
    __syncthreads();
    if (l == 0) sh[w] = __popc(m);
    __syncthreads();
    int before = 0, all = 0;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) {
        if (i < w) before += sh[i];
        all += sh[i];
    }
    *total = all;
    return before + in_warp;
}

constexpr int kSmallNode = 64;   // nodes this small are built by one thread
constexpr int kWideNode = 4096;  // nodes above this are built by many CTAs (k_wide_*)

// children of node id (ranges [first, mid), [mid, first + count)); they join
// the next level's big list (next[0..]), small list (next[n_next[2]..]) or
// wide list (next[n_next[4]..]); n_next[0, 1, 3] count them
__device__ void make_children(BNode* nodes, int id, int first, int count, int mid, int* next, int* n_next,
                              int* n_nodes) {
    int c = atomicAdd(n_nodes, 2);
    BNode l{}, r{};
    l.first = first;
    l.count = mid - first;
    l.parent = id;
    r.first = mid;
    r.count = first + count - mid;
    r.parent = id;
    nodes[c] = l;
    nodes[c + 1] = r;
    nodes[id].left = c;
    nodes[id].right = c + 1;
    for (int k = 0; k < 2; ++k) {
        const int n = k ? r.count : l.count;
        const int list = n <= kSmallNode ? 1 : (n > kWideNode ? 2 : 0);
        const int cnt = list == 2 ? 3 : list, base = list == 0 ? 0 : n_next[list == 1 ? 2 : 4];
        int t = atomicAdd(&n_next[cnt], 1);
        next[base + t] = c + k;
    }
}

// SahBuilder's split choice over the 7 bin boundaries (-1: no bin boundary
// separates the triangles)
__device__ int sah_split(const int* bc, const double (*bl)[3], const double (*bh)[3]) {
    double best_cost = kInf;
    int best = -1;
    for (int sp = 1; sp < kBinsDev; ++sp) {
        V3 llo{kInf, kInf, kInf}, lhi{-kInf, -kInf, -kInf}, rlo = llo, rhi = lhi;
        int lc = 0, rc = 0;
        for (int i = 0; i < sp; ++i) {
            if (bc[i]) {
                llo = vmin(llo, V3{bl[i][0], bl[i][1], bl[i][2]});
                lhi = vmax(lhi, V3{bh[i][0], bh[i][1], bh[i][2]});
            }
            lc += bc[i];
        }
        for (int i = sp; i < kBinsDev; ++i) {
            if (bc[i]) {
                rlo = vmin(rlo, V3{bl[i][0], bl[i][1], bl[i][2]});
                rhi = vmax(rhi, V3{bh[i][0], bh[i][1], bh[i][2]});
            }
            rc += bc[i];
        }
        if (lc == 0 || rc == 0) continue;
        double cost = box_area(llo, lhi) * lc + box_area(rlo, rhi) * rc;
        if (cost < best_cost) {
            best_cost = cost;
            best = sp;
        }
    }
    return best;
}

// one level: CTA b builds node tasks[b]
__global__ void __launch_bounds__(kBuildThreads) k_bvh_level(const BTri* tris, int* order, int* tmp, BNode* nodes,
                                                             const int* tasks, int n_tasks, int* next, int* n_next,
                                                             int* n_nodes) {
    if (int(blockIdx.x) >= n_tasks) return;
    __shared__ double shd[kBuildThreads / 32];
    __shared__ int shi[kBuildThreads / 32];
    __shared__ int s_split, s_axis;
    __shared__ double s_lo, s_width;
    const int id = tasks[blockIdx.x];
    const int first = nodes[id].first, count = nodes[id].count;
    // box and centroid box
    V3 lo{kInf, kInf, kInf}, hi{-kInf, -kInf, -kInf}, clo = lo, chi = hi;
    for (int i = first + threadIdx.x; i < first + count; i += blockDim.x) {
        const BTri& t = tris[order[i]];
        lo = vmin(vmin(vmin(lo, t.v0), t.v1), t.v2);
        hi = vmax(vmax(vmax(hi, t.v0), t.v1), t.v2);
        V3 c = (t.v0 + t.v1 + t.v2) / 3.0;
        clo = vmin(clo, c);
        chi = vmax(chi, c);
    }
    {
        __shared__ double wsh12[kBuildThreads / 32][12], out12[12];
        double v[12] = {lo.x, lo.y, lo.z, clo.x, clo.y, clo.z, hi.x, hi.y, hi.z, chi.x, chi.y, chi.z};
        block_minmax<12>(v, 6, wsh12, out12);
        lo = V3{out12[0], out12[1], out12[2]};
        clo = V3{out12[3], out12[4], out12[5]};
        hi = V3{out12[6], out12[7], out12[8]};
        chi = V3{out12[9], out12[10], out12[11]};
    }
    // tri_area: the reference's sequential sum (area += t.area over the range, in
    // order) by one thread, its operands gathered into shared memory by the block
    __shared__ double s_area[1024];
    double area = 0;
    for (int base = first; base < first + count; base += 1024) {
        const int m = min(1024, first + count - base);
        __syncthreads();
        for (int k = threadIdx.x; k < m; k += blockDim.x) s_area[k] = tris[order[base + k]].area;
        __syncthreads();
        if (threadIdx.x == 0)
            for (int k = 0; k < m; ++k) area += s_area[k];
    }
    if (threadIdx.x == 0) {
        BNode& nd = nodes[id];
        nd.lo = lo;
        nd.hi = hi;
        nd.tri_area = area;
        nd.left = nd.right = -1;
    }
    if (count <= 4) return;  // leaf
    if (threadIdx.x == 0) {
        V3 ext = chi - clo;
        int axis = ext.x > ext.y ? (ext.x > ext.z ? 0 : 2) : (ext.y > ext.z ? 1 : 2);
        s_axis = axis;
        s_lo = comp(clo, axis);
        s_width = comp(ext, axis);
    }
    __syncthreads();
    const int axis = s_axis;
    const double blo = s_lo, width = s_width;
    int mid = first + count / 2;
    if (!(width < 1e-12)) {
        auto bin_of = [&](const BTri& t) {
            double c = (centroid_axis(t, axis) - blo) / width;
            int b = int(c * kBinsDev);
            return b < kBinsDev - 1 ? b : kBinsDev - 1;
        };
        int bc[kBinsDev];
        V3 bl[kBinsDev], bh[kBinsDev];
#pragma unroll
        for (int k = 0; k < kBinsDev; ++k) {
            bc[k] = 0;
            bl[k] = V3{kInf, kInf, kInf};
            bh[k] = V3{-kInf, -kInf, -kInf};
        }
        for (int i = first + threadIdx.x; i < first + count; i += blockDim.x) {
            const BTri& t = tris[order[i]];
            int b = bin_of(t);
#pragma unroll
            for (int k = 0; k < kBinsDev; ++k)
                if (k == b) {
                    bc[k]++;
                    bl[k] = vmin(vmin(vmin(bl[k], t.v0), t.v1), t.v2);
                    bh[k] = vmax(vmax(vmax(bh[k], t.v0), t.v1), t.v2);
                }
        }
        __shared__ int s_bc[kBinsDev];
        __shared__ double s_bl[kBinsDev][3], s_bh[kBinsDev][3];
        {  // all bins at once: 24 minima, 24 maxima; counts by warp sums
            __shared__ double wsh48[kBuildThreads / 32][48], out48[48];
            double v[48];
#pragma unroll
            for (int k = 0; k < kBinsDev; ++k) {
                v[3 * k + 0] = bl[k].x;
                v[3 * k + 1] = bl[k].y;
                v[3 * k + 2] = bl[k].z;
                v[24 + 3 * k + 0] = bh[k].x;
                v[24 + 3 * k + 1] = bh[k].y;
                v[24 + 3 * k + 2] = bh[k].z;
            }
            block_minmax<48>(v, 24, wsh48, out48);
            __shared__ int wc[kBuildThreads / 32][kBinsDev];
#pragma unroll
            for (int k = 0; k < kBinsDev; ++k)
                for (int o = 16; o > 0; o >>= 1) bc[k] += __shfl_xor_sync(0xffffffffu, bc[k], o);
            if ((threadIdx.x & 31) == 0)
#pragma unroll
                for (int k = 0; k < kBinsDev; ++k) wc[threadIdx.x >> 5][k] = bc[k];
            __syncthreads();
            if (threadIdx.x < kBinsDev) {
                const int k = threadIdx.x;
                int c = 0;
                for (int i = 0; i < int(blockDim.x >> 5); ++i) c += wc[i][k];
                s_bc[k] = c;
                for (int a = 0; a < 3; ++a) {
                    s_bl[k][a] = out48[3 * k + a];
                    s_bh[k][a] = out48[24 + 3 * k + a];
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) s_split = sah_split(s_bc, s_bl, s_bh);  // SahBuilder's cost loop
        __syncthreads();
        const int split = s_split;
        if (split >= 0) {
            // stable partition of [first, first + count) by bin < split: chunks of
            // 4 consecutive elements per thread, one count scan per chunk
            constexpr int kPer = 4;
            const int chunk = kPer * int(blockDim.x);
            int n_left = 0;
            for (int base = first; base < first + count; base += chunk) {
                int c = 0;
                for (int e = 0; e < kPer; ++e) {
                    int i = base + kPer * int(threadIdx.x) + e;
                    if (i < first + count) c += int(bin_of(tris[order[i]]) < split);
                }
                n_left += block_sum(c, shi);
            }
            int lpos = first, rpos = first + n_left;
            for (int base = first; base < first + count; base += chunk) {
                int ids[kPer], fl[kPer], c = 0, live_n = 0;
                for (int e = 0; e < kPer; ++e) {
                    int i = base + kPer * int(threadIdx.x) + e;
                    bool live = i < first + count;
                    ids[e] = live ? order[i] : -1;
                    fl[e] = live ? int(bin_of(tris[ids[e]]) < split) : 0;
                    c += fl[e];
                    live_n += live ? 1 : 0;
                }
                int tot_l = 0;
                const int pl = block_scan_count(c, shi, &tot_l);
                // elements before this thread's in the chunk, minus the left ones among them
                const int before = min(kPer * int(threadIdx.x), max(0, first + count - base));
                int l = pl, r = before - pl;
                for (int e = 0; e < kPer; ++e) {
                    if (ids[e] < 0) continue;
                    if (fl[e])
                        tmp[lpos + l++] = ids[e];
                    else
                        tmp[rpos + r++] = ids[e];
                }
                const int chunk_n = min(chunk, first + count - base);
                lpos += tot_l;
                rpos += chunk_n - tot_l;
                (void)live_n;
            }
            __syncthreads();
            for (int i = first + threadIdx.x; i < first + count; i += blockDim.x) order[i] = tmp[i];
            mid = first + n_left;
            if (mid == first || mid == first + count) mid = first + count / 2;
        }
    }
    if (threadIdx.x == 0) make_children(nodes, id, first, count, mid, next, n_next, n_nodes);
}

// one warp per node of <= kSmallNode triangles (the bottom levels): the node's
// triangles staged in shared memory, box / centroid box by shuffles, the
// sequential tri_area by lane 0, bin boxes by lanes 0-7 (one bin each), the SAH
// choice by lane 0 (the host loop), the stable partition by ballots
constexpr int kWarpNodes = 4;  // warps (nodes) per CTA
__global__ void __launch_bounds__(32 * kWarpNodes) k_bvh_level_warp(const BTri* tris, int* order, BNode* nodes,
                                                                    const int* tasks, int n_tasks, int* next,
                                                                    int* n_next, int* n_nodes) {
    static_assert(kSmallNode <= 64, "two triangles per lane");
    __shared__ BTri s_tri[kWarpNodes][kSmallNode];
    __shared__ signed char s_bin[kWarpNodes][kSmallNode];
    __shared__ double s_bb[kWarpNodes][kBinsDev][6];
    __shared__ int s_bc[kWarpNodes][kBinsDev];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = blockIdx.x * kWarpNodes + w;
    if (k >= n_tasks) return;  // whole warps
    const int id = tasks[k];
    const int first = nodes[id].first, count = nodes[id].count;
    BTri* st = s_tri[w];
    int ids[2];
    for (int e = 0; e < 2; ++e) {
        const int j = lane + 32 * e;
        ids[e] = j < count ? order[first + j] : -1;
        if (j < count) st[j] = tris[ids[e]];
    }
    __syncwarp();
    V3 lo{kInf, kInf, kInf}, hi{-kInf, -kInf, -kInf}, clo = lo, chi = hi;
    for (int j = lane; j < count; j += 32) {
        const BTri& t = st[j];
        lo = vmin(vmin(vmin(lo, t.v0), t.v1), t.v2);
        hi = vmax(vmax(vmax(hi, t.v0), t.v1), t.v2);
        V3 c = (t.v0 + t.v1 + t.v2) / 3.0;
        clo = vmin(clo, c);
        chi = vmax(chi, c);
    }
    double v[12] = {lo.x, lo.y, lo.z, clo.x, clo.y, clo.z, hi.x, hi.y, hi.z, chi.x, chi.y, chi.z};
#pragma unroll
    for (int q = 0; q < 12; ++q)
        for (int o = 16; o > 0; o >>= 1) {
            double x = __shfl_xor_sync(0xffffffffu, v[q], o);
            v[q] = q < 6 ? dmin(v[q], x) : dmax(v[q], x);
        }
    lo = V3{v[0], v[1], v[2]};
    clo = V3{v[3], v[4], v[5]};
    hi = V3{v[6], v[7], v[8]};
    chi = V3{v[9], v[10], v[11]};
    if (lane == 0) {
        double area = 0;
        for (int j = 0; j < count; ++j) area += st[j].area;
        BNode& nd = nodes[id];
        nd.lo = lo;
        nd.hi = hi;
        nd.tri_area = area;
        nd.left = nd.right = -1;
    }
    if (count <= 4) return;  // leaf
    V3 ext = chi - clo;
    const int axis = ext.x > ext.y ? (ext.x > ext.z ? 0 : 2) : (ext.y > ext.z ? 1 : 2);
    const double blo = comp(clo, axis), width = comp(ext, axis);
    int mid = first + count / 2;
    int split = -1;
    int fl[2] = {0, 0};
    if (!(width < 1e-12)) {
        for (int e = 0; e < 2; ++e) {
            const int j = lane + 32 * e;
            if (j < count) {
                double c = (centroid_axis(st[j], axis) - blo) / width;
                int b = int(c * kBinsDev);
                s_bin[w][j] = static_cast<signed char>(b < kBinsDev - 1 ? b : kBinsDev - 1);
            }
        }
        __syncwarp();
        if (lane < kBinsDev) {  // bin `lane`: count and box over its triangles
            V3 bl{kInf, kInf, kInf}, bh{-kInf, -kInf, -kInf};
            int bc = 0;
            for (int j = 0; j < count; ++j)
                if (s_bin[w][j] == lane) {
                    const BTri& t = st[j];
                    bc++;
                    bl = vmin(vmin(vmin(bl, t.v0), t.v1), t.v2);
                    bh = vmax(vmax(vmax(bh, t.v0), t.v1), t.v2);
                }
            s_bc[w][lane] = bc;
            double* o = s_bb[w][lane];
            o[0] = bl.x;
            o[1] = bl.y;
            o[2] = bl.z;
            o[3] = bh.x;
            o[4] = bh.y;
            o[5] = bh.z;
        }
        __syncwarp();
        if (lane == 0) {
            double bl[kBinsDev][3], bh[kBinsDev][3];
            for (int q = 0; q < kBinsDev; ++q)
                for (int ax = 0; ax < 3; ++ax) {
                    bl[q][ax] = s_bb[w][q][ax];
                    bh[q][ax] = s_bb[w][q][3 + ax];
                }
            split = sah_split(s_bc[w], bl, bh);
        }
        split = __shfl_sync(0xffffffffu, split, 0);
        if (split >= 0) {  // std::stable_partition by bin < split
            for (int e = 0; e < 2; ++e) {
                const int j = lane + 32 * e;
                fl[e] = j < count ? int(s_bin[w][j] < split) : 0;
            }
            const unsigned b0 = __ballot_sync(0xffffffffu, fl[0]), b1 = __ballot_sync(0xffffffffu, fl[1]);
            const unsigned lt = (1u << lane) - 1;
            const int n_left = __popc(b0) + __popc(b1);
            for (int e = 0; e < 2; ++e) {
                const int j = lane + 32 * e;
                if (j >= count) continue;
                const int left_before = e ? __popc(b0) + __popc(b1 & lt) : __popc(b0 & lt);
                order[first + (fl[e] ? left_before : n_left + (j - left_before))] = ids[e];
            }
            mid = first + n_left;
            if (mid == first || mid == first + count) mid = first + count / 2;
        }
    }
    if (lane == 0) make_children(nodes, id, first, count, mid, next, n_next, n_nodes);
}

// ---------------------------------------------------------------------------
// Wide nodes (more than kWideNode triangles: the top levels) are built by many
// CTAs each: one CTA per kChunk-triangle chunk of the node's range, in five
// launches per level (plan, bounds, bins, count, scatter) and one CTA per node
// to finish.  Box and bin minima / maxima go through 64-bit atomics on an
// order-preserving integer image of the doubles (exact in any order); the
// stable partition scans the chunks' left counts in chunk order.  tri_area
// (the reference's sequential sum) is the one order-dependent step: the level's
// areas are copied, in the level's triangle order, into a snapshot slot and
// summed by one thread per node on the slot's side stream, off the build's
// critical path and concurrently across levels (the root's sum is a chain of
// nt dependent adds, ~11 cycles each).

constexpr int kChunk = 4 * kBuildThreads;  // triangles per CTA
constexpr int kAreaSlots = 8;              // snapshot ring of the side-stream sums

__device__ __forceinline__ unsigned long long okey(double d) {  // monotone: a < b <=> okey(a) < okey(b)
    unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(d));
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_inv(unsigned long long k) {
    return __longlong_as_double(static_cast<long long>((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

struct WideAcc {                // one wide node's reductions over its chunks
    unsigned long long box[12];  // lo, clo (min keys), hi, chi (max keys)
    unsigned long long bl[kBinsDev][3], bh[kBinsDev][3];
    int bc[kBinsDev];
    int split, n_left, c0, nch;  // SAH split (-1: none), left count, first chunk, chunks
};
struct WideChunk {
    int node, acc, lo, hi;  // node id, its accumulator, triangle range [lo, hi)
};

// the node's split axis / origin / width from its centroid box
struct WideAxis {
    int axis;
    double blo, width;
};
__device__ WideAxis wide_axis(const WideAcc& a) {
    V3 clo{okey_inv(a.box[3]), okey_inv(a.box[4]), okey_inv(a.box[5])};
    V3 chi{okey_inv(a.box[9]), okey_inv(a.box[10]), okey_inv(a.box[11])};
    V3 ext = chi - clo;
    WideAxis w;
    w.axis = ext.x > ext.y ? (ext.x > ext.z ? 0 : 2) : (ext.y > ext.z ? 1 : 2);
    w.blo = comp(clo, w.axis);
    w.width = comp(ext, w.axis);
    return w;
}
__device__ __forceinline__ int wide_bin(const BTri& t, const WideAxis& w) {
    double c = (centroid_axis(t, w.axis) - w.blo) / w.width;
    int b = int(c * kBinsDev);
    return b < kBinsDev - 1 ? b : kBinsDev - 1;
}

// chunk map of the level's wide nodes, accumulators reset (one thread: nw is small)
__global__ void k_wide_plan(const BNode* nodes, const int* tasks, int nw, WideAcc* acc, WideChunk* chunks,
                            int* n_chunks) {
    int c = 0;
    for (int k = 0; k < nw; ++k) {
        const int id = tasks[k], first = nodes[id].first, count = nodes[id].count;
        acc[k].c0 = c;
        acc[k].nch = (count + kChunk - 1) / kChunk;
        for (int lo = first; lo < first + count; lo += kChunk) chunks[c++] = WideChunk{id, k, lo, min(lo + kChunk, first + count)};
    }
    *n_chunks = c;
}
__global__ void k_wide_reset(WideAcc* acc, int nw) {
    const int k = blockIdx.x;
    if (k >= nw) return;
    WideAcc& a = acc[k];
    const int t = threadIdx.x;
    if (t < 12) a.box[t] = t < 6 ? ~0ull : 0ull;
    if (t < 3 * kBinsDev) {
        a.bl[t / 3][t % 3] = ~0ull;
        a.bh[t / 3][t % 3] = 0ull;
    }
    if (t < kBinsDev) a.bc[t] = 0;
    if (t == 0) {
        a.split = -1;
        a.n_left = 0;
    }
}

// boxes and centroid boxes; the chunk's areas into the level's snapshot
__global__ void __launch_bounds__(kBuildThreads) k_wide_bounds(const BTri* tris, const int* order,
                                                               const WideChunk* chunks, const int* n_chunks,
                                                               WideAcc* acc, double* area_snap) {
    if (int(blockIdx.x) >= *n_chunks) return;
    const WideChunk ch = chunks[blockIdx.x];
    V3 lo{kInf, kInf, kInf}, hi{-kInf, -kInf, -kInf}, clo = lo, chi = hi;
    for (int i = ch.lo + threadIdx.x; i < ch.hi; i += blockDim.x) {
        const BTri& t = tris[order[i]];
        lo = vmin(vmin(vmin(lo, t.v0), t.v1), t.v2);
        hi = vmax(vmax(vmax(hi, t.v0), t.v1), t.v2);
        V3 c = (t.v0 + t.v1 + t.v2) / 3.0;
        clo = vmin(clo, c);
        chi = vmax(chi, c);
        area_snap[i] = t.area;
    }
    __shared__ double wsh12[kBuildThreads / 32][12], out12[12];
    double v[12] = {lo.x, lo.y, lo.z, clo.x, clo.y, clo.z, hi.x, hi.y, hi.z, chi.x, chi.y, chi.z};
    block_minmax<12>(v, 6, wsh12, out12);
    if (threadIdx.x < 12) {
        const int k = threadIdx.x;
        unsigned long long* dst = &acc[ch.acc].box[k];
        if (k < 6)
            atomicMin(dst, okey(out12[k]));
        else
            atomicMax(dst, okey(out12[k]));
    }
}

// bin counts and bin boxes
__global__ void __launch_bounds__(kBuildThreads) k_wide_bins(const BTri* tris, const int* order,
                                                             const WideChunk* chunks, const int* n_chunks,
                                                             WideAcc* acc) {
    if (int(blockIdx.x) >= *n_chunks) return;
    const WideChunk ch = chunks[blockIdx.x];
    WideAcc& a = acc[ch.acc];
    const WideAxis w = wide_axis(a);
    if (w.width < 1e-12) return;  // no split: the node is halved
    int bc[kBinsDev];
    V3 bl[kBinsDev], bh[kBinsDev];
#pragma unroll
    for (int k = 0; k < kBinsDev; ++k) {
        bc[k] = 0;
        bl[k] = V3{kInf, kInf, kInf};
        bh[k] = V3{-kInf, -kInf, -kInf};
    }
    for (int i = ch.lo + threadIdx.x; i < ch.hi; i += blockDim.x) {
        const BTri& t = tris[order[i]];
        const int b = wide_bin(t, w);
#pragma unroll
        for (int k = 0; k < kBinsDev; ++k)
            if (k == b) {
                bc[k]++;
                bl[k] = vmin(vmin(vmin(bl[k], t.v0), t.v1), t.v2);
                bh[k] = vmax(vmax(vmax(bh[k], t.v0), t.v1), t.v2);
            }
    }
    __shared__ double wsh48[kBuildThreads / 32][48], out48[48];
    __shared__ int wc[kBuildThreads / 32][kBinsDev];
    double v[48];
#pragma unroll
    for (int k = 0; k < kBinsDev; ++k) {
        v[3 * k + 0] = bl[k].x;
        v[3 * k + 1] = bl[k].y;
        v[3 * k + 2] = bl[k].z;
        v[24 + 3 * k + 0] = bh[k].x;
        v[24 + 3 * k + 1] = bh[k].y;
        v[24 + 3 * k + 2] = bh[k].z;
    }
    block_minmax<48>(v, 24, wsh48, out48);  // ends with a barrier
#pragma unroll
    for (int k = 0; k < kBinsDev; ++k)
        for (int o = 16; o > 0; o >>= 1) bc[k] += __shfl_xor_sync(0xffffffffu, bc[k], o);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int k = 0; k < kBinsDev; ++k) wc[threadIdx.x >> 5][k] = bc[k];
    __syncthreads();
    const int t = threadIdx.x;
    if (t < 48) {  // empty bins keep their identity keys, as the host's untouched bins
        const int k = (t % 24) / 3, ax = t % 3;
        if (t < 24)
            atomicMin(&a.bl[k][ax], okey(out48[t]));
        else
            atomicMax(&a.bh[k][ax], okey(out48[t]));
    } else if (t < 48 + kBinsDev) {
        const int k = t - 48;
        int c = 0;
        for (int i = 0; i < int(blockDim.x >> 5); ++i) c += wc[i][k];
        if (c) atomicAdd(&a.bc[k], c);
    }
}

// the split (every chunk derives the same) and the chunk's left count
__global__ void __launch_bounds__(kBuildThreads) k_wide_count(const BTri* tris, const int* order,
                                                              const WideChunk* chunks, const int* n_chunks,
                                                              WideAcc* acc, int* chunk_left) {
    if (int(blockIdx.x) >= *n_chunks) return;
    const WideChunk ch = chunks[blockIdx.x];
    WideAcc& a = acc[ch.acc];
    const WideAxis w = wide_axis(a);
    __shared__ int s_split;
    __shared__ int shi[kBuildThreads / 32];
    if (threadIdx.x == 0) {
        int split = -1;
        if (!(w.width < 1e-12)) {
            double bl[kBinsDev][3], bh[kBinsDev][3];
            for (int k = 0; k < kBinsDev; ++k)
                for (int ax = 0; ax < 3; ++ax) {
                    bl[k][ax] = okey_inv(a.bl[k][ax]);
                    bh[k][ax] = okey_inv(a.bh[k][ax]);
                }
            split = sah_split(a.bc, bl, bh);
        }
        s_split = split;
        if (int(blockIdx.x) == a.c0) a.split = split;
    }
    __syncthreads();
    const int split = s_split;
    int c = 0;
    if (split >= 0)
        for (int i = ch.lo + threadIdx.x; i < ch.hi; i += blockDim.x) c += int(wide_bin(tris[order[i]], w) < split);
    const int n = block_sum(c, shi);
    if (threadIdx.x == 0) chunk_left[blockIdx.x] = n;
}

// stable partition: the chunk's left / right elements after the node's earlier
// chunks' ones (chunks in range order), into tmp
__global__ void __launch_bounds__(kBuildThreads) k_wide_scatter(const BTri* tris, const int* order, int* tmp,
                                                                const BNode* nodes, const WideChunk* chunks,
                                                                const int* n_chunks, WideAcc* acc,
                                                                const int* chunk_left) {
    if (int(blockIdx.x) >= *n_chunks) return;
    const WideChunk ch = chunks[blockIdx.x];
    WideAcc& a = acc[ch.acc];
    if (a.split < 0) return;
    const int split = a.split;
    const WideAxis w = wide_axis(a);
    __shared__ int s_before, s_total;
    __shared__ int shi[kBuildThreads / 32];
    if (threadIdx.x == 0) {
        int before = 0, total = 0;
        for (int c = a.c0; c < a.c0 + a.nch; ++c) {
            if (c < int(blockIdx.x)) before += chunk_left[c];
            total += chunk_left[c];
        }
        s_before = before;
        s_total = total;
        if (int(blockIdx.x) == a.c0) a.n_left = total;
    }
    __syncthreads();
    const int first = nodes[ch.node].first;
    // left elements of this chunk go after `before` left ones; right elements
    // after the node's n_left left ones and the (ch.lo - first - before) right
    // ones of the earlier chunks
    const int lbase = first + s_before, rbase = first + s_total + (ch.lo - first - s_before);
    constexpr int kPer = 4;
    int ids[kPer], fl[kPer], c = 0;
    for (int e = 0; e < kPer; ++e) {
        const int i = ch.lo + kPer * int(threadIdx.x) + e;
        const bool live = i < ch.hi;
        ids[e] = live ? order[i] : -1;
        fl[e] = live ? int(wide_bin(tris[ids[e]], w) < split) : 0;
        c += fl[e];
    }
    int tot_l = 0;
    const int pl = block_scan_count(c, shi, &tot_l);
    const int before = min(kPer * int(threadIdx.x), max(0, ch.hi - ch.lo));
    int l = pl, r = before - pl;
    for (int e = 0; e < kPer; ++e) {
        if (ids[e] < 0) continue;
        if (fl[e])
            tmp[lbase + l++] = ids[e];
        else
            tmp[rbase + r++] = ids[e];
    }
}

// one CTA per chunk: the partitioned chunk back into order; the node's first
// chunk's thread 0 writes the node's box and makes its children
__global__ void k_wide_finish(BNode* nodes, int* order, const int* tmp, const WideChunk* chunks, const int* n_chunks,
                              const WideAcc* acc, int* next, int* n_next, int* n_nodes) {
    if (int(blockIdx.x) >= *n_chunks) return;
    const WideChunk ch = chunks[blockIdx.x];
    const WideAcc& a = acc[ch.acc];
    if (a.split >= 0)
        for (int i = ch.lo + threadIdx.x; i < ch.hi; i += blockDim.x) order[i] = tmp[i];
    if (threadIdx.x != 0 || int(blockIdx.x) != a.c0) return;
    const int id = ch.node;
    const int first = nodes[id].first, count = nodes[id].count;
    BNode& nd = nodes[id];  // field by field: tri_area is the side stream's
    nd.lo = V3{okey_inv(a.box[0]), okey_inv(a.box[1]), okey_inv(a.box[2])};
    nd.hi = V3{okey_inv(a.box[6]), okey_inv(a.box[7]), okey_inv(a.box[8])};
    nd.left = nd.right = -1;
    int mid = first + count / 2;
    if (a.split >= 0) {
        mid = first + a.n_left;
        if (mid == first || mid == first + count) mid = first + count / 2;
    }
    make_children(nodes, id, first, count, mid, next, n_next, n_nodes);
}

// side stream: tri_area of the level's wide nodes, the sequential sum over the
// snapshot (staged through shared memory, one thread adds)
__global__ void __launch_bounds__(kBuildThreads) k_wide_area(BNode* nodes, const int* tasks, int nw,
                                                             const double* area_snap) {
    const int k = blockIdx.x;
    if (k >= nw) return;
    const int id = tasks[k];
    const int first = nodes[id].first, count = nodes[id].count;
    __shared__ double s_area[2][2048];
    double area = 0;
    int buf = 0;
    for (int k2 = threadIdx.x; k2 < min(2048, count); k2 += blockDim.x) s_area[0][k2] = area_snap[first + k2];
    __syncthreads();
    for (int base = first; base < first + count; base += 2048) {
        const int m = min(2048, first + count - base), nb = base + 2048;
        if (threadIdx.x == 0) {
            const double* a = s_area[buf];
            int j = 0;
            for (; j + 16 <= m; j += 16) {  // 16 loads ahead of the dependent adds
                double x[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) x[q] = a[j + q];
#pragma unroll
                for (int q = 0; q < 16; ++q) area += x[q];
            }
            for (; j < m; ++j) area += a[j];
        } else if (threadIdx.x >= 32 && nb < first + count) {  // the next block (warps 1..) while thread 0 adds
            for (int k2 = threadIdx.x - 32; k2 < min(2048, first + count - nb); k2 += blockDim.x - 32)
                s_area[buf ^ 1][k2] = area_snap[nb + k2];
        }
        __syncthreads();
        buf ^= 1;
    }
    if (threadIdx.x == 0) nodes[id].tri_area = area;
}

// subtree sizes, bottom-up over one level's nodes
__global__ void k_bvh_sizes(const BNode* nodes, const int* level, int n, int* size) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int id = level[k];
    const BNode& nd = nodes[id];
    size[id] = nd.left < 0 ? 1 : 1 + size[nd.left] + size[nd.right];
}
// pre-order indices and escape links, top-down over one level's nodes
// (pack_frame: esc[right] = left, esc[left] = esc[parent])
__global__ void k_bvh_preorder(const BNode* nodes, const int* level, int n, const int* size, int* pre, int* esc) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int id = level[k];
    const BNode& nd = nodes[id];
    if (nd.left < 0) return;
    pre[nd.left] = pre[id] + 1;
    pre[nd.right] = pre[id] + 1 + size[nd.left];
    esc[nd.right] = pre[nd.left];
    esc[nd.left] = esc[id];
}
// node arrays of the snapshot (GNode, GNodeAux) at pre-order positions, and the
// leaf of every triangle
__global__ void k_bvh_pack_nodes(const BNode* nodes, int nn, const int* pre, const int* esc, const int* order,
                                 GNode* gn, GNodeAux* ga, GTriInfo* info) {
    int id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= nn) return;
    const BNode& h = nodes[id];
    const int p = pre[id];
    const bool leaf = h.left < 0;
    GNode g;
    g.lo[0] = h.lo.x;
    g.lo[1] = h.lo.y;
    g.lo[2] = h.lo.z;
    g.hi[0] = h.hi.x;
    g.hi[1] = h.hi.y;
    g.hi[2] = h.hi.z;
    g.first = leaf ? h.first : 0;
    g.count = leaf ? h.count : 0;
    g.miss_next = esc[id];
    g.hit_next = leaf ? esc[id] : pre[h.right];
    gn[p] = g;
    GNodeAux a;
    a.tri_area = h.tri_area;
    a.left = leaf ? -1 : pre[h.left];
    a.right = leaf ? -1 : pre[h.right];
    a.parent = h.parent < 0 ? -1 : pre[h.parent];
    a.first = g.first;
    a.count = g.count;
    a.pad = 0;
    ga[p] = a;
    if (leaf)
        for (int i = h.first; i < h.first + h.count; ++i) {
            info[order[i]].leaf = p;
            info[order[i]].leaf_slot = i;
        }
}
// per-triangle arrays: leaf-order intersection records, ids, info, tangent frames
__global__ void k_bvh_pack_tris(const BTri* tris, const int* order, int nt, GTriIsect* isect, int* tri_id,
                                GTriInfo* info, Frame2* tframe) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nt) return;
    const BTri& o = tris[order[j]];
    isect[j].v0 = o.v0;
    isect[j].e1 = o.v1 - o.v0;
    isect[j].e2 = o.v2 - o.v0;
    tri_id[j] = order[j];
    const BTri& t = tris[j];  // info and frames by original triangle id
    GTriInfo& in = info[j];
    in.n = t.n;
    in.mat = t.material;
    in.obj = t.object;
    in.area = t.area;
    in.pad2 = 0;
    tframe[j] = tangent_frame_of(t.n, t.v1 - t.v0, t.v2 - t.v0);
}
__global__ void k_iota(int* a, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = i;
}

void ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw std::runtime_error(std::string("device bvh ") + what + ": " + cudaGetErrorString(e));
    }
}

}  // namespace

DeviceBvh::~DeviceBvh() { release(); }
void DeviceBvh::release() {
    for (void** p : {&tris, &order, &tmp, &nodes, &bfs, &next_lists, &size, &pre, &esc, &ctr, &host_ctr, &acc, &chunks,
                     &chunk_left, &area_snap}) {
        if (*p) {
            if (p == &host_ctr)
                cudaFreeHost(*p);
            else
                cudaFree(*p);
            *p = nullptr;
        }
    }
    if (fork) cudaEventDestroy(fork);
    fork = nullptr;
    for (cudaEvent_t& e : slot_done) {
        if (e) cudaEventDestroy(e);
        e = nullptr;
    }
    for (cudaStream_t& q : side) {
        if (q) cudaStreamDestroy(q);
        q = nullptr;
    }
    cap = 0;
}
void DeviceBvh::ensure(int nt) {
    if (nt <= cap) return;
    release();
    const size_t n = size_t(nt), nn = 2 * n, nw = n / kWideNode + 4, nch = n / kChunk + nw + 4;
    ok(cudaMalloc(&tris, n * sizeof(BTri)), "alloc");
    ok(cudaMalloc(&order, n * sizeof(int)), "alloc");
    ok(cudaMalloc(&tmp, n * sizeof(int)), "alloc");
    ok(cudaMalloc(&nodes, nn * sizeof(BNode)), "alloc");
    ok(cudaMalloc(&bfs, nn * sizeof(int)), "alloc");
    // next level's lists: big at 0, small at 2n, wide at 4n (n <= nt nodes per level)
    ok(cudaMalloc(&next_lists, (4 * n + nw + 16) * sizeof(int)), "alloc");
    ok(cudaMalloc(&size, nn * sizeof(int)), "alloc");
    ok(cudaMalloc(&pre, nn * sizeof(int)), "alloc");
    ok(cudaMalloc(&esc, nn * sizeof(int)), "alloc");
    ok(cudaMalloc(&ctr, 32), "alloc");
    ok(cudaMallocHost(&host_ctr, 32), "alloc");
    ok(cudaMalloc(&acc, nw * sizeof(WideAcc)), "alloc");
    ok(cudaMalloc(&chunks, nch * sizeof(WideChunk)), "alloc");
    ok(cudaMalloc(&chunk_left, nch * sizeof(int)), "alloc");
    ok(cudaMalloc(&area_snap, kAreaSlots * n * sizeof(double)), "alloc");
    ok(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming), "event");
    side.assign(kAreaSlots, nullptr);
    for (cudaStream_t& q : side) ok(cudaStreamCreateWithFlags(&q, cudaStreamNonBlocking), "stream");
    slot_done.assign(kAreaSlots, nullptr);
    for (cudaEvent_t& e : slot_done) ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    cap = nt;
}

// the level's wide nodes (tasks[0, nw)): chunk plan, the five chunked passes,
// the per-node finish; their tri_area sums on the side stream
void DeviceBvh::wide_level(const int* tasks, int nw, int wide_levels, cudaStream_t s) {
    const BTri* tr = static_cast<const BTri*>(tris);
    int* ord = static_cast<int*>(order);
    int* tm = static_cast<int*>(tmp);
    BNode* nd = static_cast<BNode*>(nodes);
    WideAcc* ac = static_cast<WideAcc*>(acc);
    WideChunk* ch = static_cast<WideChunk*>(chunks);
    int* cl = static_cast<int*>(chunk_left);
    int* ctr_i = static_cast<int*>(ctr);
    int* nxt = static_cast<int*>(next_lists);
    const int slot = wide_levels % kAreaSlots;
    double* snap = static_cast<double*>(area_snap) + size_t(slot) * size_t(nt);
    if (wide_levels >= kAreaSlots) ok(cudaStreamWaitEvent(s, slot_done[size_t(slot)], 0), "wait");  // slot's last sums
    const int grid = nt / kChunk + nw + 1;
    {
        KScope ks("k_wide_plan", s);
        k_wide_plan<<<1, 1, 0, s>>>(nd, tasks, nw, ac, ch, ctr_i + 6);
    }
    {
        KScope ks("k_wide_reset", s);
        k_wide_reset<<<nw, 64, 0, s>>>(ac, nw);
    }
    {
        KScope ks("k_wide_bounds", s);
        k_wide_bounds<<<grid, kBuildThreads, 0, s>>>(tr, ord, ch, ctr_i + 6, ac, snap);
    }
    ok(cudaEventRecord(fork, s), "record");
    cudaStream_t q = side[size_t(slot)];  // a stream per slot: the levels' sums run concurrently
    ok(cudaStreamWaitEvent(q, fork, 0), "wait");
    {
        KScope ks("k_wide_area", q);
        k_wide_area<<<nw, kBuildThreads, 0, q>>>(nd, tasks, nw, snap);
    }
    ok(cudaEventRecord(slot_done[size_t(slot)], q), "record");
    {
        KScope ks("k_wide_bins", s);
        k_wide_bins<<<grid, kBuildThreads, 0, s>>>(tr, ord, ch, ctr_i + 6, ac);
    }
    {
        KScope ks("k_wide_count", s);
        k_wide_count<<<grid, kBuildThreads, 0, s>>>(tr, ord, ch, ctr_i + 6, ac, cl);
    }
    {
        KScope ks("k_wide_scatter", s);
        k_wide_scatter<<<grid, kBuildThreads, 0, s>>>(tr, ord, tm, nd, ch, ctr_i + 6, ac, cl);
    }
    {
        KScope ks("k_wide_finish", s);
        k_wide_finish<<<grid, kBuildThreads, 0, s>>>(nd, ord, tm, ch, ctr_i + 6, ac, nxt, ctr_i + 1, ctr_i);
    }
}

int DeviceBvh::build(const void* host_tris, int n_tris, cudaStream_t s) {
    const int nt = n_tris;
    static_assert(sizeof(BTri) == 112, "BTri mirrors HTri");
    ensure(nt);
    this->nt = nt;
    ok(cudaMemcpyAsync(tris, host_tris, size_t(nt) * sizeof(BTri), cudaMemcpyHostToDevice, s), "upload");
    {
        KScope ks("k_iota", s);
        k_iota<<<(nt + 255) / 256, 256, 0, s>>>(static_cast<int*>(order), nt);
    }
    BNode root{};
    root.first = 0;
    root.count = nt;
    root.parent = -1;
    ok(cudaMemcpyAsync(nodes, &root, sizeof(BNode), cudaMemcpyHostToDevice, s), "root");
    int* bfs_i = static_cast<int*>(bfs);
    int* nxt = static_cast<int*>(next_lists);
    // [0] nodes made; the next level's [1] big tasks, [2] small tasks, [3] the
    // small list's offset in `nxt`, [4] wide tasks, [5] the wide list's offset;
    // [6] the wide level's chunks
    int* ctr_i = static_cast<int*>(ctr);
    int* hc = static_cast<int*>(host_ctr);
    const int root_kind = nt <= kSmallNode ? 1 : (nt > kWideNode ? 2 : 0);
    int init[4] = {1, 0, 0, 0};
    ok(cudaMemcpyAsync(ctr_i, init, 16, cudaMemcpyHostToDevice, s), "ctr");
    ok(cudaMemcpyAsync(bfs_i, &init[3], 4, cudaMemcpyHostToDevice, s), "bfs");  // level 0 = node 0
    level_off.assign(1, 0);
    level_n.assign(1, 1);
    level_nw.assign(1, root_kind == 2 ? 1 : 0);
    level_nb.assign(1, root_kind == 0 ? 1 : 0);
    int wide_levels = 0;
    for (int L = 0; level_n.back() > 0; ++L) {
        if (L > 62) throw std::runtime_error("bvh deeper than supported");
        const int off = level_off.back(), n = level_n.back(), nw = level_nw.back(), nb = level_nb.back();
        const int ns = n - nw - nb;
        int c[5] = {0, 0, 2 * n, 0, 4 * n};  // children of n nodes: <= 2n per list
        ok(cudaMemcpyAsync(ctr_i + 1, c, 20, cudaMemcpyHostToDevice, s), "ctr");
        if (nw) wide_level(bfs_i + off, nw, wide_levels++, s);
        if (nb) {
            KScope ks("k_bvh_level", s);
            k_bvh_level<<<nb, kBuildThreads, 0, s>>>(static_cast<const BTri*>(tris), static_cast<int*>(order),
                                                      static_cast<int*>(tmp), static_cast<BNode*>(nodes),
                                                      bfs_i + off + nw, nb, nxt, ctr_i + 1, ctr_i);
        }
        if (ns) {
            KScope ks("k_bvh_level_warp", s);
            k_bvh_level_warp<<<(ns + kWarpNodes - 1) / kWarpNodes, 32 * kWarpNodes, 0, s>>>(
                static_cast<const BTri*>(tris), static_cast<int*>(order), static_cast<BNode*>(nodes),
                bfs_i + off + nw + nb, ns, nxt, ctr_i + 1, ctr_i);
        }
        ok(cudaMemcpyAsync(hc, ctr_i, 20, cudaMemcpyDeviceToHost, s), "ctr");
        ok(cudaStreamSynchronize(s), "level");
        const int nb2 = hc[1], ns2 = hc[2], nw2 = hc[4];
        // the next level: [wide tasks | big tasks | small tasks], contiguous after this one
        int* dst = bfs_i + off + n;
        if (nw2) ok(cudaMemcpyAsync(dst, nxt + 4 * n, size_t(nw2) * 4, cudaMemcpyDeviceToDevice, s), "level");
        if (nb2) ok(cudaMemcpyAsync(dst + nw2, nxt, size_t(nb2) * 4, cudaMemcpyDeviceToDevice, s), "level");
        if (ns2) ok(cudaMemcpyAsync(dst + nw2 + nb2, nxt + 2 * n, size_t(ns2) * 4, cudaMemcpyDeviceToDevice, s), "level");
        level_off.push_back(off + n);
        level_n.push_back(nw2 + nb2 + ns2);
        level_nw.push_back(nw2);
        level_nb.push_back(nb2);
    }
    n_nodes = hc[0];
    depth = int(level_n.size()) - 1;
    ok(cudaGetLastError(), "levels");
    // the reference's depth-first numbering: subtree sizes, then pre-order
    const BNode* nd = static_cast<const BNode*>(nodes);
    for (int L = depth - 1; L >= 0; --L) {
        int n = level_n[L];
        KScope ks("k_bvh_sizes", s);
        k_bvh_sizes<<<(n + 255) / 256, 256, 0, s>>>(nd, bfs_i + level_off[L], n, static_cast<int*>(size));
    }
    int root_pre_esc[2] = {0, -1};
    ok(cudaMemcpyAsync(pre, &root_pre_esc[0], 4, cudaMemcpyHostToDevice, s), "pre");
    ok(cudaMemcpyAsync(esc, &root_pre_esc[1], 4, cudaMemcpyHostToDevice, s), "esc");
    for (int L = 0; L < depth; ++L) {
        int n = level_n[L];
        KScope ks("k_bvh_preorder", s);
        k_bvh_preorder<<<(n + 255) / 256, 256, 0, s>>>(nd, bfs_i + level_off[L], n, static_cast<int*>(size),
                                                        static_cast<int*>(pre), static_cast<int*>(esc));
    }
    if (wide_levels) {  // the side stream's tri_area sums before anything reads the nodes
        for (int q = 0; q < std::min(wide_levels, kAreaSlots); ++q)
            ok(cudaStreamWaitEvent(s, slot_done[size_t(q)], 0), "wait");
    }
    ok(cudaGetLastError(), "pre-order");
    return n_nodes;
}

void DeviceBvh::pack(unsigned char* blob, const PackedFrame& shell, cudaStream_t s) {
    const int nt = shell.view.n_tris;
    const BNode* nd = static_cast<const BNode*>(nodes);
    GTriInfo* info = reinterpret_cast<GTriInfo*>(blob + shell.off_tri);
    {
        KScope ks("k_bvh_pack_tris", s);
        k_bvh_pack_tris<<<(nt + 255) / 256, 256, 0, s>>>(
            static_cast<const BTri*>(tris), static_cast<const int*>(order), nt,
            reinterpret_cast<GTriIsect*>(blob + shell.off_isect), reinterpret_cast<int*>(blob + shell.off_tri_id),
            info, reinterpret_cast<Frame2*>(blob + shell.off_tframe));
    }
    {
        KScope ks("k_bvh_pack_nodes", s);
        k_bvh_pack_nodes<<<(n_nodes + 255) / 256, 256, 0, s>>>(
            nd, n_nodes, static_cast<const int*>(pre), static_cast<const int*>(esc), static_cast<const int*>(order),
            reinterpret_cast<GNode*>(blob + shell.off_nodes), reinterpret_cast<GNodeAux*>(blob + shell.off_aux), info);
    }
    ok(cudaGetLastError(), "pack");
}

void DeviceBvh::dump(double* nodes_out, int32_t* parent_out, int32_t* order_out, cudaStream_t s) {
    // the host builder's dump layout (tofr_scene_dump_bvh): per node lo, hi,
    // tri_area, left, right, first, count in pre-order, the parents, tri_order
    std::vector<BNode> h(static_cast<size_t>(n_nodes));
    std::vector<int> pre_h(static_cast<size_t>(n_nodes));
    ok(cudaMemcpyAsync(h.data(), nodes, h.size() * sizeof(BNode), cudaMemcpyDeviceToHost, s), "dump");
    ok(cudaMemcpyAsync(pre_h.data(), pre, pre_h.size() * sizeof(int), cudaMemcpyDeviceToHost, s), "dump");
    ok(cudaMemcpyAsync(order_out, order, size_t(nt) * sizeof(int), cudaMemcpyDeviceToHost, s), "dump");
    ok(cudaStreamSynchronize(s), "dump");
    for (size_t id = 0; id < h.size(); ++id) {
        const BNode& b = h[id];
        double* o = nodes_out + 11 * size_t(pre_h[id]);
        const bool leaf = b.left < 0;
        o[0] = b.lo.x;
        o[1] = b.lo.y;
        o[2] = b.lo.z;
        o[3] = b.hi.x;
        o[4] = b.hi.y;
        o[5] = b.hi.z;
        o[6] = b.tri_area;
        o[7] = leaf ? -1 : pre_h[size_t(b.left)];
        o[8] = leaf ? -1 : pre_h[size_t(b.right)];
        o[9] = leaf ? b.first : 0;
        o[10] = leaf ? b.count : 0;
        parent_out[pre_h[id]] = b.parent < 0 ? -1 : pre_h[size_t(b.parent)];
    }
}

}  // namespace tofr_b200
