// halo_transport.h -- native transports of the row-band reservoir halos
// (one exchange step per spatial pass, up/down neighbour only).
//
// A band session packs its edge rows into send_lo / send_hi (rows it owns
// that the band above / below reads) and unpacks recv_lo / recv_hi (the
// neighbours' rows it reads).  A transport moves send -> the neighbour's recv
// on the session stream, with no host callback per pass:
//
//   * NcclHaloTransport   one process per GPU: ncclSend / ncclRecv with ranks
//                         rank - 1 and rank + 1 inside one NCCL group on the
//                         session stream (communicator from an ncclUniqueId the
//                         host side broadcasts; libnccl is dlopen'ed, so the
//                         library has no link-time NCCL dependency).
//   * PeerHaloTransport   several band sessions in one process (one host thread
//                         per band, any devices): cudaMemcpyPeerAsync from the
//                         neighbour's send buffer into this band's recv buffer
//                         (NVLink P2P when the devices differ), ordered by
//                         cross-stream events; host threads only wait for the
//                         neighbour to have *enqueued* its pack, never for the
//                         GPU.
//
// Errors throw std::runtime_error (mapped to TOFR_ERR_* by the C ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>

namespace tofr_b200 {

struct HaloBufs {
    void* send_lo = nullptr;
    void* recv_lo = nullptr;
    size_t bytes_lo = 0;
    void* send_hi = nullptr;
    void* recv_hi = nullptr;
    size_t bytes_hi = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
};

struct HaloTransport {
    virtual ~HaloTransport() = default;
    // before this band overwrites its send buffers (the neighbours must have
    // finished reading the previous exchange's rows)
    virtual void before_pack(const HaloBufs&) {}
    // after the pack kernels are enqueued: move the rows; unpack follows on the stream
    virtual void exchange(const HaloBufs&, int pass) = 0;
    virtual const char* name() const = 0;
};

// NCCL: true if libnccl could be loaded (dlopen libnccl.so.2)
bool nccl_available();
void nccl_unique_id(uint8_t out[128]);
std::unique_ptr<HaloTransport> make_nccl_transport(const uint8_t id[128], int rank, int world, int device);

// In-process peer links: one PeerEndpoint per band session; link(upper, lower)
// joins two adjacent bands (upper.y1 == lower.y0).
struct PeerEndpoint;
std::shared_ptr<PeerEndpoint> make_peer_endpoint(const HaloBufs& bufs);
void peer_link(const std::shared_ptr<PeerEndpoint>& upper, const std::shared_ptr<PeerEndpoint>& lower);
std::unique_ptr<HaloTransport> make_peer_transport(const std::shared_ptr<PeerEndpoint>& self);

}  // namespace tofr_b200
