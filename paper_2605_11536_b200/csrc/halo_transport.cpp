// halo_transport.cpp -- NCCL and in-process peer transports of the row-band
// halos (see halo_transport.h).
#include "halo_transport.h"

#include <dlfcn.h>
#include <nccl.h>  // types and enums only: the entry points are dlopen'ed

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <type_traits>

namespace tofr_b200 {

namespace {

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw std::runtime_error(std::string("halo ") + what + ": " + cudaGetErrorString(e));
    }
}

// ---------------------------------------------------------------------------
// NCCL, loaded at run time.  A process that already loaded libnccl.so.2 (e.g.
// torch.distributed's) gets that same library back from dlopen.

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            return fn != nullptr;
        };
        a.ok = sym(a.GetUniqueId, "ncclGetUniqueId") && sym(a.CommInitRank, "ncclCommInitRank") &&
               sym(a.CommDestroy, "ncclCommDestroy") && sym(a.Send, "ncclSend") && sym(a.Recv, "ncclRecv") &&
               sym(a.GroupStart, "ncclGroupStart") && sym(a.GroupEnd, "ncclGroupEnd") &&
               sym(a.GetErrorString, "ncclGetErrorString");
        return a;
    }();
    return api;
}

void nccl_ok(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw std::runtime_error(std::string("halo nccl ") + what + ": " +
                                 (nccl().GetErrorString ? nccl().GetErrorString(r) : "error"));
}

struct NcclHaloTransport : HaloTransport {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
    ~NcclHaloTransport() override {
        if (comm) nccl().CommDestroy(comm);
    }
    // send_lo (this band's top rows) goes to the band above (rank - 1), which
    // receives it in its recv_hi; send_hi goes to rank + 1's recv_lo.  Both
    // directions in one group: NCCL pairs the sends and receives and runs them
    // on the session stream after the pack kernels.
    void exchange(const HaloBufs& b, int) override {
        const NcclApi& n = nccl();
        nccl_ok(n.GroupStart(), "group start");
        // the group is always closed, also when an enqueue fails
        ncclResult_t r = ncclSuccess;
        if (rank > 0 && b.bytes_lo) {
            if (r == ncclSuccess) r = n.Send(b.send_lo, b.bytes_lo, ncclUint8, rank - 1, comm, b.stream);
            if (r == ncclSuccess) r = n.Recv(b.recv_lo, b.bytes_lo, ncclUint8, rank - 1, comm, b.stream);
        }
        if (rank < world - 1 && b.bytes_hi) {
            if (r == ncclSuccess) r = n.Send(b.send_hi, b.bytes_hi, ncclUint8, rank + 1, comm, b.stream);
            if (r == ncclSuccess) r = n.Recv(b.recv_hi, b.bytes_hi, ncclUint8, rank + 1, comm, b.stream);
        }
        ncclResult_t e = n.GroupEnd();
        nccl_ok(r, "send/recv");
        nccl_ok(e, "group end");
    }
    const char* name() const override { return "nccl"; }
};

}  // namespace

bool nccl_available() { return nccl().ok; }

void nccl_unique_id(uint8_t out[128]) {
    if (!nccl().ok) throw std::runtime_error("libnccl.so.2 not loadable");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    nccl_ok(nccl().GetUniqueId(&id), "unique id");
    std::memcpy(out, &id, 128);
}

std::unique_ptr<HaloTransport> make_nccl_transport(const uint8_t id[128], int rank, int world, int device) {
    if (!nccl().ok) throw std::runtime_error("libnccl.so.2 not loadable");
    if (world < 1 || rank < 0 || rank >= world) throw std::runtime_error("halo nccl: bad rank / world");
    auto t = std::make_unique<NcclHaloTransport>();
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    cuda_ok(cudaSetDevice(device), "set device");
    nccl_ok(nccl().CommInitRank(&t->comm, world, uid, rank), "comm init");
    t->rank = rank;
    t->world = world;
    return t;
}

// ---------------------------------------------------------------------------
// in-process peer transport

struct PeerEndpoint {
    HaloBufs bufs;
    cudaEvent_t packed = nullptr;  // recorded after this band's pack kernels
    cudaEvent_t copied = nullptr;  // recorded after this band's copies from its neighbours
    std::weak_ptr<PeerEndpoint> up, down;  // the bands above (smaller rows) and below
    std::mutex mu;
    std::condition_variable cv;
    int64_t gen = 0;         // exchanges this band started
    int64_t packed_gen = 0;  // `packed` holds the record of exchange packed_gen
    int64_t copied_gen = 0;  // `copied` holds the record of exchange copied_gen
    ~PeerEndpoint() {
        if (packed) cudaEventDestroy(packed);
        if (copied) cudaEventDestroy(copied);
    }
};

namespace {

void publish(PeerEndpoint& e, int64_t PeerEndpoint::*field, int64_t g) {
    {
        std::lock_guard<std::mutex> lk(e.mu);
        e.*field = g;
    }
    e.cv.notify_all();
}

// host wait until the neighbour has ENQUEUED (recorded) its event of exchange g
void await(PeerEndpoint& n, int64_t PeerEndpoint::*field, int64_t g) {
    std::unique_lock<std::mutex> lk(n.mu);
    if (!n.cv.wait_for(lk, std::chrono::seconds(120), [&] { return n.*field >= g; }))
        throw std::runtime_error("halo peer: neighbour band did not reach the exchange (drive each band from its "
                                 "own host thread)");
}

struct PeerHaloTransport : HaloTransport {
    std::shared_ptr<PeerEndpoint> self;
    void before_pack(const HaloBufs&) override {
        PeerEndpoint& s = *self;
        if (s.gen == 0) return;
        for (auto* w : {&s.up, &s.down}) {
            auto n = w->lock();
            if (!n) continue;
            await(*n, &PeerEndpoint::copied_gen, s.gen);  // its copies out of our send buffers
            cuda_ok(cudaStreamWaitEvent(s.bufs.stream, n->copied, 0), "wait");
        }
    }
    void exchange(const HaloBufs&, int) override {
        PeerEndpoint& s = *self;
        const int64_t g = ++s.gen;
        cuda_ok(cudaEventRecord(s.packed, s.bufs.stream), "record");
        publish(s, &PeerEndpoint::packed_gen, g);
        if (auto n = s.up.lock()) {  // our top halo rows = the band above's bottom owned rows
            if (n->bufs.bytes_hi != s.bufs.bytes_lo) throw std::runtime_error("halo peer: band halo sizes differ");
            await(*n, &PeerEndpoint::packed_gen, g);
            cuda_ok(cudaStreamWaitEvent(s.bufs.stream, n->packed, 0), "wait");
            cuda_ok(cudaMemcpyPeerAsync(s.bufs.recv_lo, s.bufs.device, n->bufs.send_hi, n->bufs.device,
                                        s.bufs.bytes_lo, s.bufs.stream),
                    "peer copy");
        }
        if (auto n = s.down.lock()) {
            if (n->bufs.bytes_lo != s.bufs.bytes_hi) throw std::runtime_error("halo peer: band halo sizes differ");
            await(*n, &PeerEndpoint::packed_gen, g);
            cuda_ok(cudaStreamWaitEvent(s.bufs.stream, n->packed, 0), "wait");
            cuda_ok(cudaMemcpyPeerAsync(s.bufs.recv_hi, s.bufs.device, n->bufs.send_lo, n->bufs.device,
                                        s.bufs.bytes_hi, s.bufs.stream),
                    "peer copy");
        }
        cuda_ok(cudaEventRecord(s.copied, s.bufs.stream), "record");
        publish(s, &PeerEndpoint::copied_gen, g);
    }
    const char* name() const override { return "peer"; }
};

}  // namespace

std::shared_ptr<PeerEndpoint> make_peer_endpoint(const HaloBufs& bufs) {
    auto e = std::make_shared<PeerEndpoint>();
    e->bufs = bufs;
    cuda_ok(cudaSetDevice(bufs.device), "set device");
    cuda_ok(cudaEventCreateWithFlags(&e->packed, cudaEventDisableTiming), "event");
    cuda_ok(cudaEventCreateWithFlags(&e->copied, cudaEventDisableTiming), "event");
    return e;
}

void peer_link(const std::shared_ptr<PeerEndpoint>& upper, const std::shared_ptr<PeerEndpoint>& lower) {
    if (upper->gen || lower->gen) throw std::runtime_error("halo peer: link bands before their first frame");
    upper->down = lower;
    lower->up = upper;
    int a = upper->bufs.device, b = lower->bufs.device;
    if (a != b) {  // NVLink P2P between the two devices (both directions)
        int ab = 0, ba = 0;
        cudaDeviceCanAccessPeer(&ab, a, b);
        cudaDeviceCanAccessPeer(&ba, b, a);
        int cur = 0;
        cudaGetDevice(&cur);
        if (ab) {
            cudaSetDevice(a);
            cudaDeviceEnablePeerAccess(b, 0);
        }
        if (ba) {
            cudaSetDevice(b);
            cudaDeviceEnablePeerAccess(a, 0);
        }
        cudaGetLastError();  // "already enabled" is fine; without P2P the copies stage through the host
        cudaSetDevice(cur);
    }
}

std::unique_ptr<HaloTransport> make_peer_transport(const std::shared_ptr<PeerEndpoint>& self) {
    auto t = std::make_unique<PeerHaloTransport>();
    t->self = self;
    return t;
}

}  // namespace tofr_b200
