// ktime.cpp -- see ktime.h
#include "ktime.h"

#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

namespace tofr_b200 {
namespace {

struct Pending {
    int kernel;
    int device;
    cudaEvent_t a, b;
};

struct Totals {
    double ms = 0;
    uint64_t launches = 0;
};

std::mutex mu;
std::atomic<bool> enabled{false};
std::atomic<uint64_t> launches{0};
std::vector<std::string> names;
std::map<std::string, int> index;
std::vector<Totals> totals;
std::vector<Pending> pending;
std::map<int, std::vector<cudaEvent_t>> pool;  // free events per device

int kernel_id(const char* name) {
    auto it = index.find(name);
    if (it != index.end()) return it->second;
    int id = int(names.size());
    names.emplace_back(name);
    index.emplace(name, id);
    totals.emplace_back();
    return id;
}

cudaEvent_t take_event(int dev) {
    auto& v = pool[dev];
    if (!v.empty()) {
        cudaEvent_t e = v.back();
        v.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

}  // namespace

KScope::KScope(const char* name, cudaStream_t s) : slot(-1), stream(s) {
    launches.fetch_add(1, std::memory_order_relaxed);
    if (!enabled.load(std::memory_order_relaxed)) return;
    std::lock_guard<std::mutex> g(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    Pending p{kernel_id(name), dev, take_event(dev), take_event(dev)};
    cudaEventRecord(p.a, s);
    slot = int(pending.size());
    pending.push_back(p);
}

KScope::~KScope() {
    if (slot < 0) return;
    std::lock_guard<std::mutex> g(mu);
    if (slot < int(pending.size())) cudaEventRecord(pending[slot].b, stream);
}

void kt_set_enabled(bool on) { enabled.store(on); }
bool kt_enabled() { return enabled.load(); }
uint64_t kt_launches() { return launches.load(); }

void kt_collect() {
    std::lock_guard<std::mutex> g(mu);
    std::vector<Pending> keep;
    for (const Pending& p : pending) {
        if (cudaEventQuery(p.b) != cudaSuccess) {
            keep.push_back(p);
            continue;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, p.a, p.b);
        totals[p.kernel].ms += ms;
        totals[p.kernel].launches++;
        pool[p.device].push_back(p.a);
        pool[p.device].push_back(p.b);
    }
    cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not an error
    pending.swap(keep);
}

int kt_read(char* out_names, int name_len, double* ms, uint64_t* n, int cap) {
    std::lock_guard<std::mutex> g(mu);
    int k = 0;
    for (size_t i = 0; i < names.size() && k < cap; ++i) {
        if (!totals[i].launches) continue;
        if (out_names && name_len > 0) {
            std::strncpy(out_names + size_t(k) * name_len, names[i].c_str(), size_t(name_len) - 1);
            out_names[size_t(k) * name_len + name_len - 1] = 0;
        }
        if (ms) ms[k] = totals[i].ms;
        if (n) n[k] = totals[i].launches;
        ++k;
    }
    return k;
}

void kt_reset() {
    std::lock_guard<std::mutex> g(mu);
    for (Totals& t : totals) t = Totals{};
}

}  // namespace tofr_b200
