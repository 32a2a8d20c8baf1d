// ktime.h -- launch accounting of the library's kernels.
//
// Every kernel launch goes through a KScope: it counts the launch and, when
// timing is enabled (tofr_gpu_kernel_timing), brackets it with CUDA events on
// the launching stream.  Completed pairs are folded into per-kernel totals by
// kt_collect() (called after a stream sync), so a caller (bench.py) gets each
// kernel's average launch duration measured live on its own stream.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tofr_b200 {

struct KScope {
    int slot;
    cudaStream_t stream;
    KScope(const char* name, cudaStream_t s);
    ~KScope();
    KScope(const KScope&) = delete;
    KScope& operator=(const KScope&) = delete;
};

void kt_set_enabled(bool on);
bool kt_enabled();
uint64_t kt_launches();  // cumulative launches of the library's kernels
void kt_collect();       // fold completed event pairs into the totals
// per-kernel totals: names (cap x name_len chars), total ms, launches; returns the count
int kt_read(char* names, int name_len, double* ms, uint64_t* launches, int cap);
void kt_reset();

}  // namespace tofr_b200
