// context.cuh -- the bsg_ctx object behind the C ABI: device binding, cached
// device workspace (grown on demand, never freed on the warm path), host
// staging for BSG_MEM_HOST calls, launch accounting and error reporting.
#pragma once
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <string>

#include <cuda_runtime.h>

#include "../../include/bsg.h"
#include "radix.cuh"
#include "timer.cuh"

namespace bsg {

void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

// A device buffer that only grows.
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t want) {
        if (want <= bytes) return cudaSuccess;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
        size_t b = want < 256 ? 256 : want;
        cudaError_t e = cudaMalloc(&ptr, b);
        if (e == cudaSuccess) bytes = b;
        return e;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
    }
    template <class T> T* as() const { return static_cast<T*>(ptr); }
};

} // namespace bsg

struct bsg_ctx {
    int device = 0;
    std::mutex mu;
    uint64_t launches = 0;
    bsg::KTimer timer;
    // radix workspace
    bsg::DevBuf tmp, status, hist, base, plan;
    // host-path staging and PR / network scratch
    bsg::DevBuf stage_in, stage_out, stage_b;
    bsg::DevBuf pr_counts, pr_sorted, pr_recv, pr_block, pr_misc, pr_delta;
    bsg::DevBuf net_sched, cnt32;
    bsg::DevBuf mt_ws; // device generator: segment start windows + jump polynomials

    // Ensures the radix workspace for n keys and returns a view of it.
    int radix_ws(uint64_t n, bsg::RadixWorkspace* ws);
};

namespace bsg {

// RAII: make ctx->device current for the duration of a call.
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) err = cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

} // namespace bsg
