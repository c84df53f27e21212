// context.cuh -- the bsg_ctx object behind the C ABI: device binding, cached
// device workspace (grown on demand, never freed on the warm path), host
// staging for BSG_MEM_HOST calls, launch accounting and error reporting.
#pragma once
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

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
    bsg::DevBuf proto; // protocol-check flag word (bsp_error equivalent, pr.cu)
    bsg::DevBuf mt_ws; // device generator: segment start windows + jump polynomials
    bsg::DevBuf msd_ws; // hybrid route: plan, 16-bit histogram, reservations (msd.cu)
    // Cross-stream ordering of the shared workspace: every call records
    // `last_use` on its stream; a call on a different stream first waits on
    // it, so device-mode calls issued on two streams never run on the same
    // scratch buffers at once (the mutex alone only serialises the host side).
    cudaEvent_t last_use = nullptr;
    cudaStream_t last_stream = nullptr;
    bool used = false;

    // Multi-GPU group (bsg_ctx_create_group): one member context per listed
    // device (owned), each with its own workspace and stream; peer access
    // enabled between distinct member devices; NCCL communicators built
    // lazily by the first BSG_PR_NCCL call (ncclCommInitAll over the
    // members).  Empty for single-device contexts.
    std::vector<bsg_ctx*> members;
    std::vector<cudaStream_t> member_streams;
    bool peer_ok = true;    // every pair of distinct member devices can reach each other
    void* nccl = nullptr;   // bsg::NcclGroup* (pr.cu)
    bsg::DevBuf grp_cur, grp_nxt, grp_recv; // per-member range buffers (members only)
    // pinned chunk buffers for pageable BSG_MEM_HOST copies (staging.cu)
    void* pin_buf[2] = {nullptr, nullptr};
    cudaEvent_t pin_ev[2] = {nullptr, nullptr};

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

// Host<->device copies of BSG_MEM_HOST calls (staging.cu): pageable host
// memory is pipelined through the context's pinned chunk buffers.
int copy_h2d(bsg_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t s);
int copy_d2h(bsg_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t s);
void release_stage(bsg_ctx* c);

// RAII: order this call's stream after the context's previous call (see
// bsg_ctx::last_use).  Construct with the context mutex held and the
// context's device current.
struct StreamOrder {
    bsg_ctx* c;
    cudaStream_t s;
    StreamOrder(bsg_ctx* ctx, cudaStream_t stream) : c(ctx), s(stream) {
        if (c->used && c->last_stream != s) cudaStreamWaitEvent(s, c->last_use, 0);
    }
    ~StreamOrder() {
        if (!c->last_use && cudaEventCreateWithFlags(&c->last_use, cudaEventDisableTiming) != cudaSuccess) {
            c->last_use = nullptr;
            return;
        }
        if (cudaEventRecord(c->last_use, s) == cudaSuccess) {
            c->last_stream = s;
            c->used = true;
        }
    }
};

} // namespace bsg
