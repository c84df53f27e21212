// timer.cuh -- optional per-launch CUDA-event timing of kernel classes on the
// launching stream (bsg_ctx_set_timing / bsg_ctx_get_timing).  bench.py uses
// it to time the dominant kernel live, inside its own timed loop's stream.
#pragma once
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

namespace bsg {

struct KTimer {
    bool enabled = false;
    struct Rec {
        int cls;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;

    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    void reset() {
        for (auto& r : recs) {
            pool.push_back(r.a);
            pool.push_back(r.b);
        }
        recs.clear();
    }
    ~KTimer() {
        reset();
        for (auto e : pool) cudaEventDestroy(e);
    }
};

// The timer of the context whose API call is running on this thread.
extern thread_local KTimer* tl_timer;

// Records CUDA events around the launches in its scope when timing is on.
struct TimedScope {
    KTimer* t;
    int cls;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    static const char* class_name(int c) {
        static const char* const names[] = {"K3 one-sweep pass", "K1 histogram", "block network", "PR plan/rebuild",
                                            "K3f first pass", "K3r value-stable pass", "hybrid: histogram + plan",
                                            "hybrid: byte partitions", "hybrid: local sort"};
        return c >= 0 && c < 9 ? names[c] : "kernel";
    }
    TimedScope(int cls_, cudaStream_t s_) : t(tl_timer), cls(cls_), s(s_) {
        nvtxRangePushA(class_name(cls_)); // the launches of one kernel class (host-side range)
        if (t && t->enabled) {
            a = t->get();
            cudaEventRecord(a, s);
        }
    }
    ~TimedScope() {
        nvtxRangePop();
        if (a) {
            cudaEvent_t b = t->get();
            cudaEventRecord(b, s);
            t->recs.push_back({cls, a, b});
        }
    }
};

} // namespace bsg
