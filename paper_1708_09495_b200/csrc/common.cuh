// common.cuh -- shared device helpers for the sm_100a kernels (PTX wrappers
// for relaxed/acquire global accesses, mbarrier + cp.async.bulk (TMA bulk
// copy), lane masks) and the launch-accounting hook.
#pragma once
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

namespace bsg {

constexpr int kSmCountB200 = 148;
constexpr int kMaxDevices = 64;

// Kernel attributes (max dynamic shared memory) are per device, so every
// launcher caches "attribute set + resident CTAs per SM" per device ordinal:
// a context on cuda:1 must not launch a >48 KB-smem kernel whose attribute
// was only set on cuda:0.  Returns the CTAs per SM (>= 1) for the current
// device.  Racing first calls from two host threads both set the same value.
struct PerDeviceOccupancy {
    int per_sm[kMaxDevices] = {};
};
template <typename K>
inline int kernel_occupancy(PerDeviceOccupancy& cache, K kern, int threads, size_t smem) {
    int dev = 0;
    cudaGetDevice(&dev);
    int& v = cache.per_sm[dev & (kMaxDevices - 1)];
    if (v == 0) {
        int per = 0;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, smem);
        v = per < 1 ? -1 : per; // -1: does not fit (recorded so it is not re-queried)
    }
    return v;
}
// Development knobs (BSG_OS_CFG, BSG_OS_RANK, BSG_SMALL, ...): environment
// variables are read only in development builds (-DBSG_DEV_KNOBS=1, see
// scripts/build_variant.sh); the product library always uses the defaults.
#ifndef BSG_DEV_KNOBS
#define BSG_DEV_KNOBS 0
#endif
inline int dev_knob(const char* name, int def) {
    if (!BSG_DEV_KNOBS) return def;
    const char* e = getenv(name);
    return e ? atoi(e) : def;
}
inline int current_sm_count() {
    int dev = 0, sms = kSmCountB200;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

__device__ __forceinline__ uint32_t lane_id() {
    uint32_t l;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(l));
    return l;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Relaxed gpu-scope accesses for decoupled look-back status words.  The
// status word carries its own payload (flag | count), so no ordering with
// other data is needed: relaxed atomicity is sufficient.
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_gpu(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Generic-proxy global writes (made visible by a grid barrier) -> visible to
// subsequent TMA (async-proxy) reads issued by this thread.
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Streaming 128-bit global load that does not allocate in L1.
__device__ __forceinline__ uint4 ldg_stream_v4(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// ---- mbarrier + bulk async copy (TMA engine, non-tensor form) -----------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared, completion signalled on `bar`.
// dst, src and bytes must be multiples of 16.
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <class T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= static_cast<uint32_t>(o)) v += u;
    }
    return v;
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

} // namespace bsg
