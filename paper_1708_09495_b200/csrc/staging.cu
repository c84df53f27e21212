// staging.cu -- host<->device copies of BSG_MEM_HOST calls.  Pinned caller
// memory goes straight to cudaMemcpyAsync; PAGEABLE memory (a std::vector
// handed to the reference-style API) is pipelined through two pinned chunk
// buffers owned by the context: host threads copy chunk i+1 into one buffer
// while the copy engine moves chunk i out of the other (the driver's own
// pageable path runs at ~11 GB/s on the B200 hosts, pinned at ~55 GB/s).
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "context.cuh"

namespace bsg {

namespace {

constexpr size_t kStageChunk = size_t{64} << 20;  // bytes per pinned chunk
constexpr size_t kDirectBelow = size_t{4} << 20;  // small copies: plain cudaMemcpyAsync

bool is_pageable(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

// memcpy split over a few host threads (one host thread reaches ~14 GB/s)
void par_memcpy(void* dst, const void* src, size_t bytes) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t T = std::min<size_t>({8, std::max(1u, hw / 2), std::max<size_t>(1, bytes >> 22)});
    if (T <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const size_t part = (bytes / T + 63) & ~size_t{63};
    std::vector<std::thread> th;
    th.reserve(T - 1);
    for (size_t t = 1; t < T; ++t) {
        const size_t a = std::min(bytes, t * part), b = std::min(bytes, (t + 1) * part);
        if (b > a)
            th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a); });
    }
    std::memcpy(dst, src, std::min(bytes, part));
    for (auto& x : th) x.join();
}

int ensure_stage(bsg_ctx* c) {
    cudaError_t e;
    for (int i = 0; i < 2; ++i) {
        if (!c->pin_buf[i] && (e = cudaHostAlloc(&c->pin_buf[i], kStageChunk, cudaHostAllocDefault)) != cudaSuccess) {
            c->pin_buf[i] = nullptr;
            return cuda_fail(e, "pinned staging buffer");
        }
        if (!c->pin_ev[i] && (e = cudaEventCreateWithFlags(&c->pin_ev[i], cudaEventDisableTiming)) != cudaSuccess)
            return cuda_fail(e, "staging event");
    }
    return BSG_OK;
}

} // namespace

int copy_h2d(bsg_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t s) {
    cudaError_t e;
    if (bytes < kDirectBelow || !is_pageable(src)) {
        if ((e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s)) != cudaSuccess) return cuda_fail(e, "H2D copy");
        return BSG_OK;
    }
    if (int rc = ensure_stage(c)) return rc;
    for (size_t off = 0, i = 0; off < bytes; off += kStageChunk, ++i) {
        const int b = static_cast<int>(i & 1);
        const size_t len = std::min(kStageChunk, bytes - off);
        if (i >= 2 && (e = cudaEventSynchronize(c->pin_ev[b])) != cudaSuccess) return cuda_fail(e, "H2D staging");
        par_memcpy(c->pin_buf[b], static_cast<const char*>(src) + off, len);
        if ((e = cudaMemcpyAsync(static_cast<char*>(dst) + off, c->pin_buf[b], len, cudaMemcpyHostToDevice, s)) !=
                cudaSuccess ||
            (e = cudaEventRecord(c->pin_ev[b], s)) != cudaSuccess)
            return cuda_fail(e, "H2D copy");
    }
    return BSG_OK;
}

// Leaves `dst` complete when it returns (the stream is synchronised for
// pageable destinations; pinned ones are completed by the caller's sync).
int copy_d2h(bsg_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t s) {
    cudaError_t e;
    if (bytes < kDirectBelow || !is_pageable(dst)) {
        if ((e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return cuda_fail(e, "D2H copy");
        return BSG_OK;
    }
    if (int rc = ensure_stage(c)) return rc;
    const size_t chunks = (bytes + kStageChunk - 1) / kStageChunk;
    auto issue = [&](size_t i) -> cudaError_t {
        const int b = static_cast<int>(i & 1);
        const size_t off = i * kStageChunk, len = std::min(kStageChunk, bytes - off);
        cudaError_t r = cudaMemcpyAsync(c->pin_buf[b], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, s);
        return r == cudaSuccess ? cudaEventRecord(c->pin_ev[b], s) : r;
    };
    if ((e = issue(0)) != cudaSuccess) return cuda_fail(e, "D2H copy");
    for (size_t i = 0; i < chunks; ++i) {
        const int b = static_cast<int>(i & 1);
        if (i + 1 < chunks && (e = issue(i + 1)) != cudaSuccess) return cuda_fail(e, "D2H copy");
        if ((e = cudaEventSynchronize(c->pin_ev[b])) != cudaSuccess) return cuda_fail(e, "D2H staging");
        const size_t off = i * kStageChunk, len = std::min(kStageChunk, bytes - off);
        par_memcpy(static_cast<char*>(dst) + off, c->pin_buf[b], len);
    }
    return BSG_OK;
}

void release_stage(bsg_ctx* c) {
    for (int i = 0; i < 2; ++i) {
        if (c->pin_buf[i]) cudaFreeHost(c->pin_buf[i]);
        if (c->pin_ev[i]) cudaEventDestroy(c->pin_ev[i]);
        c->pin_buf[i] = nullptr;
        c->pin_ev[i] = nullptr;
    }
}

} // namespace bsg
