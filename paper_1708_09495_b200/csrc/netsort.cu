// netsort.cu -- batched BTN / OET block-network sorts and merge_split for
// sm_100a.
//
// Restates netsort.hpp:124-199 (prepare_blocks + run_block_network) for a
// batch of independent arrays: one CTA owns one (or, for short arrays,
// several) array(s) entirely in shared memory.  The p BSP workers become p
// blocks of L = ceil(len/p) keys inside the CTA; the reference's supersteps
// become __syncthreads() between ping-pong shared-memory buffers:
//   superstep 0  -- local sort of every block (netsort.hpp:167): 16-key
//                   register sorting networks (Batcher), then merge-path
//                   merges inside each block;
//   superstep s  -- merge_split of every (worker, partner) pair of stage s
//                   (netsort.hpp:170-179): each thread produces 16 consecutive
//                   outputs of the pair's merged sequence after a merge-path
//                   binary search; the keep_low worker takes outputs [0, L),
//                   its partner [L, 2L); idle OET edge workers copy.
// Padding with 0xFFFFFFFF and the final strip follow netsort.hpp:131-139, 197.
// Stage partners are computed on the fly from the closed forms of
// bitonic_schedule (netsort.hpp:76-88) and odd_even_rounds (netsort.hpp:99-105).
#include <algorithm>

#include "common.cuh"
#include "netsort.cuh"
#include "timer.cuh"

namespace bsg {

namespace {

constexpr int kNK = 16;         // outputs per thread-chunk
constexpr int kNetThreads = 256;
constexpr uint32_t kPad = 0xFFFFFFFFu;

__device__ __forceinline__ void cas(uint32_t& a, uint32_t& b) {
    const uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

// Batcher's odd-even merge sort network on 16 registers (63 comparators,
// generated and checked against all 2^16 zero-one inputs).
__device__ __forceinline__ void sort16(uint32_t (&v)[16]) {
    cas(v[0], v[1]);
    cas(v[2], v[3]);
    cas(v[4], v[5]);
    cas(v[6], v[7]);
    cas(v[8], v[9]);
    cas(v[10], v[11]);
    cas(v[12], v[13]);
    cas(v[14], v[15]);
    cas(v[0], v[2]);
    cas(v[1], v[3]);
    cas(v[4], v[6]);
    cas(v[5], v[7]);
    cas(v[8], v[10]);
    cas(v[9], v[11]);
    cas(v[12], v[14]);
    cas(v[13], v[15]);
    cas(v[1], v[2]);
    cas(v[5], v[6]);
    cas(v[9], v[10]);
    cas(v[13], v[14]);
    cas(v[0], v[4]);
    cas(v[1], v[5]);
    cas(v[2], v[6]);
    cas(v[3], v[7]);
    cas(v[8], v[12]);
    cas(v[9], v[13]);
    cas(v[10], v[14]);
    cas(v[11], v[15]);
    cas(v[2], v[4]);
    cas(v[3], v[5]);
    cas(v[10], v[12]);
    cas(v[11], v[13]);
    cas(v[1], v[2]);
    cas(v[3], v[4]);
    cas(v[5], v[6]);
    cas(v[9], v[10]);
    cas(v[11], v[12]);
    cas(v[13], v[14]);
    cas(v[0], v[8]);
    cas(v[1], v[9]);
    cas(v[2], v[10]);
    cas(v[3], v[11]);
    cas(v[4], v[12]);
    cas(v[5], v[13]);
    cas(v[6], v[14]);
    cas(v[7], v[15]);
    cas(v[4], v[8]);
    cas(v[5], v[9]);
    cas(v[6], v[10]);
    cas(v[7], v[11]);
    cas(v[2], v[4]);
    cas(v[3], v[5]);
    cas(v[6], v[8]);
    cas(v[7], v[9]);
    cas(v[10], v[12]);
    cas(v[11], v[13]);
    cas(v[1], v[2]);
    cas(v[3], v[4]);
    cas(v[5], v[6]);
    cas(v[7], v[8]);
    cas(v[9], v[10]);
    cas(v[11], v[12]);
    cas(v[13], v[14]);
}

// Shared-memory index with one pad word per 32: the stride-4/stride-8 access
// patterns of merge-path chunks (8 outputs per lane) become conflict-free.
__device__ __forceinline__ uint32_t pad(uint32_t i) { return i + (i >> 5); }

// Writes outputs [diag, diag+cnt) of merge(A, B) (ties taken from A first,
// netsort.hpp:39) into smem at logical indices dst0 .. dst0+cnt-1.  A and B
// are logical index ranges [a0, a0+na), [b0, b0+nb) of the padded buffer S.
__device__ __forceinline__ void merge_chunk_s(const uint32_t* S, uint32_t a0, int na, uint32_t b0, int nb, int diag,
                                              int cnt, uint32_t* D, uint32_t dst0) {
    int lo = max(0, diag - nb), hi = min(diag, na);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (S[pad(a0 + mid)] <= S[pad(b0 + diag - 1 - mid)]) lo = mid + 1;
        else hi = mid;
    }
    int i = lo, j = diag - lo;
    uint32_t av = i < na ? S[pad(a0 + i)] : 0u, bv = j < nb ? S[pad(b0 + j)] : 0u;
#pragma unroll
    for (int k = 0; k < kNK; ++k) {
        if (k < cnt) {
            const bool take_a = i < na && (j >= nb || av <= bv);
            D[pad(dst0 + k)] = take_a ? av : bv;
            i += take_a ? 1 : 0;
            j += take_a ? 0 : 1;
            const bool more = take_a ? i < na : j < nb;
            const uint32_t nxt = more ? S[pad(take_a ? a0 + i : b0 + j)] : 0u;
            av = take_a ? nxt : av;
            bv = take_a ? bv : nxt;
        }
    }
}

// Global-memory variant for the standalone merge_split.
__device__ __forceinline__ void merge_chunk(const uint32_t* A, int na, const uint32_t* B, int nb, int diag, int cnt,
                                            uint32_t* dst) {
    int lo = max(0, diag - nb), hi = min(diag, na);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (A[mid] <= B[diag - 1 - mid]) lo = mid + 1;
        else hi = mid;
    }
    int i = lo, j = diag - lo;
    uint32_t av = i < na ? A[i] : 0u, bv = j < nb ? B[j] : 0u;
#pragma unroll
    for (int k = 0; k < kNK; ++k) {
        if (k < cnt) {
            const bool take_a = i < na && (j >= nb || av <= bv);
            if (take_a) {
                dst[k] = av;
                ++i;
                av = i < na ? A[i] : 0u;
            } else {
                dst[k] = bv;
                ++j;
                bv = j < nb ? B[j] : 0u;
            }
        }
    }
}

// bitonic_schedule (netsort.hpp:76-88) for stage s, worker i.
__device__ __forceinline__ int btn_partner(int s, int i, bool& keep_low) {
    int a = 1, base = 0;
    while (base + a <= s) {
        base += a;
        ++a;
    }
    const int jidx = s - base;
    const int k = 1 << a, j = 1 << (a - 1 - jidx);
    const int q = i ^ j;
    const bool asc = (i & k) == 0;
    keep_low = asc ? (i < q) : (i > q);
    return q;
}

// odd_even_rounds (netsort.hpp:99-105) for round r, worker i; -1 = idle.
__device__ __forceinline__ int oet_partner(int r, int i, int p, bool& keep_low) {
    const int par = r & 1;
    if (i < par) return -1;
    if (((i - par) & 1) == 0) {
        if (i + 1 < p) {
            keep_low = true;
            return i + 1;
        }
        return -1;
    }
    keep_low = false;
    return i - 1;
}

__global__ void __launch_bounds__(kNetThreads)
    block_network_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t num_arrays,
                         uint32_t len, int p, uint32_t L, int network, int run_stages, int full, int apc) {
    extern __shared__ __align__(16) uint32_t net_smem[];
    const uint32_t P = L * static_cast<uint32_t>(p);
    const uint32_t padded = pad(static_cast<uint32_t>(apc) * P) + 1;
    uint32_t* bufA = net_smem;
    uint32_t* bufB = net_smem + padded;
    const uint64_t array0 = static_cast<uint64_t>(blockIdx.x) * apc;
    const int na = static_cast<int>(min(static_cast<uint64_t>(apc), num_arrays - array0));
    const int tid = threadIdx.x;

    // prepare_blocks: load + pad (netsort.hpp:131-139)
    const uint32_t tot = static_cast<uint32_t>(na) * P;
    for (uint32_t idx = tid; idx < tot; idx += kNetThreads) {
        const uint32_t a = idx / P, e = idx - a * P;
        bufA[pad(idx)] = e < len ? __ldg(in + (array0 + a) * len + e) : kPad;
    }
    __syncthreads();

    const uint32_t cb = (L + kNK - 1) / kNK; // chunks per block
    const uint32_t items = static_cast<uint32_t>(na) * static_cast<uint32_t>(p) * cb;

    // superstep 0: local sort of every block.  (a) 16-key register sorting networks
    for (uint32_t it = tid; it < items; it += kNetThreads) {
        const uint32_t a = it / (p * cb), rem = it - a * p * cb;
        const uint32_t w = rem / cb, c = rem - w * cb;
        const uint32_t b0 = a * P + w * L;
        const uint32_t ob = c * kNK;
        const int cnt = static_cast<int>(min(static_cast<uint32_t>(kNK), L - ob));
        uint32_t v[kNK];
#pragma unroll
        for (int k = 0; k < kNK; ++k) v[k] = k < cnt ? bufA[pad(b0 + ob + k)] : kPad;
        sort16(v);
#pragma unroll
        for (int k = 0; k < kNK; ++k)
            if (k < cnt) bufA[pad(b0 + ob + k)] = v[k];
    }
    __syncthreads();
    // (b) bottom-up merge-path merges inside each block
    uint32_t* src = bufA;
    uint32_t* dst = bufB;
    for (uint32_t width = kNK; width < L; width *= 2) {
        for (uint32_t it = tid; it < items; it += kNetThreads) {
            const uint32_t a = it / (p * cb), rem = it - a * p * cb;
            const uint32_t w = rem / cb, c = rem - w * cb;
            const uint32_t bs = a * P + w * L;
            const uint32_t ob = c * kNK;
            const int cnt = static_cast<int>(min(static_cast<uint32_t>(kNK), L - ob));
            const uint32_t ps = (ob / (2 * width)) * (2 * width);
            const uint32_t a_end = min(ps + width, L), b_end = min(ps + 2 * width, L);
            merge_chunk_s(src, bs + ps, static_cast<int>(a_end - ps), bs + a_end, static_cast<int>(b_end - a_end),
                          static_cast<int>(ob - ps), cnt, dst, bs + ob);
        }
        __syncthreads();
        uint32_t* t = src;
        src = dst;
        dst = t;
    }

    // supersteps 1..S: merge_split stages
    for (int s = 0; s < run_stages; ++s) {
        for (uint32_t it = tid; it < items; it += kNetThreads) {
            const uint32_t a = it / (p * cb), rem = it - a * p * cb;
            const int i = static_cast<int>(rem / cb);
            const uint32_t c = rem - static_cast<uint32_t>(i) * cb;
            const uint32_t ob = c * kNK;
            const int cnt = static_cast<int>(min(static_cast<uint32_t>(kNK), L - ob));
            bool keep_low = false;
            const int q = network == 0 ? btn_partner(s, i, keep_low) : oet_partner(s, i, p, keep_low);
            const uint32_t my0 = a * P + static_cast<uint32_t>(i) * L;
            if (q < 0) {
#pragma unroll
                for (int k = 0; k < kNK; ++k)
                    if (k < cnt) dst[pad(my0 + ob + k)] = src[pad(my0 + ob + k)];
                continue;
            }
            const int lo_w = min(i, q), hi_w = max(i, q);
            const int diag = static_cast<int>((keep_low ? 0u : L) + ob);
            merge_chunk_s(src, a * P + static_cast<uint32_t>(lo_w) * L, static_cast<int>(L),
                          a * P + static_cast<uint32_t>(hi_w) * L, static_cast<int>(L), diag, cnt, dst, my0 + ob);
        }
        __syncthreads();
        uint32_t* t = src;
        src = dst;
        dst = t;
    }

    // concatenate (+ strip the pad when the network ran to completion)
    if (full) {
        for (uint32_t idx = tid; idx < static_cast<uint32_t>(na) * len; idx += kNetThreads) {
            const uint32_t a = idx / len, e = idx - a * len;
            out[(array0 + a) * len + e] = src[pad(a * P + e)];
        }
    } else {
        for (uint32_t idx = tid; idx < tot; idx += kNetThreads) out[array0 * P + idx] = src[pad(idx)];
    }
}

constexpr int kMsThreads = 256;

__global__ void __launch_bounds__(kMsThreads)
    merge_split_kernel(const uint32_t* __restrict__ a, uint32_t na, const uint32_t* __restrict__ b, uint32_t nb,
                       uint32_t* __restrict__ low, uint32_t* __restrict__ high) {
    const uint32_t total = na + nb;
    const uint32_t chunks = (total + kNK - 1) / kNK;
    for (uint32_t c = blockIdx.x * kMsThreads + threadIdx.x; c < chunks; c += gridDim.x * kMsThreads) {
        const uint32_t o = c * kNK;
        const int cnt = static_cast<int>(min(static_cast<uint32_t>(kNK), total - o));
        uint32_t v[kNK];
        merge_chunk(a, static_cast<int>(na), b, static_cast<int>(nb), static_cast<int>(o), cnt, v);
#pragma unroll
        for (int k = 0; k < kNK; ++k) {
            if (k < cnt) {
                const uint32_t pos = o + k;
                if (pos < na) low[pos] = v[k];
                else high[pos - na] = v[k];
            }
        }
    }
}


// One merge-split stage of a large (global-memory) block network: every
// output chunk of 16 keys of worker i's new block is produced by a merge-path
// search over (block min(i,q), block max(i,q)) of the previous state.
__global__ void __launch_bounds__(kMsThreads)
    net_stage_kernel(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, int p, uint32_t L, int network,
                     int s) {
    const uint64_t cb = (L + kNK - 1) / kNK;
    const uint64_t items = cb * static_cast<uint64_t>(p);
    for (uint64_t it = static_cast<uint64_t>(blockIdx.x) * kMsThreads + threadIdx.x; it < items;
         it += static_cast<uint64_t>(gridDim.x) * kMsThreads) {
        const int i = static_cast<int>(it / cb);
        const uint32_t ob = static_cast<uint32_t>(it - static_cast<uint64_t>(i) * cb) * kNK;
        const int cnt = static_cast<int>(min(static_cast<uint32_t>(kNK), L - ob));
        bool keep_low = false;
        const int q = network == 0 ? btn_partner(s, i, keep_low) : oet_partner(s, i, p, keep_low);
        uint32_t* out = dst + static_cast<uint64_t>(i) * L + ob;
        if (q < 0) {
            const uint32_t* in = src + static_cast<uint64_t>(i) * L + ob;
            for (int k = 0; k < cnt; ++k) out[k] = in[k];
            continue;
        }
        const int lo_w = min(i, q), hi_w = max(i, q);
        uint32_t v[kNK];
        merge_chunk(src + static_cast<uint64_t>(lo_w) * L, static_cast<int>(L), src + static_cast<uint64_t>(hi_w) * L,
                    static_cast<int>(L), static_cast<int>((keep_low ? 0u : L) + ob), cnt, v);
#pragma unroll
        for (int k = 0; k < kNK; ++k)
            if (k < cnt) out[k] = v[k];
    }
}

} // namespace

int launch_net_stage(const uint32_t* src, uint32_t* dst, int p, uint32_t L, int network, int s, cudaStream_t stream) {
    const uint64_t items = ((L + kNK - 1) / kNK) * static_cast<uint64_t>(p);
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((items + kMsThreads - 1) / kMsThreads, 148 * 16)));
    TimedScope ts(2 /*BSG_K_NETWORK*/, stream);
    net_stage_kernel<<<grid, kMsThreads, 0, stream>>>(src, dst, p, L, network, s);
    return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

int launch_block_network(int network, const uint32_t* in, uint32_t* out, uint64_t num_arrays, uint32_t len, int p,
                         int run_stages, bool full, cudaStream_t stream) {
    const uint32_t L = (len + static_cast<uint32_t>(p) - 1) / static_cast<uint32_t>(p);
    const uint32_t P = L * static_cast<uint32_t>(p);
    if (P == 0 || P > kNetMaxPadded) return -1;
    const int apc = static_cast<int>(std::max<uint32_t>(1, 4096 / P));
    const size_t padded = static_cast<size_t>(apc) * P + (static_cast<size_t>(apc) * P >> 5) + 1;
    const size_t smem = 2ull * padded * sizeof(uint32_t);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(block_network_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(2 * (kNetMaxPadded + kNetMaxPadded / 32 + 1) * sizeof(uint32_t)));
        attr = true;
    }
    const uint64_t grid = (num_arrays + apc - 1) / apc;
    if (grid > 0x7FFFFFFFull) return -1;
    TimedScope ts(2 /*BSG_K_NETWORK*/, stream);
    block_network_kernel<<<static_cast<unsigned>(grid), kNetThreads, smem, stream>>>(in, out, num_arrays, len, p, L,
                                                                                   network, run_stages, full ? 1 : 0, apc);
    return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

int launch_merge_split(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb, uint32_t* low, uint32_t* high,
                       cudaStream_t stream) {
    const uint64_t total = na + nb;
    if (total == 0) return 0;
    const uint64_t chunks = (total + kNK - 1) / kNK;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((chunks + kMsThreads - 1) / kMsThreads, 148 * 16));
    merge_split_kernel<<<grid, kMsThreads, 0, stream>>>(a, static_cast<uint32_t>(na), b, static_cast<uint32_t>(nb), low,
                                                       high);
    return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

} // namespace bsg
