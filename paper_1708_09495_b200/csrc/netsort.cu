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

constexpr int kNK = 16;         // keys per thread-chunk: register sort, global merges
#ifndef BSG_NET_MK
#define BSG_NET_MK 16
#endif
constexpr int kMK = BSG_NET_MK;
#ifndef BSG_NET_MINB
#define BSG_NET_MINB 5
#endif
#ifndef BSG_NET_REG
#define BSG_NET_REG 1 // register/shuffle network for power-of-two block lengths >= 16
#endif
#ifndef BSG_NET_FMA_SORT16
#define BSG_NET_FMA_SORT16 1 // register network: sort16 maxima on the FMA pipe
#endif
#ifndef BSG_NET_SORT32
#define BSG_NET_SORT32 1
#endif // outputs per thread-chunk of the shared-memory merges
constexpr uint32_t kPad = 0xFFFFFFFFu;

// x / d without a division instruction sequence: m = ceil(2^32 / d) is exact
// for x * d < 2^32 (indices and divisors here are < 2^16).
struct FastDiv {
    uint32_t d, m;
    FastDiv() = default;
    __host__ __device__ __forceinline__ explicit FastDiv(uint32_t dv) : d(dv), m(dv > 1 ? 0xFFFFFFFFu / dv + 1u : 0u) {}
    __device__ __forceinline__ uint32_t div(uint32_t x) const { return d > 1 ? __umulhi(x, m) : x; }
};

__device__ __forceinline__ void cas(uint32_t& a, uint32_t& b) {
    const uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

// Batcher's odd-even merge sort network on 16 registers (63 comparators,
// generated and checked against all 2^16 zero-one inputs).
__device__ constexpr uint8_t kSort16[63][2] = {{0, 1}, {2, 3}, {4, 5}, {6, 7}, {8, 9}, {10, 11}, {12, 13}, {14, 15}, {0, 2}, {1, 3}, {4, 6}, {5, 7}, {8, 10}, {9, 11}, {12, 14}, {13, 15}, {1, 2}, {5, 6}, {9, 10}, {13, 14}, {0, 4}, {1, 5}, {2, 6}, {3, 7}, {8, 12}, {9, 13}, {10, 14}, {11, 15}, {2, 4}, {3, 5}, {10, 12}, {11, 13}, {1, 2}, {3, 4}, {5, 6}, {9, 10}, {11, 12}, {13, 14}, {0, 8}, {1, 9}, {2, 10}, {3, 11}, {4, 12}, {5, 13}, {6, 14}, {7, 15}, {4, 8}, {5, 9}, {6, 10}, {7, 11}, {2, 4}, {3, 5}, {6, 8}, {7, 9}, {10, 12}, {11, 13}, {1, 2}, {3, 4}, {5, 6}, {7, 8}, {9, 10}, {11, 12}, {13, 14}};
template <typename Cas>
__device__ __forceinline__ void sort16(uint32_t (&v)[16], const Cas& c) {
#pragma unroll
    for (int k = 0; k < 63; ++k) c(v[kSort16[k][0]], v[kSort16[k][1]]);
}
struct CasAlu {
    __device__ __forceinline__ void operator()(uint32_t& a, uint32_t& b) const { cas(a, b); }
};
__device__ __forceinline__ void sort16(uint32_t (&v)[16]) { sort16(v, CasAlu{}); }

// Compare-exchange with the maximum on the FMA pipe: hi = a + b - min(a, b)
// (exact mod 2^32) as two IMADs.  `one` = 1 and `neg1` = -1 are runtime values
// so that ptxas keeps the IMADs instead of folding them into an IADD3 on the
// integer ALU pipe, which min/max already saturate.
struct CasFma {
    uint32_t one;
    uint32_t neg1;
    __device__ __forceinline__ void operator()(uint32_t& a, uint32_t& b) const {
        const uint32_t lo = min(a, b);
        uint32_t s, hi;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(s) : "r"(a), "r"(one), "r"(b));
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(hi) : "r"(lo), "r"(neg1), "r"(s));
        a = lo;
        b = hi;
    }
};

// Shared-memory index with one pad word per 32: the stride-4/stride-8 access
// patterns of merge-path chunks (8 outputs per lane) become conflict-free.
__device__ __forceinline__ uint32_t pad(uint32_t i) { return i + (i >> 5); }

// Writes outputs [diag, diag+cnt) of merge(A, B) (netsort.hpp:30-51) into
// smem at logical indices dst0 .. dst0+cnt-1.  A and B are logical index
// ranges [a0, a0+na), [b0, b0+nb) of the padded buffer S.
//
// After the merge-path split (i, j) of `diag`, the next kNK outputs are the
// kNK smallest of A[i, i+kNK) u B[j, j+kNK) (MAX past the ends): with x
// ascending and y ascending, min(x[k], y[kNK-1-k]) is that set as a bitonic
// sequence, sorted by a 4-stage bitonic network.  Only key values are
// produced, so which of two equal keys is taken (or a MAX pad instead of a
// real 0xFFFFFFFF key) cannot change the output.
template <int K>
__device__ __forceinline__ void merge_chunk_s(const uint32_t* S, uint32_t a0, int na, uint32_t b0, int nb, int diag,
                                              int cnt, uint32_t* D, uint32_t dst0) {
    int lo = max(0, diag - nb), hi = min(diag, na);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (S[pad(a0 + mid)] <= S[pad(b0 + diag - 1 - mid)]) lo = mid + 1;
        else hi = mid;
    }
    const int i = lo, j = diag - lo;
    const int ra = na - i, rb = nb - j;
    const uint32_t pa = a0 + i, pb = b0 + j;
    uint32_t x[K], y[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        x[k] = k < ra ? S[pad(pa + k)] : kPad;
        y[k] = k < rb ? S[pad(pb + k)] : kPad;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) x[k] = min(x[k], y[K - 1 - k]);
#pragma unroll
    for (int d = K / 2; d >= 1; d >>= 1)
#pragma unroll
        for (int k = 0; k < K; ++k)
            if ((k & d) == 0) cas(x[k], x[k + d]);
#pragma unroll
    for (int k = 0; k < K; ++k)
        if (k < cnt) D[pad(dst0 + k)] = x[k];
}

// Global-memory variant (standalone merge_split, large-array stages): same
// merge-path split + bitonic selection of the next kNK outputs.
__device__ __forceinline__ void merge_chunk(const uint32_t* A, int na, const uint32_t* B, int nb, int diag, int cnt,
                                            uint32_t* dst) {
    (void)cnt;
    int lo = max(0, diag - nb), hi = min(diag, na);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(A + mid) <= __ldg(B + diag - 1 - mid)) lo = mid + 1;
        else hi = mid;
    }
    const int i = lo, j = diag - lo;
    const int ra = na - i, rb = nb - j;
    uint32_t y[kNK];
#pragma unroll
    for (int k = 0; k < kNK; ++k) {
        dst[k] = k < ra ? __ldg(A + i + k) : kPad;
        y[k] = k < rb ? __ldg(B + j + k) : kPad;
    }
#pragma unroll
    for (int k = 0; k < kNK; ++k) dst[k] = min(dst[k], y[kNK - 1 - k]);
#pragma unroll
    for (int d = kNK / 2; d >= 1; d >>= 1)
#pragma unroll
        for (int k = 0; k < kNK; ++k)
            if ((k & d) == 0) cas(dst[k], dst[k + d]);
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

// THREADS x MINB: 256 x 5 for padded arrays <= 8192 keys (several CTAs per
// SM), 1024 x 1 above, where the two shared-memory copies allow one CTA per
// SM (keeps 32 warps resident instead of 8).
// Launch-uniform divisors with their multipliers precomputed on the host.
struct NetDivs {
    FastDiv P, pcb, cb, pcbm, cbm, len;
};

template <int kNetThreads, int MINB>
__global__ void __launch_bounds__(kNetThreads, MINB)
    block_network_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t num_arrays,
                         uint32_t len, int p, uint32_t L, int network, int run_stages, int full, int apc,
                         const NetDivs dv) {
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
    const FastDiv& divP = dv.P;
    for (uint32_t idx = tid; idx < tot; idx += kNetThreads) {
        const uint32_t a = divP.div(idx), e = idx - a * P;
        bufA[pad(idx)] = e < len ? __ldg(in + (array0 + a) * len + e) : kPad;
    }
    __syncthreads();

#if BSG_NET_SORT32
    // superstep 0: local sort of every block.  (a) 32-key register sorts
    // (two Batcher 16-networks + a bitonic merge), one chunk per thread
    constexpr int kSK = 2 * kNK;
    const uint32_t cb = (L + kSK - 1) / kSK; // sort chunks per block
    const uint32_t items = static_cast<uint32_t>(na) * static_cast<uint32_t>(p) * cb;
    const FastDiv &div_pcb = dv.pcb, &div_cb = dv.cb;
    for (uint32_t it = tid; it < items; it += kNetThreads) {
        const uint32_t a = div_pcb.div(it), rem = it - a * p * cb;
        const uint32_t w = div_cb.div(rem), c = rem - w * cb;
        const uint32_t b0 = a * P + w * L;
        const uint32_t ob = c * kSK;
        const int cnt = static_cast<int>(min(static_cast<uint32_t>(kSK), L - ob));
        uint32_t v[kNK], u[kNK];
#pragma unroll
        for (int k = 0; k < kNK; ++k) {
            v[k] = k < cnt ? bufA[pad(b0 + ob + k)] : kPad;
            u[k] = k + kNK < cnt ? bufA[pad(b0 + ob + kNK + k)] : kPad;
        }
        sort16(v);
        sort16(u);
        // half-cleaner of v ++ reverse(u): v = 16 smallest, u = 16 largest (bitonic each)
#pragma unroll
        for (int k = 0; k < kNK; ++k) cas(v[k], u[kNK - 1 - k]);
#pragma unroll
        for (int d = kNK / 2; d >= 1; d >>= 1)
#pragma unroll
            for (int k = 0; k < kNK; ++k)
                if ((k & d) == 0) {
                    cas(v[k], v[k + d]);
                    cas(u[k], u[k + d]);
                }
#pragma unroll
        for (int k = 0; k < kNK; ++k) {
            if (k < cnt) bufA[pad(b0 + ob + k)] = v[k];
            if (k + kNK < cnt) bufA[pad(b0 + ob + kNK + k)] = u[k];
        }
    }
    __syncthreads();
#else
    // superstep 0: local sort of every block.  (a) 16-key register sorting networks
    constexpr int kSK = kNK;
    const uint32_t cb = (L + kSK - 1) / kSK; // sort chunks per block
    const uint32_t items = static_cast<uint32_t>(na) * static_cast<uint32_t>(p) * cb;
    const FastDiv &div_pcb = dv.pcb, &div_cb = dv.cb;
    for (uint32_t it = tid; it < items; it += kNetThreads) {
        const uint32_t a = div_pcb.div(it), rem = it - a * p * cb;
        const uint32_t w = div_cb.div(rem), c = rem - w * cb;
        const uint32_t b0 = a * P + w * L;
        const uint32_t ob = c * kSK;
        const int cnt = static_cast<int>(min(static_cast<uint32_t>(kSK), L - ob));
        uint32_t v[kNK];
#pragma unroll
        for (int k = 0; k < kNK; ++k) v[k] = k < cnt ? bufA[pad(b0 + ob + k)] : kPad;
        sort16(v);
#pragma unroll
        for (int k = 0; k < kNK; ++k)
            if (k < cnt) bufA[pad(b0 + ob + k)] = v[k];
    }
    __syncthreads();
#endif
    // (b) bottom-up merge-path merges inside each block
    uint32_t* src = bufA;
    uint32_t* dst = bufB;
    const uint32_t cbm = (L + kMK - 1) / kMK; // merge chunks per block
    const uint32_t mitems = static_cast<uint32_t>(na) * static_cast<uint32_t>(p) * cbm;
    const FastDiv &div_pcbm = dv.pcbm, &div_cbm = dv.cbm;
    for (uint32_t width = kSK; width < L; width *= 2) {
        for (uint32_t it = tid; it < mitems; it += kNetThreads) {
            const uint32_t a = div_pcbm.div(it), rem = it - a * p * cbm;
            const uint32_t w = div_cbm.div(rem), c = rem - w * cbm;
            const uint32_t bs = a * P + w * L;
            const uint32_t ob = c * kMK;
            const int cnt = static_cast<int>(min(static_cast<uint32_t>(kMK), L - ob));
            const uint32_t ps = ob & ~(2 * width - 1); // width is a power of two
            const uint32_t a_end = min(ps + width, L), b_end = min(ps + 2 * width, L);
            merge_chunk_s<kMK>(src, bs + ps, static_cast<int>(a_end - ps), bs + a_end, static_cast<int>(b_end - a_end),
                          static_cast<int>(ob - ps), cnt, dst, bs + ob);
        }
        __syncthreads();
        uint32_t* t = src;
        src = dst;
        dst = t;
    }

    // supersteps 1..S: merge_split stages
    for (int s = 0; s < run_stages; ++s) {
        for (uint32_t it = tid; it < mitems; it += kNetThreads) {
            const uint32_t a = div_pcbm.div(it), rem = it - a * p * cbm;
            const int i = static_cast<int>(div_cbm.div(rem));
            const uint32_t c = rem - static_cast<uint32_t>(i) * cbm;
            const uint32_t ob = c * kMK;
            const int cnt = static_cast<int>(min(static_cast<uint32_t>(kMK), L - ob));
            bool keep_low = false;
            const int q = network == 0 ? btn_partner(s, i, keep_low) : oet_partner(s, i, p, keep_low);
            const uint32_t my0 = a * P + static_cast<uint32_t>(i) * L;
            if (q < 0) {
#pragma unroll
                for (int k = 0; k < kMK; ++k)
                    if (k < cnt) dst[pad(my0 + ob + k)] = src[pad(my0 + ob + k)];
                continue;
            }
            const int lo_w = min(i, q), hi_w = max(i, q);
            const int diag = static_cast<int>((keep_low ? 0u : L) + ob);
            merge_chunk_s<kMK>(src, a * P + static_cast<uint32_t>(lo_w) * L, static_cast<int>(L),
                          a * P + static_cast<uint32_t>(hi_w) * L, static_cast<int>(L), diag, cnt, dst, my0 + ob);
        }
        __syncthreads();
        uint32_t* t = src;
        src = dst;
        dst = t;
    }

    // concatenate (+ strip the pad when the network ran to completion)
    if (full) {
        const FastDiv& div_len = dv.len;
        for (uint32_t idx = tid; idx < static_cast<uint32_t>(na) * len; idx += kNetThreads) {
            const uint32_t a = div_len.div(idx), e = idx - a * len;
            out[(array0 + a) * len + e] = src[pad(a * P + e)];
        }
    } else {
        for (uint32_t idx = tid; idx < tot; idx += kNetThreads) out[array0 * P + idx] = src[pad(idx)];
    }
}

// ---------------------------------------------------------------------------
// Register block network (block length L a power of two, 16 <= L, p*L <=
// kNetMaxPadded).  Every thread holds R (16 or 32) consecutive keys of the
// CTA's key space in registers for the whole run.
//
// All networks are written in the "ascending only" bitonic form: phase k of
// the local sort first compares key e with its mirror e ^ (k-1) inside the
// k-group, then e with e ^ j for j = k/4 .. 1; the lower index always keeps
// the minimum.  A merge_split stage (netsort.hpp:30-51) is the same mirror
// step between worker i's block and its partner's block (the keep_low worker
// keeps min(own[k], partner[L-1-k]), the other the max: the L smallest resp.
// largest keys of the pair, as a bitonic sequence) followed by the bitonic
// merge j = L/2 .. 1.  Only key values move, so which of two equal keys is
// taken cannot change a block state.  An idle OET edge worker runs the merge
// steps on its sorted block, which leaves it unchanged.
//
// Two register layouts of a warp's 32R keys (e = warp-local key index):
//   A: lane l holds e = R*l + r: the low log2(R) key bits in registers;
//   B: lane l holds e = 32*r + l: key bits 5 .. 4+log2(R) in registers.
// A step on a register bit is one compare-exchange per pair inside the
// thread; a step on a lane bit costs a shuffle and a select per key (min/max
// run on the integer ALU pipe, the bound here).  Merges over key bits >= 5
// inside the warp therefore run in layout B, reached by a warp-local
// transpose through shared memory (the exchange buffer the next CTA exchange
// will use: its previous readers are past the last barrier); with R = 16, key
// bit 4 stays a shuffle in A.  Partner distances beyond the warp go through a
// CTA exchange (double-buffered, one barrier each).
//
// Shared memory holds CTA key E at word E + 4*(E >> 5): 128-bit accesses of A
// chunks and 32-bit accesses of B rows are both bank-conflict-free, and every
// address is a per-thread base plus a compile-time offset.
// ---------------------------------------------------------------------------
#ifndef BSG_NET_R
#define BSG_NET_R 16 // keys per thread of the register network (16 or 32; 32 measured slower)
#endif
#ifndef BSG_NET_BMIN16
#define BSG_NET_BMIN16 7 // R = 16: merges from key bit >= this run their bits >= 5 in layout B
#endif
#ifndef BSG_NET_BMIN32
#define BSG_NET_BMIN32 5 // R = 32: same
#endif
#ifndef BSG_NET_FMA_STEPS
#define BSG_NET_FMA_STEPS 0xF // register steps (masks) whose maxima go to the FMA pipe
#endif
#ifndef BSG_NET_CTA_KEYS
#define BSG_NET_CTA_KEYS 4096 // keys per CTA of the register network (arrays shorter than this share a CTA)
#endif
#ifndef BSG_NET_REG_TPSM
#define BSG_NET_REG_TPSM 1024 // threads per SM the register network is compiled for (64 registers)
#endif

__device__ __forceinline__ uint32_t minmax_sel(uint32_t a, uint32_t b, bool up) { return up ? max(a, b) : min(a, b); }

template <int R>
struct RegShape {
    static constexpr int LR = R == 32 ? 5 : 4; // log2 R
    static constexpr int BMIN = R == 32 ? BSG_NET_BMIN32 : BSG_NET_BMIN16;
    // word of thread u's key 0
    static __device__ __forceinline__ uint32_t a_word(uint32_t u) { return R == 32 ? 36u * u : 16u * u + 4u * (u >> 1); }
};

template <int R>
__device__ __forceinline__ void put_a(uint32_t* S, uint32_t u, const uint32_t (&v)[R]) {
    uint4* p = reinterpret_cast<uint4*>(S + RegShape<R>::a_word(u));
#pragma unroll
    for (int c = 0; c < R / 4; ++c) p[c] = make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
}
template <int R>
__device__ __forceinline__ void get_a(const uint32_t* S, uint32_t u, uint32_t (&v)[R]) {
    const uint4* p = reinterpret_cast<const uint4*>(S + RegShape<R>::a_word(u));
#pragma unroll
    for (int c = 0; c < R / 4; ++c) {
        const uint4 q = p[c];
        v[4 * c] = q.x;
        v[4 * c + 1] = q.y;
        v[4 * c + 2] = q.z;
        v[4 * c + 3] = q.w;
    }
}
// v[r] = OP(v[r], thread u's key r) (or key R-1-r if REV)
template <int R, bool REV, typename Op>
__device__ __forceinline__ void apply_a(const uint32_t* S, uint32_t u, uint32_t (&v)[R], Op op) {
    const uint4* p = reinterpret_cast<const uint4*>(S + RegShape<R>::a_word(u));
#pragma unroll
    for (int c = 0; c < R / 4; ++c) {
        const uint4 q = p[REV ? R / 4 - 1 - c : c];
        v[4 * c] = op(v[4 * c], REV ? q.w : q.x);
        v[4 * c + 1] = op(v[4 * c + 1], REV ? q.z : q.y);
        v[4 * c + 2] = op(v[4 * c + 2], REV ? q.y : q.z);
        v[4 * c + 3] = op(v[4 * c + 3], REV ? q.x : q.w);
    }
}

// bitonic steps on register masks J, J/2, .., 1 (ascending); the masks in
// BSG_NET_FMA_STEPS take their maxima on the FMA pipe
template <int J, int R>
__device__ __forceinline__ void reg_steps(uint32_t (&v)[R], const CasFma& f) {
#pragma unroll
    for (int j = J; j >= 1; j >>= 1)
#pragma unroll
        for (int r = 0; r < R; ++r)
            if ((r & j) == 0) {
                if (BSG_NET_FMA_STEPS & j) f(v[r], v[r + j]);
                else cas(v[r], v[r + j]);
            }
}

struct OpMin {
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return min(a, b); }
};
struct OpMax {
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return max(a, b); }
};
struct OpSel {
    bool up;
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return minmax_sel(a, b, up); }
};

template <int R>
struct RegNet {
    using Sh = RegShape<R>;
    uint32_t* S;     // two exchange buffers of `stride` words
    uint32_t stride; // (R + R/8) * blockDim.x words per buffer
    uint32_t b = 0;  // word offset of the buffer the next exchange uses
    uint32_t t, lane, warp;
    CasFma fc;

    // v[r] = OP(v[r], thread tp's key r (REV: R-1-r)), the lower thread of
    // a pair keeping the min
    template <bool REV>
    __device__ __forceinline__ void exchange_step(uint32_t (&v)[R], uint32_t tp, bool up) {
        uint32_t* buf = S + b;
        put_a<R>(buf, t, v);
        __syncthreads();
        if (up) apply_a<R, REV>(buf, tp, v, OpMax{});
        else apply_a<R, REV>(buf, tp, v, OpMin{});
        b ^= stride;
    }
    // warp-local transposes A -> B and B -> A
    __device__ __forceinline__ void to_B(uint32_t (&v)[R]) {
        uint32_t* buf = S + b;
        put_a<R>(buf, t, v);
        __syncwarp();
        const uint32_t* row = buf + 36u * R * warp + lane;
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = row[36 * r];
        __syncwarp();
    }
    __device__ __forceinline__ void to_A(uint32_t (&v)[R]) {
        uint32_t* buf = S + b;
        uint32_t* row = buf + 36u * R * warp + lane;
#pragma unroll
        for (int r = 0; r < R; ++r) row[36 * r] = v[r];
        __syncwarp();
        get_a<R>(buf, t, v);
        __syncwarp();
    }
    // compare with thread t ^ TM, same register
    template <uint32_t TM>
    __device__ __forceinline__ void cross_step(uint32_t (&v)[R]) {
        const bool up = (t & TM) != 0;
        if constexpr (TM < 32) {
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = minmax_sel(v[r], __shfl_xor_sync(0xffffffffu, v[r], TM), up);
        } else {
            exchange_step<false>(v, t ^ TM, up);
        }
    }
    // mirror step of a group of 2*HALF threads: thread t pairs with
    // t ^ (2*HALF-1), register r with R-1-r
    template <uint32_t HALF>
    __device__ __forceinline__ void mirror_step(uint32_t (&v)[R]) {
        constexpr uint32_t TM = 2 * HALF - 1;
        const bool up = (t & HALF) != 0;
        if constexpr (TM < 32) {
#pragma unroll
            for (int r = 0; r < R / 2; ++r) {
                const uint32_t xa = __shfl_xor_sync(0xffffffffu, v[R - 1 - r], TM);
                const uint32_t xb = __shfl_xor_sync(0xffffffffu, v[r], TM);
                v[r] = minmax_sel(v[r], xa, up);
                v[R - 1 - r] = minmax_sel(v[R - 1 - r], xb, up);
            }
        } else {
            exchange_step<true>(v, t ^ TM, up);
        }
    }
    // bitonic merge steps on key bits TOP, TOP-1, .., 0
    template <int TOP>
    __device__ __forceinline__ void merge_bits(uint32_t (&v)[R]) {
        if constexpr (TOP < 0) {
        } else if constexpr (TOP >= Sh::LR + 5) { // another warp
            cross_step<(1u << (TOP - Sh::LR))>(v);
            merge_bits<TOP - 1>(v);
        } else if constexpr (TOP >= 5 && TOP >= Sh::BMIN) { // bits TOP..5 in layout B
            to_B(v);
            reg_steps<(1 << (TOP - 5))>(v, fc);
            to_A(v);
            merge_bits<4>(v);
        } else if constexpr (TOP >= Sh::LR) { // another lane
            cross_step<(1u << (TOP - Sh::LR))>(v);
            merge_bits<TOP - 1>(v);
        } else {
            reg_steps<(1 << TOP)>(v, fc);
        }
    }
    // in-thread sort of the R keys
    __device__ __forceinline__ void sort_r(uint32_t (&v)[R]) {
        if constexpr (R == 16) {
            if (BSG_NET_FMA_SORT16) sort16(v, fc);
            else sort16(v);
        } else {
            uint32_t(&lo)[16] = *reinterpret_cast<uint32_t(*)[16]>(&v[0]);
            uint32_t(&hi)[16] = *reinterpret_cast<uint32_t(*)[16]>(&v[16]);
            if (BSG_NET_FMA_SORT16) {
                sort16(lo, fc);
                sort16(hi, fc);
            } else {
                sort16(lo);
                sort16(hi);
            }
#pragma unroll
            for (int r = 0; r < 16; ++r) fc(v[r], v[31 - r]);
            reg_steps<8>(v, fc);
        }
    }
    // local-sort phases k = 2^M .. 2^LOGL (the first LR phases are sort_r)
    template <int M, int LOGL>
    __device__ __forceinline__ void sort_phases(uint32_t (&v)[R]) {
        if constexpr (M <= LOGL) {
            mirror_step<(1u << (M - 1 - Sh::LR))>(v);
            merge_bits<M - 2>(v);
            sort_phases<M + 1, LOGL>(v);
        }
    }
};

template <int R, int kThreads, int MINB, int LOGL>
__global__ void __launch_bounds__(kThreads, MINB)
    block_network_reg_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t num_arrays,
                             uint32_t len, int p, int network, int run_stages, int full, int apc, int vec_in,
                             int vec_out, uint32_t one, uint32_t neg1) {
    extern __shared__ __align__(16) uint32_t reg_smem[];
    using Sh = RegShape<R>;
    constexpr uint32_t L = 1u << LOGL;
    constexpr uint32_t spt = L / R; // threads per block (worker)
    static_assert(spt >= 1, "block shorter than a thread's keys");
    RegNet<R> net;
    net.t = threadIdx.x;
    net.lane = threadIdx.x & 31;
    net.warp = threadIdx.x >> 5;
    net.fc = CasFma{one, neg1};
    net.S = reg_smem;
    net.stride = blockDim.x * (R + R / 8);
    const uint32_t t = threadIdx.x;
    const uint32_t P = L * static_cast<uint32_t>(p);
    const uint64_t array0 = static_cast<uint64_t>(blockIdx.x) * apc;
    const uint32_t na = static_cast<uint32_t>(min(static_cast<uint64_t>(apc), num_arrays - array0));
    const uint32_t seg = t / spt; // worker block of this thread in the CTA
    const uint32_t c = t % spt;   // chunk inside the block
    const uint32_t a = seg / static_cast<uint32_t>(p);
    const int i = static_cast<int>(seg - a * static_cast<uint32_t>(p));
    const uint32_t o = static_cast<uint32_t>(i) * L + c * R; // offset in the (padded) array
    const bool live = a < na;

    // prepare_blocks: load + pad (netsort.hpp:131-139)
    uint32_t v[R];
    {
        const uint32_t* src = in + (array0 + a) * len + o;
        if (live && vec_in) {
#pragma unroll
            for (int q = 0; q < R / 4; ++q) {
                if (o + 4 * q < len) {
                    const uint4 w = __ldg(reinterpret_cast<const uint4*>(src) + q);
                    v[4 * q] = w.x;
                    v[4 * q + 1] = w.y;
                    v[4 * q + 2] = w.z;
                    v[4 * q + 3] = w.w;
                } else {
                    v[4 * q] = v[4 * q + 1] = v[4 * q + 2] = v[4 * q + 3] = kPad;
                }
            }
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = (live && o + r < len) ? __ldg(src + r) : kPad;
        }
    }

    // superstep 0: local sort of every block (in-thread network, then the
    // bitonic phases k = 2R .. L)
    net.sort_r(v);
    net.template sort_phases<Sh::LR + 1, LOGL>(v);

    // supersteps 1..S: merge_split stages.  BTN stage partners are advanced
    // incrementally (bitonic_schedule, netsort.hpp:76-88: merge level a,
    // step jidx of a).
    int lvl = 1, jidx = 0;
    for (int s = 0; s < run_stages; ++s) {
        if (network == 1 && p - (s & 1) < 2) continue; // an OET round with no pair (p = 2, odd rounds)
        bool keep_low = false;
        int q = -1;
        if (live) {
            if (network == 0) {
                q = i ^ (1 << (lvl - 1 - jidx));
                keep_low = ((i >> lvl) & 1) == 0 ? (i < q) : (i > q);
            } else {
                q = oet_partner(s, i, p, keep_low);
            }
        }
        if (++jidx == lvl) {
            ++lvl;
            jidx = 0;
        }
        const uint32_t pseg = seg - static_cast<uint32_t>(i) + static_cast<uint32_t>(max(q, 0)); // partner block
        // the keep_low worker keeps the L smallest keys of the pair, the other
        // the L largest (warp-uniform for blocks of >= 32R keys)
        const bool lo = q >= 0 && keep_low, hi = q >= 0 && !keep_low;
        constexpr bool DIRECT_B = spt == 32 && Sh::BMIN <= LOGL - 1;
        if constexpr (DIRECT_B) {
            // one block per warp: read the own block and the partner's
            // reversed block straight into layout B
            uint32_t* buf = net.S + net.b;
            put_a<R>(buf, t, v);
            __syncthreads();
            if (__all_sync(0xffffffffu, q < 0)) { // idle OET edge worker: its sorted block stays
                net.b ^= net.stride;
                continue;
            }
            const uint32_t* own = buf + 36u * R * net.warp + net.lane;
            const uint32_t* par = buf + 36u * R * pseg + 36u * R - 5u - net.lane;
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = own[36 * r];
            if (__all_sync(0xffffffffu, lo)) {
#pragma unroll
                for (int r = 0; r < R; ++r) v[r] = min(v[r], par[-36 * r]);
            } else if (__all_sync(0xffffffffu, hi)) {
#pragma unroll
                for (int r = 0; r < R; ++r) v[r] = max(v[r], par[-36 * r]);
            } else if (q >= 0) {
#pragma unroll
                for (int r = 0; r < R; ++r) v[r] = minmax_sel(v[r], par[-36 * r], !keep_low);
            }
            net.b ^= net.stride;
            reg_steps<(1 << (LOGL - 6))>(v, net.fc);
            net.to_A(v);
            net.template merge_bits<4>(v);
        } else {
            uint32_t* buf = net.S + net.b;
            put_a<R>(buf, t, v);
            __syncthreads();
            if (LOGL - 1 < Sh::LR + 5 && __all_sync(0xffffffffu, q < 0)) {
                // idle OET edge workers only (their merge steps stay inside the warp)
                net.b ^= net.stride;
                continue;
            }
            const uint32_t tp = pseg * spt + (spt - 1 - c);
            if (__all_sync(0xffffffffu, lo)) apply_a<R, true>(buf, tp, v, OpMin{});
            else if (__all_sync(0xffffffffu, hi)) apply_a<R, true>(buf, tp, v, OpMax{});
            else if (q >= 0) apply_a<R, true>(buf, tp, v, OpSel{!keep_low});
            net.b ^= net.stride;
            net.template merge_bits<LOGL - 1>(v);
        }
    }

    // concatenate (+ strip the pad when the network ran to completion)
    if (!live) return;
    if (full) {
        uint32_t* dst = out + (array0 + a) * len + o;
        if (vec_out) {
#pragma unroll
            for (int q = 0; q < R / 4; ++q)
                if (o + 4 * q < len)
                    reinterpret_cast<uint4*>(dst)[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (o + r < len) dst[r] = v[r];
        }
    } else {
        uint32_t* dst = out + (array0 + a) * P + o;
        if (vec_out) {
#pragma unroll
            for (int q = 0; q < R / 4; ++q)
                reinterpret_cast<uint4*>(dst)[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) dst[r] = v[r];
        }
    }
}

template <int R, int kThreads, int MINB, int LOGL>
int launch_reg_network(const uint32_t* in, uint32_t* out, uint64_t num_arrays, uint32_t len, int p, int network,
                       int run_stages, int full, int apc, int vec_in, int vec_out, unsigned grid, unsigned threads,
                       cudaStream_t stream) {
    constexpr size_t kWords = R + R / 8; // words per thread per exchange buffer
    static PerDeviceOccupancy occ;
    kernel_occupancy(occ, block_network_reg_kernel<R, kThreads, MINB, LOGL>, kThreads, 2 * kThreads * kWords * 4);
    block_network_reg_kernel<R, kThreads, MINB, LOGL><<<grid, threads, 2 * threads * kWords * 4, stream>>>(
        in, out, num_arrays, len, p, network, run_stages, full, apc, vec_in, vec_out, 1u, 0xFFFFFFFFu);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

template <int R, int kThreads, int MINB, int LOGL = 4>
int dispatch_reg_network(int logl, const uint32_t* in, uint32_t* out, uint64_t num_arrays, uint32_t len, int p,
                         int network, int run_stages, int full, int apc, int vec_in, int vec_out, unsigned grid,
                         unsigned threads, cudaStream_t stream) {
    if constexpr ((1 << LOGL) > kThreads * R) {
        return -1;
    } else if constexpr ((1 << LOGL) < R) {
        return dispatch_reg_network<R, kThreads, MINB, LOGL + 1>(logl, in, out, num_arrays, len, p, network,
                                                                 run_stages, full, apc, vec_in, vec_out, grid, threads,
                                                                 stream);
    } else {
        if (logl == LOGL)
            return launch_reg_network<R, kThreads, MINB, LOGL>(in, out, num_arrays, len, p, network, run_stages, full,
                                                               apc, vec_in, vec_out, grid, threads, stream);
        return dispatch_reg_network<R, kThreads, MINB, LOGL + 1>(logl, in, out, num_arrays, len, p, network,
                                                                 run_stages, full, apc, vec_in, vec_out, grid, threads,
                                                                 stream);
    }
}

// Register network launch: R keys per thread, one CTA per apc arrays.
template <int R>
int launch_reg(int logl, const uint32_t* in, uint32_t* out, uint64_t num_arrays, uint32_t len, int p, uint32_t P,
               int network, int run_stages, int full, int apc, int vec_in, int vec_out, cudaStream_t stream) {
    const uint64_t grid = (num_arrays + apc - 1) / apc;
    if (grid > 0x7FFFFFFFull) return -1;
    const uint32_t threads = ((static_cast<uint32_t>(apc) * P / R) + 31u) & ~31u;
    const unsigned g = static_cast<unsigned>(grid);
    constexpr int T0 = BSG_NET_CTA_KEYS / R;      // threads of a CTA of BSG_NET_CTA_KEYS keys
    constexpr int M0 = BSG_NET_REG_TPSM / T0;     // CTAs per SM (register cap 65536 / BSG_NET_REG_TPSM)
    if (threads <= T0)
        return dispatch_reg_network<R, T0, M0>(logl, in, out, num_arrays, len, p, network, run_stages, full, apc,
                                                vec_in, vec_out, g, threads, stream);
    if (threads <= 2 * T0)
        return dispatch_reg_network<R, 2 * T0, (M0 / 2 > 0 ? M0 / 2 : 1)>(logl, in, out, num_arrays, len, p, network,
                                                                         run_stages, full, apc, vec_in, vec_out, g,
                                                                         threads, stream);
    return dispatch_reg_network<R, 4 * T0, (M0 / 4 > 0 ? M0 / 4 : 1)>(logl, in, out, num_arrays, len, p, network,
                                                                     run_stages, full, apc, vec_in, vec_out, g,
                                                                     threads, stream);
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
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_block_network(int network, const uint32_t* in, uint32_t* out, uint64_t num_arrays, uint32_t len, int p,
                         int run_stages, bool full, cudaStream_t stream) {
    const uint32_t L = (len + static_cast<uint32_t>(p) - 1) / static_cast<uint32_t>(p);
    const uint32_t P = L * static_cast<uint32_t>(p);
    if (P == 0 || P > kNetMaxPadded) return -1;
    if (BSG_NET_REG && L >= 16 && (L & (L - 1)) == 0) {
        const int apc = static_cast<int>(std::max<uint32_t>(1, BSG_NET_CTA_KEYS / P));
        const int vec_in = (len % 4 == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0) ? 1 : 0;
        const int vec_out = (len % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) ? 1 : 0;
        int logl = 0;
        while ((1u << logl) < L) ++logl;
        TimedScope ts(2 /*BSG_K_NETWORK*/, stream);
        const int f = full ? 1 : 0;
        if constexpr (BSG_NET_R == 32) {
            if (L >= 32)
                return launch_reg<32>(logl, in, out, num_arrays, len, p, P, network, run_stages, f, apc, vec_in,
                                      vec_out, stream);
        }
        return launch_reg<16>(logl, in, out, num_arrays, len, p, P, network, run_stages, f, apc, vec_in, vec_out,
                              stream);
    }
    const int apc = static_cast<int>(std::max<uint32_t>(1, 4096 / P));
    const size_t padded =static_cast<size_t>(apc) * P + (static_cast<size_t>(apc) * P >> 5) + 1;
    const size_t smem = 2ull * padded * sizeof(uint32_t);
    const uint64_t grid = (num_arrays + apc - 1) / apc;
    if (grid > 0x7FFFFFFFull) return -1;
    {
        // per device (kernel attributes do not carry over to other GPUs)
        const size_t max_smem = 2 * (kNetMaxPadded + kNetMaxPadded / 32 + 1) * sizeof(uint32_t);
        static PerDeviceOccupancy occ_small, occ_big;
        kernel_occupancy(occ_small, block_network_kernel<256, BSG_NET_MINB>, 256, max_smem);
        kernel_occupancy(occ_big, block_network_kernel<1024, 1>, 1024, max_smem);
    }
    const uint64_t resident = static_cast<uint64_t>(apc) * P;
    const bool big = resident > 8192;
    NetDivs dv;
    {
        constexpr uint32_t sk = BSG_NET_SORT32 ? 2 * kNK : kNK; // register-sort chunk (kernel: kSK)
        const uint32_t cb = (L + sk - 1) / sk, cbm = (L + kMK - 1) / kMK;
        dv.P = FastDiv(P);
        dv.pcb = FastDiv(static_cast<uint32_t>(p) * cb);
        dv.cb = FastDiv(cb);
        dv.pcbm = FastDiv(static_cast<uint32_t>(p) * cbm);
        dv.cbm = FastDiv(cbm);
        dv.len = FastDiv(len);
    }
    TimedScope ts(2 /*BSG_K_NETWORK*/, stream);
    if (!big)
        block_network_kernel<256, BSG_NET_MINB><<<static_cast<unsigned>(grid), 256, smem, stream>>>(
            in, out, num_arrays, len, p, L, network, run_stages, full ? 1 : 0, apc, dv);
    else
        block_network_kernel<1024, 1><<<static_cast<unsigned>(grid), 1024, smem, stream>>>(
            in, out, num_arrays, len, p, L, network, run_stages, full ? 1 : 0, apc, dv);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_merge_split(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb, uint32_t* low, uint32_t* high,
                       cudaStream_t stream) {
    const uint64_t total = na + nb;
    if (total == 0) return 0;
    const uint64_t chunks = (total + kNK - 1) / kNK;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((chunks + kMsThreads - 1) / kMsThreads, 148 * 16));
    merge_split_kernel<<<grid, kMsThreads, 0, stream>>>(a, static_cast<uint32_t>(na), b, static_cast<uint32_t>(nb), low,
                                                       high);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

} // namespace bsg
