// pr.cu -- parallel LSD radix sort (PR4 at r = 2^8, PR2 at r = 2^16).
//
// Restates one BSP round of run_parallel_radix (radix.hpp:260-303) per
// worker as device steps, so no per-key owner_of() division and no per-slice
// vector copies are needed:
//   count   -- count_digits (radix.hpp:127-132): digit histogram of the block.
//   plan    -- digit_starts + the routing of sort_and_scatter
//              (radix.hpp:137-179): from the p x r count matrix compute, per
//              worker, how many keys go to / come from each worker and, for the
//              rebuild, where the keys of (source v, digit d) land.  Because
//              global positions increase along a digit-sorted block, every
//              slice is a contiguous range, found from counts alone.
//   local   -- the stable local pass of sort_and_scatter (count_sort_round).
//   rebuild -- gather_slices (radix.hpp:184-222): walking (digit, source) in
//              order is a stable digit scatter of the source-major receive
//              buffer, block[delta[v][d] + j] = recv[j].
// In-process (p logical workers on one GPU, run_parallel_radix_local) the
// count matrix is read off the sorted blocks (run starts), the routing is
// O(p r) table work, and the exchange + rebuild of all workers is a single
// scatter of the sorted blocks.  Across GPUs,
// paper_1708_09495_b200/distributed.py interleaves the count / plan / local /
// rebuild steps with NCCL all-gather / all-to-all-v.
#include <dlfcn.h>
#include <mutex>
#include <nccl.h>
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "context.cuh"
#include "pr.cuh"
#include "radix.cuh"
#include "timer.cuh"

namespace bsg {

namespace {

// Binds the context's kernel timer to this thread for one C-ABI call.
struct TimerBinding {
    explicit TimerBinding(KTimer* t) { tl_timer = t; }
    ~TimerBinding() { tl_timer = nullptr; }
};

constexpr int kPlanThreads = 256;

__device__ __forceinline__ uint64_t part_size(uint64_t n, int p, int w) {
    return n / static_cast<uint64_t>(p) + (static_cast<uint64_t>(w) < n % static_cast<uint64_t>(p) ? 1 : 0);
}
__device__ __forceinline__ uint64_t part_offset(uint64_t n, int p, int w) {
    const uint64_t uw = static_cast<uint64_t>(w), big = n % static_cast<uint64_t>(p);
    return uw * (n / static_cast<uint64_t>(p)) + (uw < big ? uw : big);
}
__device__ __forceinline__ int part_owner(uint64_t n, int p, uint64_t pos) {
    const uint64_t small = n / static_cast<uint64_t>(p), bigc = n % static_cast<uint64_t>(p);
    const uint64_t big = small + 1, split = bigc * big;
    if (pos < split) return static_cast<int>(pos / big);
    return static_cast<int>(bigc + (pos - split) / small);
}
__device__ __forceinline__ uint64_t overlap(uint64_t a0, uint64_t a1, uint64_t b0, uint64_t b1) {
    const uint64_t lo = a0 > b0 ? a0 : b0, hi = a1 < b1 ? a1 : b1;
    return hi > lo ? hi - lo : 0;
}

__global__ void __launch_bounds__(kPlanThreads)
    pr_plan2_kernel(uint64_t n, int p, int me, int radix, const uint64_t* __restrict__ recv_counts,
                    const uint64_t* __restrict__ split, int64_t* __restrict__ delta) {
    const int v = blockIdx.x;
    uint64_t recv_off = 0;
    for (int u = 0; u < v; ++u) recv_off += recv_counts[u];
    const int64_t adj = static_cast<int64_t>(split[v]) - static_cast<int64_t>(recv_off) -
                        static_cast<int64_t>(part_offset(n, p, me));
    for (int d = threadIdx.x; d < radix; d += kPlanThreads) delta[static_cast<uint64_t>(v) * radix + d] += adj;
}

constexpr int kRebuildThreads = 256;
constexpr int kMaxP = 1024;

__global__ void __launch_bounds__(kRebuildThreads)
    pr_rebuild_kernel(const uint32_t* __restrict__ recv, uint64_t recv_len, int p,
                      const uint64_t* __restrict__ recv_counts,
                      uint32_t mask, int shift, int radix, const int64_t* __restrict__ delta,
                      uint32_t* __restrict__ block, uint32_t* __restrict__ proto) {
    __shared__ uint64_t s_off[kMaxP + 1];
    if (threadIdx.x == 0) {
        uint64_t run = 0;
        for (int v = 0; v < p; ++v) {
            s_off[v] = run;
            run += recv_counts[v];
        }
        s_off[p] = run;
        // the received slices must fill the block exactly (radix.hpp:207-220)
        if (run != recv_len && proto && blockIdx.x == 0) atomicOr(proto, 1u);
    }
    __syncthreads();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kRebuildThreads;
    for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * kRebuildThreads + threadIdx.x; j < recv_len; j += stride) {
        int lo = 0, hi = p - 1; // largest v with s_off[v] <= j
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_off[mid] <= j) lo = mid;
            else hi = mid - 1;
        }
        const int v = lo;
        const uint32_t key = recv[j];
        const uint32_t d = (key >> shift) & mask;
        const int64_t dst = delta[static_cast<uint64_t>(v) * radix + d] + static_cast<int64_t>(j);
        if (dst < 0 || static_cast<uint64_t>(dst) >= recv_len) { // a slice disagrees with the counts
            if (proto) atomicOr(proto, 1u);
            continue;
        }
        block[dst] = key;
    }
}

// 16-bit digit histogram: 65536 16-bit counters packed in 128 KiB of shared
// memory; a counter that reaches 2^15 carries 2^15 to the global uint64 bin.
constexpr int kHist16Threads = 1024;

__global__ void __launch_bounds__(kHist16Threads)
    hist16_kernel(const uint32_t* __restrict__ in, uint64_t n, int shift, unsigned long long* __restrict__ counts) {
    extern __shared__ uint32_t h16[]; // 32768 words
    for (int i = threadIdx.x; i < 32768; i += kHist16Threads) h16[i] = 0;
    __syncthreads();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kHist16Threads;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kHist16Threads + threadIdx.x; i < n; i += stride) {
        const uint32_t d = (__ldg(in + i) >> shift) & 0xFFFFu;
        const uint32_t sh = (d & 1u) * 16u;
        const uint32_t old = atomicAdd(&h16[d >> 1], 1u << sh);
        if (((old >> sh) & 0xFFFFu) == 0x7FFFu) {
            atomicSub(&h16[d >> 1], 0x8000u << sh);
            atomicAdd(&counts[d], 0x8000ull);
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 65536; d += kHist16Threads) {
        const uint32_t c = (h16[d >> 1] >> ((d & 1) * 16)) & 0xFFFFu;
        if (c) atomicAdd(&counts[d], static_cast<unsigned long long>(c));
    }
}

// ---- in-process round (p logical workers on one GPU) ----------------------
// The rebuild of every worker together is one scatter of the locally sorted
// blocks: key i of worker v's sorted block with digit d lands at
//   np(v,d) + (i - ls(v,d)),  np(v,d) = start[d] + sum_{u<v} cnt(u,d)
// (radix.hpp:146-179 next_pos / gather order), ls(v,d) = first index of d in
// v's sorted block.  All tables are O(p r) work.

// ls(v,d) for d in [0, r]: lower bound of digit d in v's sorted block (the
// block's digit counts are ls(v,d+1) - ls(v,d), as count_digits would give).
__global__ void pr_run_starts_kernel(const uint32_t* __restrict__ sorted, uint64_t n, int p, int shift,
                                     uint32_t mask, int radix, uint64_t* __restrict__ starts) {
    const int v = blockIdx.y;
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d > static_cast<uint32_t>(radix)) return;
    const uint64_t off = part_offset(n, p, v), len = part_size(n, p, v);
    const uint32_t* blk = sorted + off;
    uint64_t lo = 0, hi = len;
    if (d == static_cast<uint32_t>(radix)) lo = len;
    else
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (((__ldg(blk + mid) >> shift) & mask) < d) lo = mid + 1;
            else hi = mid;
        }
    starts[static_cast<uint64_t>(v) * (radix + 1) + d] = lo;
}

// Digit tables are processed in chunks of kDigChunk digits, one CTA each
// (coalesced, no single-CTA loops over r).
constexpr int kDigChunk = 1024;

// Block-wide exclusive scan (kDigChunk threads); returns the block total.
__device__ __forceinline__ uint64_t chunk_excl_scan(uint64_t v, uint64_t& excl) {
    __shared__ uint64_t s_warp[kDigChunk / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t incl = warp_inclusive_scan(v);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint64_t pre = 0, total = 0;
    for (int w = 0; w < kDigChunk / 32; ++w) {
        const uint64_t x = s_warp[w];
        pre += w < warp ? x : 0;
        total += x;
    }
    excl = pre + incl - v;
    __syncthreads();
    return total;
}

// Sum of tab[0 .. k) computed by warp 0 and broadcast (k <= a few hundred).
__device__ __forceinline__ uint64_t chunk_base(const uint64_t* tab, int k) {
    __shared__ uint64_t s_base;
    if (threadIdx.x < 32) {
        uint64_t acc = 0;
        for (int i = threadIdx.x; i < k; i += 32) acc += tab[i];
        acc = warp_sum(acc);
        if (threadIdx.x == 0) s_base = acc;
    }
    __syncthreads();
    return s_base;
}

// Column prefix over workers from the run starts: gd[v][d] = sum_{u<v}
// cnt(u,d) - ls(v,d); coltot[d] = sum_u cnt(u,d); colchunk[c] = chunk sums.
__global__ void __launch_bounds__(kDigChunk)
    pr_col_prefix_kernel(const uint64_t* __restrict__ starts, int p, int radix, int64_t* __restrict__ gd,
                         uint64_t* __restrict__ coltot, uint64_t* __restrict__ colchunk) {
    const int d = blockIdx.x * kDigChunk + threadIdx.x;
    uint64_t before = 0;
    if (d < radix) {
        for (int v = 0; v < p; ++v) {
            const uint64_t* row = starts + static_cast<uint64_t>(v) * (radix + 1);
            const uint64_t ls = row[d], c = row[d + 1] - ls;
            gd[static_cast<uint64_t>(v) * radix + d] = static_cast<int64_t>(before) - static_cast<int64_t>(ls);
            before += c;
        }
        coltot[d] = before;
    }
    uint64_t ex;
    const uint64_t tot = chunk_excl_scan(before, ex);
    if (threadIdx.x == 0) colchunk[blockIdx.x] = tot;
}

// start[d] = exclusive scan of coltot over all digits (digit_starts).
__global__ void __launch_bounds__(kDigChunk)
    pr_digit_start_kernel(const uint64_t* __restrict__ coltot, const uint64_t* __restrict__ colchunk, int radix,
                          uint64_t* __restrict__ start) {
    const uint64_t base = chunk_base(colchunk, blockIdx.x);
    const int d = blockIdx.x * kDigChunk + threadIdx.x;
    const uint64_t c = d < radix ? coltot[d] : 0;
    uint64_t ex;
    chunk_excl_scan(c, ex);
    if (d < radix) start[d] = base + ex;
}

// Exchange + rebuild of all workers: one coalesced scatter (digit runs of a
// sorted block land on consecutive positions).
constexpr int kScatterThreads = 256, kScatterItems = 16;
__global__ void __launch_bounds__(kScatterThreads)
    pr_scatter_kernel(const uint32_t* __restrict__ sorted, uint64_t n, int p, int shift, uint32_t mask, int radix,
                      const uint64_t* __restrict__ start, const int64_t* __restrict__ gd, uint32_t* __restrict__ out) {
    const int v = blockIdx.y;
    const uint64_t off = part_offset(n, p, v), len = part_size(n, p, v);
    const uint32_t* blk = sorted + off;
    const int64_t* gdv = gd + static_cast<uint64_t>(v) * radix;
    const uint64_t step = static_cast<uint64_t>(gridDim.x) * kScatterThreads;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kScatterThreads + threadIdx.x; i < len; i += step) {
        const uint32_t key = __ldg(blk + i);
        const uint32_t d = (key >> shift) & mask;
        out[static_cast<uint64_t>(static_cast<int64_t>(__ldg(start + d)) + __ldg(gdv + d) + static_cast<int64_t>(i))] =
            key;
    }
}

// BSP accounting only (RunStats): send[v][w] = keys of worker v's block that
// land in worker w's partition (the slices of radix.hpp:165-178).
constexpr int kSendThreads = 256;
__global__ void __launch_bounds__(kSendThreads)
    pr_send_counts_kernel(const uint64_t* __restrict__ starts, const uint64_t* __restrict__ start,
                          const int64_t* __restrict__ gd, uint64_t n, int p, int radix, uint64_t* __restrict__ send) {
    extern __shared__ unsigned long long s_cnt[]; // p entries
    const int v = blockIdx.y;
    for (int w = threadIdx.x; w < p; w += kSendThreads) s_cnt[w] = 0;
    __syncthreads();
    const int d = blockIdx.x * kSendThreads + threadIdx.x;
    if (d < radix) {
        const uint64_t* row = starts + static_cast<uint64_t>(v) * (radix + 1);
        const uint64_t ls = row[d], cv = row[d + 1] - ls;
        if (cv) {
            const uint64_t np = static_cast<uint64_t>(static_cast<int64_t>(start[d]) + gd[static_cast<uint64_t>(v) * radix + d] +
                                                      static_cast<int64_t>(ls));
            const int w0 = part_owner(n, p, np), w1 = part_owner(n, p, np + cv - 1);
            for (int w = w0; w <= w1; ++w) {
                const uint64_t lo = part_offset(n, p, w);
                const uint64_t o = overlap(np, np + cv, lo, lo + part_size(n, p, w));
                if (o) atomicAdd(&s_cnt[w], static_cast<unsigned long long>(o));
            }
        }
    }
    __syncthreads();
    for (int w = threadIdx.x; w < p; w += kSendThreads)
        if (s_cnt[w]) atomicAdd(reinterpret_cast<unsigned long long*>(send + static_cast<uint64_t>(v) * p + w), s_cnt[w]);
}

// ---- routing plan of one worker `me` (distributed path, bsg_pr_plan) ------
// Same O(p r) tables as the in-process round, from the gathered count matrix:
//   col:  delta[v][d] = sum_{u<v} cnt(u,d) (temporary), coltot[d]
//   scan: dstart[d] = exclusive scan of coltot (digit_starts)
//   row:  one CTA per source v: ls(v,d) = row prefix of cnt(v,.), np(v,d) =
//         dstart[d] + before(v,d); recv/split overlaps with me's partition;
//         send slices of me (radix.hpp:165-178); delta[v][d] = np - ls.
//   adj:  pr_plan2_kernel rebases delta onto me's receive buffer.
__global__ void __launch_bounds__(kDigChunk)
    pr_plan_col_kernel(const uint64_t* __restrict__ counts, int p, int radix, int64_t* __restrict__ delta,
                       uint64_t* __restrict__ coltot, uint64_t* __restrict__ colchunk,
                       uint32_t* __restrict__ skew = nullptr, uint64_t n = 0) {
    const int d = blockIdx.x * kDigChunk + threadIdx.x;
    uint64_t before = 0;
    if (d < radix) {
        bool heavy = false;
        for (int v = 0; v < p; ++v) {
            delta[static_cast<uint64_t>(v) * radix + d] = static_cast<int64_t>(before);
            const uint64_t c = counts[static_cast<uint64_t>(v) * radix + d];
            before += c;
            heavy = heavy || c * 16 > part_size(n, p, v);
        }
        coltot[d] = before;
        // a digit holding > 1/16 of some block: that round's pass ranks first
        if (skew && heavy) atomicOr(skew, 1u);
    }
    uint64_t ex;
    const uint64_t tot = chunk_excl_scan(before, ex);
    if (threadIdx.x == 0) colchunk[blockIdx.x] = tot;
}

// rowchunk[v][c] = sum of cnt(v, chunk c)
__global__ void __launch_bounds__(kDigChunk)
    pr_plan_rowchunk_kernel(const uint64_t* __restrict__ counts, int radix, uint64_t* __restrict__ rowchunk) {
    const int v = blockIdx.y, d = blockIdx.x * kDigChunk + threadIdx.x;
    const uint64_t c = d < radix ? counts[static_cast<uint64_t>(v) * radix + d] : 0;
    uint64_t ex;
    const uint64_t tot = chunk_excl_scan(c, ex);
    if (threadIdx.x == 0) rowchunk[static_cast<uint64_t>(v) * gridDim.x + blockIdx.x] = tot;
}

// One CTA per (digit chunk, source v).  recv_counts / split / send_counts
// must be zero on entry (accumulated with atomics).
__global__ void __launch_bounds__(kDigChunk)
    pr_plan_row_kernel(const uint64_t* __restrict__ counts, const uint64_t* __restrict__ dstart,
                       const uint64_t* __restrict__ rowchunk, uint64_t n, int p, int me, int radix,
                       uint64_t* __restrict__ send_counts, uint64_t* __restrict__ recv_counts,
                       int64_t* __restrict__ delta, uint64_t* __restrict__ split) {
    extern __shared__ unsigned long long s_send[]; // p entries (v == me only)
    __shared__ uint64_t s_red[2][kDigChunk / 32];
    const int v = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (v == me)
        for (int w = tid; w < p; w += kDigChunk) s_send[w] = 0;
    const uint64_t lbase = chunk_base(rowchunk + static_cast<uint64_t>(v) * gridDim.x, blockIdx.x);
    const int d = blockIdx.x * kDigChunk + tid;
    const uint64_t cv = d < radix ? counts[static_cast<uint64_t>(v) * radix + d] : 0;
    uint64_t ex;
    chunk_excl_scan(cv, ex);
    uint64_t acc_recv = 0, acc_split = 0;
    if (d < radix) {
        const uint64_t ls = lbase + ex;
        int64_t* dp = delta + static_cast<uint64_t>(v) * radix + d;
        const uint64_t np = dstart[d] + static_cast<uint64_t>(*dp);
        const uint64_t lo_me = part_offset(n, p, me), hi_me = lo_me + part_size(n, p, me);
        acc_recv = overlap(np, np + cv, lo_me, hi_me);
        acc_split = overlap(np, np + cv, 0, lo_me);
        *dp = static_cast<int64_t>(np) - static_cast<int64_t>(ls);
        if (v == me && cv) {
            const int w0 = part_owner(n, p, np), w1 = part_owner(n, p, np + cv - 1);
            for (int w = w0; w <= w1; ++w) {
                const uint64_t lo = part_offset(n, p, w);
                const uint64_t o = overlap(np, np + cv, lo, lo + part_size(n, p, w));
                if (o) atomicAdd(&s_send[w], static_cast<unsigned long long>(o));
            }
        }
    }
    const uint64_t r1 = warp_sum(acc_recv), r2 = warp_sum(acc_split);
    if (lane == 0) {
        s_red[0][warp] = r1;
        s_red[1][warp] = r2;
    }
    __syncthreads();
    if (tid == 0) {
        uint64_t a = 0, b = 0;
        for (int w = 0; w < kDigChunk / 32; ++w) {
            a += s_red[0][w];
            b += s_red[1][w];
        }
        if (a) atomicAdd(reinterpret_cast<unsigned long long*>(recv_counts + v), static_cast<unsigned long long>(a));
        if (b) atomicAdd(reinterpret_cast<unsigned long long*>(split + v), static_cast<unsigned long long>(b));
    }
    if (v == me)
        for (int w = tid; w < p; w += kDigChunk)
            if (s_send[w]) atomicAdd(reinterpret_cast<unsigned long long*>(send_counts + w), s_send[w]);
}

// ---- fused exchange + rebuild over peer memory (bsg_pr_peer_scatter) -----
// gd[d] = digit_start[d] + sum_{u<me} cnt(u,d) - ls(me,d): the destination of
// key i (digit d) of me's sorted block is gd[d] + i (radix.hpp:146-179).
// `before` holds sum_{u<me} cnt(u,d) (pr_plan_col_kernel's delta row me).
__global__ void __launch_bounds__(kDigChunk)
    pr_peer_gd_kernel(const uint64_t* __restrict__ cnt_me, const int64_t* __restrict__ before,
                      const uint64_t* __restrict__ dstart, int radix, int64_t* __restrict__ gd) {
    __shared__ uint64_t s_part[kDigChunk / 32];
    // row prefix of me's counts up to this chunk
    uint64_t acc = 0;
    for (int d = threadIdx.x; d < static_cast<int>(blockIdx.x) * kDigChunk; d += kDigChunk) acc += cnt_me[d];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = acc;
    __syncthreads();
    uint64_t lbase = 0;
    for (int w = 0; w < kDigChunk / 32; ++w) lbase += s_part[w];
    const int d = blockIdx.x * kDigChunk + threadIdx.x;
    const uint64_t c = d < radix ? cnt_me[d] : 0;
    uint64_t ex;
    chunk_excl_scan(c, ex);
    if (d < radix)
        gd[d] = static_cast<int64_t>(dstart[d]) + before[d] - static_cast<int64_t>(lbase + ex);
}

// Owner by p boundary compares (no per-key division, cf. radix.hpp:113-117).
__global__ void __launch_bounds__(kScatterThreads)
    pr_peer_scatter_kernel(const uint32_t* __restrict__ sorted, uint64_t len, int shift, uint32_t mask,
                           const int64_t* __restrict__ gd, int p, const __grid_constant__ PeerTable tab) {
    const uint64_t step = static_cast<uint64_t>(gridDim.x) * kScatterThreads;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kScatterThreads + threadIdx.x; i < len; i += step) {
        const uint32_t key = __ldg(sorted + i);
        const uint64_t pos = static_cast<uint64_t>(__ldg(gd + ((key >> shift) & mask)) + static_cast<int64_t>(i));
        if (pos >= tab.offset[p]) continue; // inconsistent count matrix (reported by the row check)
        int w = 0;
        for (int j = 1; j < p; ++j) w += pos >= tab.offset[j] ? 1 : 0;
        tab.blocks[w][pos - tab.offset[w]] = key;
    }
    __threadfence_system(); // peer stores performed before the round's barrier
}

// Protocol check of an exchanged count matrix (the reference's bsp_error,
// radix.hpp:207-220 and 283-286): row v (worker v's digit counts) must sum to
// Partition(n, p).size_of(v).  One CTA per row; a mismatch sets *flag.
__global__ void __launch_bounds__(256) pr_check_rows_kernel(const uint64_t* __restrict__ counts, int p, int radix,
                                                            uint64_t n, uint32_t* __restrict__ flag) {
    __shared__ uint64_t s_part[8];
    const int v = blockIdx.x;
    uint64_t sum = 0;
    for (int d = threadIdx.x; d < radix; d += 256) sum += counts[static_cast<uint64_t>(v) * radix + d];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t tot = 0;
        for (int w = 0; w < 8; ++w) tot += s_part[w];
        const uint64_t want = n / static_cast<uint64_t>(p) + (static_cast<uint64_t>(v) < n % static_cast<uint64_t>(p) ? 1 : 0);
        if (tot != want) atomicOr(flag, 1u);
    }
}

// digit_base[d] = digit_start[d] + sum_{u<me} cnt(u,d): global position of
// the first digit-d key of me's block (one-sweep digit bases of the fused round)
__global__ void pr_fused_base_kernel(const uint64_t* __restrict__ dstart, const int64_t* __restrict__ before_me,
                                     int radix, uint64_t* __restrict__ base) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d < radix) base[d] = dstart[d] + static_cast<uint64_t>(before_me[d]);
}

// count_digits of every worker block in one launch (grid.y = worker).
// Lane-private shared counters (counter c of lane l at word c*32 + l: a
// warp's 32 increments never share a bank, as in K1), 4 loads in flight per
// thread; one global atomic per (CTA, digit).  counts must be zero on entry.
constexpr int kSegCountThreads = 512;
template <int RADIX>
__global__ void __launch_bounds__(kSegCountThreads)
    pr_seg_count_kernel(const uint32_t* __restrict__ keys, uint64_t n, int p, int shift,
                        unsigned long long* __restrict__ counts) {
    __shared__ uint32_t h[RADIX * 32];
    for (int i = threadIdx.x; i < RADIX * 32; i += kSegCountThreads) h[i] = 0;
    __syncthreads();
    const int w = blockIdx.y;
    const uint64_t off = part_offset(n, p, w), len = part_size(n, p, w);
    uint32_t* mine = h + (threadIdx.x & 31);
    const uint32_t* blk = keys + off;
    const uint64_t step = static_cast<uint64_t>(gridDim.x) * kSegCountThreads;
    uint64_t i = static_cast<uint64_t>(blockIdx.x) * kSegCountThreads + threadIdx.x;
    if constexpr (RADIX == 256) {
        // byte digits: 16-byte loads (four in flight per thread), one PRMT +
        // one IMAD per key; the block's unaligned head and tail scalar
        const uint32_t sel = 0x4440u | static_cast<uint32_t>(shift >> 3);
        const uint32_t lane4 = (threadIdx.x & 31u) * 4u;
        auto cnt = [&](uint32_t k) {
            atomicAdd(reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(h) + __byte_perm(k, 0u, sel) * 128u +
                                                  lane4),
                      1u);
        };
        const uint64_t mis = (reinterpret_cast<uintptr_t>(blk) >> 2) & 3u;
        const uint64_t head = min(len, mis ? 4 - mis : 0);
        const uint4* body = reinterpret_cast<const uint4*>(blk + head);
        const uint64_t nvec = (len - head) / 4;
        uint64_t v = i;
        for (; v + 3 * step < nvec; v += 4 * step) {
            const uint4 a = ldg_stream_v4(body + v), b = ldg_stream_v4(body + v + step),
                        c = ldg_stream_v4(body + v + 2 * step), e = ldg_stream_v4(body + v + 3 * step);
            cnt(a.x); cnt(a.y); cnt(a.z); cnt(a.w);
            cnt(b.x); cnt(b.y); cnt(b.z); cnt(b.w);
            cnt(c.x); cnt(c.y); cnt(c.z); cnt(c.w);
            cnt(e.x); cnt(e.y); cnt(e.z); cnt(e.w);
        }
        for (; v < nvec; v += step) {
            const uint4 a = ldg_stream_v4(body + v);
            cnt(a.x); cnt(a.y); cnt(a.z); cnt(a.w);
        }
        if (blockIdx.x == 0) {
            for (uint64_t j = threadIdx.x; j < head; j += kSegCountThreads) cnt(__ldg(blk + j));
            for (uint64_t j = head + nvec * 4 + threadIdx.x; j < len; j += kSegCountThreads) cnt(__ldg(blk + j));
        }
        i = len; // done
    }
    for (; i + 3 * step < len; i += 4 * step) {
        const uint32_t k0 = __ldg(blk + i), k1 = __ldg(blk + i + step), k2 = __ldg(blk + i + 2 * step),
                       k3 = __ldg(blk + i + 3 * step);
        atomicAdd(mine + ((k0 >> shift) & (RADIX - 1)) * 32, 1u);
        atomicAdd(mine + ((k1 >> shift) & (RADIX - 1)) * 32, 1u);
        atomicAdd(mine + ((k2 >> shift) & (RADIX - 1)) * 32, 1u);
        atomicAdd(mine + ((k3 >> shift) & (RADIX - 1)) * 32, 1u);
    }
    for (; i < len; i += step) atomicAdd(mine + ((__ldg(blk + i) >> shift) & (RADIX - 1)) * 32, 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < RADIX; d += kSegCountThreads) {
        uint32_t c = 0;
#pragma unroll 8
        for (int l = 0; l < 32; ++l) c += h[d * 32 + ((l + d) & 31)]; // rotated: no bank conflicts
        if (c) atomicAdd(&counts[static_cast<uint64_t>(w) * RADIX + d], static_cast<unsigned long long>(c));
    }
}

int launch_pr_seg_count(const uint32_t* keys, uint64_t n, int p, int bits, int shift, uint64_t* counts,
                        cudaStream_t stream) {
    const int radix = 1 << bits;
    if (cudaMemsetAsync(counts, 0, static_cast<uint64_t>(p) * radix * sizeof(uint64_t), stream) != cudaSuccess)
        return -1;
    if (n == 0) return 0;
    const uint64_t per = n / static_cast<uint64_t>(p) + 1;
    const uint64_t want = (per + kSegCountThreads * 64 - 1) / (kSegCountThreads * 64);
    const unsigned gx = static_cast<unsigned>(std::max<uint64_t>(
        1, std::min<uint64_t>(want, std::max<uint64_t>(1, kSmCountB200 * 4 / static_cast<uint64_t>(p)))));
    auto* c = reinterpret_cast<unsigned long long*>(counts);
    const dim3 grid(gx, static_cast<unsigned>(p));
    switch (bits) {
    case 1: pr_seg_count_kernel<2><<<grid, kSegCountThreads, 0, stream>>>(keys, n, p, shift, c); break;
    case 2: pr_seg_count_kernel<4><<<grid, kSegCountThreads, 0, stream>>>(keys, n, p, shift, c); break;
    case 4: pr_seg_count_kernel<16><<<grid, kSegCountThreads, 0, stream>>>(keys, n, p, shift, c); break;
    case 8: pr_seg_count_kernel<256><<<grid, kSegCountThreads, 0, stream>>>(keys, n, p, shift, c); break;
    default: return -1;
    }
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// Segment-local digit bases of an 8-bit sub-pass: base[w][d] = offset_of(w) +
// sum_{d'<d} cnt(w, d'), so a segmented one-sweep pass sorts every worker's
// block in place (the two byte sub-passes of an r = 2^16 local pass).
__global__ void __launch_bounds__(256)
    pr_local_base_kernel(const uint64_t* __restrict__ counts, uint64_t n, int p, int64_t* __restrict__ base,
                         uint32_t* __restrict__ skew) {
    __shared__ uint64_t s_w[8];
    const int w = blockIdx.x, d = threadIdx.x, lane = d & 31, wp = d >> 5;
    const uint64_t c = counts[static_cast<uint64_t>(w) * 256 + d];
    if (c * 16 > part_size(n, p, w)) atomicOr(skew, 1u); // heavy byte: that sub-pass ranks first
    const uint64_t incl = warp_inclusive_scan(c);
    if (lane == 31) s_w[wp] = incl;
    __syncthreads();
    uint64_t excl = incl - c;
    for (int j = 0; j < wp; ++j) excl += s_w[j];
    base[static_cast<uint64_t>(w) * 256 + d] = static_cast<int64_t>(part_offset(n, p, w) + excl);
}

// In-process fused round: base[v][d] = digit_start[d] + sum_{u<v} cnt(u,d),
// in place over the column-prefix table.
__global__ void pr_add_dstart_kernel(int64_t* __restrict__ before, const uint64_t* __restrict__ dstart, int p,
                                     int radix) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < static_cast<uint64_t>(p) * radix) before[i] += static_cast<int64_t>(dstart[i % radix]);
}

// RunStats send counts from the count matrix: worker v's digit-d run
// [base[v][d], + cnt(v,d)) split over the partitions it overlaps.
__global__ void __launch_bounds__(kSendThreads)
    pr_send_from_counts_kernel(const uint64_t* __restrict__ counts, const int64_t* __restrict__ base, uint64_t n,
                               int p, int radix, uint64_t* __restrict__ send) {
    extern __shared__ unsigned long long s_cnt2[]; // p entries
    const int v = blockIdx.y;
    for (int w = threadIdx.x; w < p; w += kSendThreads) s_cnt2[w] = 0;
    __syncthreads();
    const int d = blockIdx.x * kSendThreads + threadIdx.x;
    if (d < radix) {
        const uint64_t cv = counts[static_cast<uint64_t>(v) * radix + d];
        if (cv) {
            const uint64_t np = static_cast<uint64_t>(base[static_cast<uint64_t>(v) * radix + d]);
            const int w0 = part_owner(n, p, np), w1 = part_owner(n, p, np + cv - 1);
            for (int w = w0; w <= w1; ++w) {
                const uint64_t lo = part_offset(n, p, w);
                const uint64_t o = overlap(np, np + cv, lo, lo + part_size(n, p, w));
                if (o) atomicAdd(&s_cnt2[w], static_cast<unsigned long long>(o));
            }
        }
    }
    __syncthreads();
    for (int w = threadIdx.x; w < p; w += kSendThreads)
        if (s_cnt2[w]) atomicAdd(reinterpret_cast<unsigned long long*>(send + static_cast<uint64_t>(v) * p + w), s_cnt2[w]);
}

// Exchange + rebuild of one group member's workers (r = 2^16 group rounds):
// key i of local worker lv's sorted block (global worker wlo + lv) with
// digit d goes to global position start[d] + gd[wlo+lv][d] + i and is stored
// in the owning member's next-round buffer (PeerTable over G members).
__global__ void __launch_bounds__(kScatterThreads)
    pr_scatter_peer_kernel(const uint32_t* __restrict__ sorted, uint64_t len, int pw, int wlo, int shift,
                           uint32_t mask, int radix, const uint64_t* __restrict__ start,
                           const int64_t* __restrict__ gd, const __grid_constant__ PeerTable tab, int G) {
    const int lv = blockIdx.y;
    const uint64_t off = part_offset(len, pw, lv), blen = part_size(len, pw, lv);
    const uint32_t* blk = sorted + off;
    const int64_t* gdv = gd + static_cast<uint64_t>(wlo + lv) * radix;
    const uint64_t step = static_cast<uint64_t>(gridDim.x) * kScatterThreads;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kScatterThreads + threadIdx.x; i < blen; i += step) {
        const uint32_t key = __ldg(blk + i);
        const uint32_t d = (key >> shift) & mask;
        const uint64_t pos =
            static_cast<uint64_t>(static_cast<int64_t>(__ldg(start + d)) + __ldg(gdv + d) + static_cast<int64_t>(i));
        int m = 0;
        for (int j = 1; j < G; ++j) m += pos >= tab.offset[j] ? 1 : 0;
        tab.blocks[m][pos - tab.offset[m]] = key;
    }
    __threadfence_system();
}

} // namespace

int launch_pr_count(bsg_ctx* ctx, const uint32_t* block, uint64_t len, int round, int bits, uint64_t* counts,
                    cudaStream_t stream) {
    const int radix = 1 << bits;
    if (bits == 16) {
        if (cudaMemsetAsync(counts, 0, radix * sizeof(uint64_t), stream) != cudaSuccess) return -1;
        if (len == 0) return 0;
        static PerDeviceOccupancy occ; // attribute per device
        kernel_occupancy(occ, hist16_kernel, kHist16Threads, 32768 * 4);
        const uint64_t want = (len + kHist16Threads * 16 - 1) / (kHist16Threads * 16);
        const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, kSmCountB200)));
        hist16_kernel<<<grid, kHist16Threads, 32768 * 4, stream>>>(block, len, 16 * round,
                                                                   reinterpret_cast<unsigned long long*>(counts));
        return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
    }
    const uint64_t chunks = len ? (len + kChunkKeys - 1) / kChunkKeys : 1;
    if (ctx->cnt32.ensure(chunks * 256 * sizeof(uint32_t)) != cudaSuccess) return -1;
    if (len == 0) {
        if (cudaMemsetAsync(counts, 0, radix * sizeof(uint64_t), stream) != cudaSuccess) return -1;
        return 0;
    }
    return launch_digit_counts(block, len, bits, round * bits, counts, ctx->cnt32.as<uint32_t>(), stream);
}

int launch_pr_plan(const uint64_t* counts, uint64_t n, int p, int me, int bits, uint64_t* send_counts,
                   uint64_t* recv_counts, int64_t* rebuild_delta, cudaStream_t stream, uint64_t* scratch) {
    if (!scratch || p > kMaxP) return -1;
    const int radix = 1 << bits;
    const int chunks = (radix + kDigChunk - 1) / kDigChunk;
    uint64_t* split = scratch;                 // [p]
    uint64_t* coltot = split + p;              // [radix]
    uint64_t* dstart = coltot + radix;         // [radix]
    uint64_t* colchunk = dstart + radix;       // [chunks]
    uint64_t* rowchunk = colchunk + chunks;    // [p][chunks]
    TimedScope ts(3 /*BSG_K_PR*/, stream);
    if (cudaMemsetAsync(split, 0, p * sizeof(uint64_t), stream) != cudaSuccess ||
        cudaMemsetAsync(recv_counts, 0, p * sizeof(uint64_t), stream) != cudaSuccess ||
        cudaMemsetAsync(send_counts, 0, p * sizeof(uint64_t), stream) != cudaSuccess)
        return -1;
    pr_plan_col_kernel<<<chunks, kDigChunk, 0, stream>>>(counts, p, radix, rebuild_delta, coltot, colchunk);
    pr_plan_rowchunk_kernel<<<dim3(chunks, p), kDigChunk, 0, stream>>>(counts, radix, rowchunk);
    pr_digit_start_kernel<<<chunks, kDigChunk, 0, stream>>>(coltot, colchunk, radix, dstart);
    pr_plan_row_kernel<<<dim3(chunks, p), kDigChunk, sizeof(uint64_t) * p, stream>>>(
        counts, dstart, rowchunk, n, p, me, radix, send_counts, recv_counts, rebuild_delta, split);
    pr_plan2_kernel<<<p, kPlanThreads, 0, stream>>>(n, p, me, radix, recv_counts, split, rebuild_delta);
    return cudaPeekAtLastError() == cudaSuccess ? 5 : -1;
}

// Protocol flag of a call: zeroed on the call's stream before its kernels
// (proto_begin), read back with a stream synchronisation after them
// (proto_end -> BSG_EPROTO).  Kernels never store outside their blocks when
// the flag is raised.
int proto_begin(bsg_ctx* ctx, cudaStream_t st, uint32_t** flag) {
    cudaError_t e = ctx->proto.ensure(sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemsetAsync(ctx->proto.as<uint32_t>(), 0, sizeof(uint32_t), st);
    if (e != cudaSuccess) return cuda_fail(e, "protocol flag");
    *flag = ctx->proto.as<uint32_t>();
    return BSG_OK;
}
int proto_end(bsg_ctx* ctx, cudaStream_t st, const char* what) {
    uint32_t h = 0;
    cudaError_t e = cudaMemcpyAsync(&h, ctx->proto.as<uint32_t>(), sizeof(uint32_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "protocol flag");
    return h ? fail(BSG_EPROTO, what) : BSG_OK;
}
int check_count_rows(const uint64_t* counts, int p, int radix, uint64_t n, uint32_t* flag, cudaStream_t st) {
    pr_check_rows_kernel<<<p, 256, 0, st>>>(counts, p, radix, n, flag);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_pr_rebuild(const uint32_t* recv, uint64_t recv_len, int bits, int shift, const int64_t* rebuild_delta,
                      uint32_t* block, cudaStream_t stream, const uint64_t* recv_counts, int p, uint32_t* proto) {
    if (p > kMaxP) return -1;
    if (recv_len == 0) return 0;
    const uint64_t want = (recv_len + kRebuildThreads * 8 - 1) / (kRebuildThreads * 8);
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, kSmCountB200 * 8)));
    TimedScope ts(3 /*BSG_K_PR*/, stream);
    pr_rebuild_kernel<<<grid, kRebuildThreads, 0, stream>>>(recv, recv_len, p, recv_counts, (1u << bits) - 1u,
                                                           shift, 1 << bits, rebuild_delta, block, proto);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int run_parallel_radix_local(bsg_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n, int p, int bits, int rounds,
                             bsg_run_stats* stats, cudaStream_t stream) {
    if (p > kMaxP) return fail(BSG_EINVAL, "parallel radix sort: p must be <= 1024 on one GPU");
    const int radix = 1 << bits;
    const uint32_t mask = static_cast<uint32_t>(radix - 1);
    const uint64_t pp = static_cast<uint64_t>(p) * p;
    cudaError_t e;
    if ((e = ctx->pr_block.ensure(std::max<uint64_t>(n, 4) * 4)) != cudaSuccess) return cuda_fail(e, "pr workspace");
    if ((e = ctx->pr_sorted.ensure(std::max<uint64_t>(n, 4) * 4)) != cudaSuccess) return cuda_fail(e, "pr workspace");
    if ((e = ctx->pr_counts.ensure(static_cast<uint64_t>(p) * (radix + 1) * 8)) != cudaSuccess)
        return cuda_fail(e, "pr workspace");
    if ((e = ctx->pr_delta.ensure(static_cast<uint64_t>(p) * radix * 8)) != cudaSuccess) return cuda_fail(e, "pr workspace");
    if ((e = ctx->pr_misc.ensure(pp * 8 + static_cast<uint64_t>(radix) * 16 + 128 * 8)) != cudaSuccess)
        return cuda_fail(e, "pr workspace");
    if (bits == 16 && (e = ctx->stage_b.ensure(std::max<uint64_t>(n, 4) * 4)) != cudaSuccess) return cuda_fail(e, "pr workspace");
    RadixWorkspace ws;
    if (int rc = ctx->radix_ws(std::max<uint64_t>(n / p + 1, 1), &ws)) return rc;

    uint32_t* A = ctx->pr_block.as<uint32_t>();
    uint32_t* S = ctx->pr_sorted.as<uint32_t>();
    uint64_t* starts = ctx->pr_counts.as<uint64_t>(); // [p][radix+1]
    int64_t* gd = ctx->pr_delta.as<int64_t>();        // [p][radix]
    uint64_t* send = ctx->pr_misc.as<uint64_t>();     // [p][p]
    uint64_t* coltot = send + pp;                      // [radix]
    uint64_t* dstart = coltot + radix;                 // [radix]
    uint64_t* colchunk = dstart + radix;               // [radix / kDigChunk]
    uint32_t* skew = reinterpret_cast<uint32_t*>(colchunk + 64); // round's skew flag

    const uint64_t max_len = n / p + (n % p ? 1 : 0);
    // r <= 2^8: each worker's whole round is ONE one-sweep pass whose digit
    // bases are the global positions of its block's first key per digit
    // (the same fused round as bsg_pr_fused_round, all blocks local)
    const bool fused = bits == 8 || (bits < 8 && max_len <= kChunkKeys); // 8-bit: 64-bit rows above 2^29
    // fused rounds read the input directly and the last one writes `out`
    // directly; only a single round over overlapping in/out goes through A
    // (r = 2^16: round 0's byte sub-passes read the input, the last round's
    // scatter writes `out`; in place is safe, the scatter runs after every read)
    const bool seg16_0 = !fused && bits == 16;
    const bool direct = (fused && rounds >= 1 &&
                         !(rounds == 1 && static_cast<const void*>(in) < static_cast<const void*>(out + n) &&
                           static_cast<const void*>(out) < static_cast<const void*>(in + n))) ||
                        (seg16_0 && rounds >= 1);
    if (n && !direct && (e = cudaMemcpyAsync(A, in, n * 4, cudaMemcpyDeviceToDevice, stream)) != cudaSuccess)
        return cuda_fail(e, "pr copy in");
    bsg_run_stats st{};
    std::vector<uint64_t> h_send(pp);
    uint64_t launches = 0;
    auto add = [&](int l) -> bool {
        if (l < 0) return false;
        launches += static_cast<uint64_t>(l);
        return true;
    };
    if (fused && (e = ctx->status.ensure(onesweep_seg_status_words(n, p) * sizeof(uint32_t))) != cudaSuccess)
        return cuda_fail(e, "pr workspace");
    uint32_t* cur = A;
    uint32_t* nxt = S;
    for (int round = 0; round < rounds && n && fused; ++round) {
        const int shift = round * bits;
        // round sources and destinations: input -> S -> A -> ... -> out
        const uint32_t* src = (direct && round == 0) ? in : cur;
        uint32_t* dst = (direct && round == rounds - 1) ? out : nxt;
        uint64_t* counts = starts; // [p][radix]
        int64_t* base = gd;        // [p][radix]
        // count_digits of every worker (radix.hpp:127-132), one launch
        if (!add(launch_pr_seg_count(src, n, p, bits, shift, counts, stream)))
            return cuda_fail(cudaGetLastError(), "pr count");
        {
            TimedScope ts(3 /*BSG_K_PR*/, stream);
            const int chunks = (radix + kDigChunk - 1) / kDigChunk;
            if ((e = cudaMemsetAsync(skew, 0, sizeof(uint32_t), stream)) != cudaSuccess)
                return cuda_fail(e, "pr plan");
            pr_plan_col_kernel<<<chunks, kDigChunk, 0, stream>>>(counts, p, radix, base, coltot, colchunk, skew, n);
            pr_digit_start_kernel<<<chunks, kDigChunk, 0, stream>>>(coltot, colchunk, radix, dstart);
            const uint64_t pr = static_cast<uint64_t>(p) * radix;
            pr_add_dstart_kernel<<<static_cast<unsigned>((pr + 255) / 256), 256, 0, stream>>>(base, dstart, p, radix);
            launches += 3;
        }
        // every worker's local stable pass, stored at the global positions
        // (sort_and_scatter + exchange + gather_slices), one segmented launch.
        // A full run whose RunStats are not asked for returns only the sorted
        // array, so its rounds may rank value-stably (radix.cu rank_stage).
        // With RunStats every round is strictly stable: which of two keys
        // equal in the low bits and the digit lands left of a block boundary
        // decides the next round's count matrix, and the message counts must
        // be the reference's.
        if (!add(launch_onesweep_seg(src, dst, n, p, bits, shift, reinterpret_cast<const uint64_t*>(base),
                                     ctx->status.as<uint32_t>(), stream, skew, rounds * bits == 32 && !stats)))
            return cuda_fail(cudaGetLastError(), "pr fused pass");
        if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "pr round");
        if (stats) {
            if ((e = cudaMemsetAsync(send, 0, pp * 8, stream)) != cudaSuccess) return cuda_fail(e, "pr stats");
            pr_send_from_counts_kernel<<<dim3((radix + kSendThreads - 1) / kSendThreads, p), kSendThreads, p * 8,
                                         stream>>>(counts, base, n, p, radix, send);
            ++launches;
            if ((e = cudaMemcpyAsync(h_send.data(), send, pp * 8, cudaMemcpyDeviceToHost, stream)) != cudaSuccess ||
                (e = cudaStreamSynchronize(stream)) != cudaSuccess)
                return cuda_fail(e, "pr stats");
            uint64_t nz = 0;
            for (uint64_t i = 0; i < pp; ++i) nz += h_send[i] ? 1 : 0;
            st.messages_sent += pp + nz;
            st.words_sent += pp * static_cast<uint64_t>(radix) + n;
        }
        std::swap(cur, nxt);
    }
    if (fused) A = cur;
    // r = 2^16: the workers' local passes as segmented byte sub-passes
    const bool seg16 = !fused && bits == 16;
    if (seg16 && (e = ctx->status.ensure(onesweep_seg_status_words(n, p) * sizeof(uint32_t))) != cudaSuccess)
        return cuda_fail(e, "pr workspace");
    for (int round = 0; round < rounds && n && !fused; ++round) {
        const int shift = round * bits;
        // local stable pass of every worker (sort_and_scatter's count_sort_round)
        for (int w = 0; w < p; ++w) {
            const uint64_t off = bsg_partition_offset_of(n, p, w), sz = bsg_partition_size_of(n, p, w);
            if (sz == 0) continue;
            if (seg16) break; // all workers' local passes at once below
            if (bits <= 8) {
                if (!add(launch_count_pass(A + off, S + off, sz, bits, shift, ws, stream, true)))
                    return cuda_fail(cudaGetLastError(), "pr local pass");
            } else {
                uint32_t* mid = ctx->stage_b.as<uint32_t>();
                if (!add(launch_count_pass(A + off, mid, sz, 8, shift, ws, stream, true)) ||
                    !add(launch_count_pass(mid, S + off, sz, 8, shift + 8, ws, stream, true)))
                    return cuda_fail(cudaGetLastError(), "pr local pass");
            }
        }
        if (seg16) {
            // r = 2^16 local pass of every worker as two segmented one-sweep
            // byte sub-passes (each block sorted in place, stably: low byte,
            // then high byte); a block holds the same keys before and after
            // the first sub-pass, so both byte histograms come from A
            uint64_t* cA = starts;
            uint64_t* cB = starts + static_cast<uint64_t>(p) * 256;
            int64_t* bA = gd;
            int64_t* bB = gd + static_cast<uint64_t>(p) * 256;
            uint32_t* mid = ctx->stage_b.as<uint32_t>();
            const uint32_t* src = (direct && round == 0) ? in : A;
            if (!add(launch_pr_seg_count(src, n, p, 8, shift, cA, stream)) ||
                !add(launch_pr_seg_count(src, n, p, 8, shift + 8, cB, stream)))
                return cuda_fail(cudaGetLastError(), "pr local count");
            if ((e = cudaMemsetAsync(skew, 0, 2 * sizeof(uint32_t), stream)) != cudaSuccess)
                return cuda_fail(e, "pr local count");
            pr_local_base_kernel<<<p, 256, 0, stream>>>(cA, n, p, bA, skew);
            pr_local_base_kernel<<<p, 256, 0, stream>>>(cB, n, p, bB, skew + 1);
            launches += 2;
            // full runs: both sub-passes may rank value-stably (a block enters
            // the round ordered by its low `shift` bits, the second sub-pass by
            // its low shift + 8 bits)
            // (without RunStats only: see the r <= 2^8 rounds above)
            const bool full_run = rounds * bits == 32 && !stats;
            if (!add(launch_onesweep_seg(src, mid, n, p, 8, shift, reinterpret_cast<const uint64_t*>(bA),
                                         ctx->status.as<uint32_t>(), stream, skew, full_run)) ||
                !add(launch_onesweep_seg(mid, S, n, p, 8, shift + 8, reinterpret_cast<const uint64_t*>(bB),
                                         ctx->status.as<uint32_t>(), stream, skew + 1, full_run)))
                return cuda_fail(cudaGetLastError(), "pr local pass");
        }
        {
            TimedScope ts(3 /*BSG_K_PR*/, stream);
            // per-worker digit counts (count_digits) as run starts of the sorted blocks
            pr_run_starts_kernel<<<dim3((radix + 1 + 255) / 256, p), 256, 0, stream>>>(S, n, p, shift, mask, radix,
                                                                                      starts);
            // count matrix -> routing (digit_starts + next_pos)
            const int chunks = (radix + kDigChunk - 1) / kDigChunk;
            pr_col_prefix_kernel<<<chunks, kDigChunk, 0, stream>>>(starts, p, radix, gd, coltot, colchunk);
            pr_digit_start_kernel<<<chunks, kDigChunk, 0, stream>>>(coltot, colchunk, radix, dstart);
            // exchange + rebuild of all workers
            const uint64_t want = (max_len + kScatterThreads * kScatterItems - 1) / (kScatterThreads * kScatterItems);
            const unsigned gx = static_cast<unsigned>(std::max<uint64_t>(
                1, std::min<uint64_t>(want, std::max<uint64_t>(1, kSmCountB200 * 8 / static_cast<uint64_t>(p)))));
            uint32_t* rebuilt = (direct && round == rounds - 1) ? out : A;
            pr_scatter_kernel<<<dim3(gx, p), kScatterThreads, 0, stream>>>(S, n, p, shift, mask, radix, dstart, gd,
                                                                          rebuilt);
            launches += 4;
        }
        if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "pr round");
        if (stats) {
            if ((e = cudaMemsetAsync(send, 0, pp * 8, stream)) != cudaSuccess) return cuda_fail(e, "pr stats");
            pr_send_counts_kernel<<<dim3((radix + kSendThreads - 1) / kSendThreads, p), kSendThreads, p * 8, stream>>>(
                starts, dstart, gd, n, p, radix, send);
            ++launches;
            if ((e = cudaMemcpyAsync(h_send.data(), send, pp * 8, cudaMemcpyDeviceToHost, stream)) != cudaSuccess ||
                (e = cudaStreamSynchronize(stream)) != cudaSuccess)
                return cuda_fail(e, "pr stats");
            uint64_t nz = 0;
            for (uint64_t i = 0; i < pp; ++i) nz += h_send[i] ? 1 : 0;
            st.messages_sent += pp + nz;
            st.words_sent += pp * static_cast<uint64_t>(radix) + n;
        }
    }
    if (stats) {
        if (n == 0) {
            // empty input: the count exchange still happens every round
            st.messages_sent = static_cast<uint64_t>(rounds) * pp;
            st.words_sent = static_cast<uint64_t>(rounds) * pp * radix;
        }
        st.supersteps = 2 * rounds + 1;
        st.messages_delivered = st.messages_sent;
        st.words_delivered = st.words_sent;
        *stats = st;
    }
    if (n && !direct && (e = cudaMemcpyAsync(out, A, n * 4, cudaMemcpyDeviceToDevice, stream)) != cudaSuccess)
        return cuda_fail(e, "pr copy out");
    ctx->launches += launches;
    return BSG_OK;
}

} // namespace bsg

// Host restatement of the routing plan (same arithmetic as pr_plan1/2).
extern "C" int bsg_pr_plan_host(const uint64_t* counts, uint64_t n, int p, int me, int radix_log2,
                                uint64_t* send_counts, uint64_t* recv_counts, int64_t* rebuild_delta) {
    using namespace bsg;
    if (p < 1 || me < 0 || me >= p) return fail(BSG_EINVAL, "pr_plan_host: worker index out of range");
    if (radix_log2 != 1 && radix_log2 != 2 && radix_log2 != 4 && radix_log2 != 8 && radix_log2 != 16)
        return fail(BSG_EINVAL, "radix must be a power of two whose bit width divides 32");
    if (!counts || !send_counts || !recv_counts || !rebuild_delta) return fail(BSG_EINVAL, "null pointer");
    const uint64_t r = uint64_t{1} << radix_log2;
    auto ov = [](uint64_t a0, uint64_t a1, uint64_t b0, uint64_t b1) -> uint64_t {
        const uint64_t lo = a0 > b0 ? a0 : b0, hi = a1 < b1 ? a1 : b1;
        return hi > lo ? hi - lo : 0;
    };
    for (int v = 0; v < p; ++v) { // bsp_error: every row sums to its worker's block size
        uint64_t row = 0;
        for (uint64_t d = 0; d < r; ++d) row += counts[static_cast<uint64_t>(v) * r + d];
        if (row != bsg_partition_size_of(n, p, v))
            return fail(BSG_EPROTO, "bsp_error: a worker's exchanged digit counts do not sum to its block size");
    }
    std::vector<uint64_t> starts(r), before(r, 0), split(p);
    uint64_t run = 0;
    for (uint64_t d = 0; d < r; ++d) {
        starts[d] = run;
        for (int u = 0; u < p; ++u) run += counts[static_cast<uint64_t>(u) * r + d];
    }
    const uint64_t lo_me = bsg_partition_offset_of(n, p, me), hi_me = lo_me + bsg_partition_size_of(n, p, me);
    for (int w = 0; w < p; ++w) send_counts[w] = 0;
    for (int v = 0; v < p; ++v) {
        uint64_t local = 0, acc_recv = 0, acc_split = 0;
        for (uint64_t d = 0; d < r; ++d) {
            const uint64_t cv = counts[static_cast<uint64_t>(v) * r + d];
            const uint64_t np = starts[d] + before[d];
            acc_recv += ov(np, np + cv, lo_me, hi_me);
            acc_split += ov(np, np + cv, 0, lo_me);
            rebuild_delta[static_cast<uint64_t>(v) * r + d] = static_cast<int64_t>(np) - static_cast<int64_t>(local);
            if (v == me && cv) {
                const int w0 = bsg_partition_owner_of(n, p, np), w1 = bsg_partition_owner_of(n, p, np + cv - 1);
                for (int w = w0; w <= w1; ++w) {
                    const uint64_t lo = bsg_partition_offset_of(n, p, w);
                    send_counts[w] += ov(np, np + cv, lo, lo + bsg_partition_size_of(n, p, w));
                }
            }
            local += cv;
        }
        recv_counts[v] = acc_recv;
        split[v] = acc_split;
        for (uint64_t d = 0; d < r; ++d) before[d] += counts[static_cast<uint64_t>(v) * r + d];
    }
    uint64_t recv_off = 0;
    for (int v = 0; v < p; ++v) {
        const int64_t adj = static_cast<int64_t>(split[v]) - static_cast<int64_t>(recv_off) - static_cast<int64_t>(lo_me);
        for (uint64_t d = 0; d < r; ++d) rebuild_delta[static_cast<uint64_t>(v) * r + d] += adj;
        recv_off += recv_counts[v];
    }
    return BSG_OK;
}

// Fused exchange + rebuild of one PR round for worker `me` (see bsg.h).
extern "C" int bsg_pr_peer_scatter(bsg_ctx* ctx, const uint32_t* sorted, uint64_t len, const uint64_t* counts_all,
                                   uint64_t n, int p, int me, int round, int radix_log2, uint32_t* const* peer_blocks,
                                   void* stream) {
    using namespace bsg;
    if (!ctx) return fail(BSG_EINVAL, "null context");
    if (radix_log2 != 1 && radix_log2 != 2 && radix_log2 != 4 && radix_log2 != 8 && radix_log2 != 16)
        return fail(BSG_EINVAL, "radix must be a power of two whose bit width divides 32");
    if (p < 1 || p > kPeerMax || me < 0 || me >= p) return fail(BSG_EINVAL, "peer scatter: worker index out of range");
    if (round < 0 || round >= 32 / radix_log2) return fail(BSG_EINVAL, "round out of range");
    if (len != bsg_partition_size_of(n, p, me)) return fail(BSG_EINVAL, "peer scatter: block size != size_of(me)");
    if (!peer_blocks || !counts_all || (len && !sorted)) return fail(BSG_EINVAL, "null pointer");
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceGuard dev(ctx->device);
    TimerBinding bind(&ctx->timer);
    const int radix = 1 << radix_log2;
    const int chunks = (radix + kDigChunk - 1) / kDigChunk;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder order(ctx, st);
    // scratch: before/delta [p][r] (int64), coltot [r], dstart [r], colchunk [chunks], gd [r]
    const uint64_t words = static_cast<uint64_t>(p) * radix + 3ull * radix + chunks;
    cudaError_t e = ctx->pr_delta.ensure(words * 8);
    if (e != cudaSuccess) return cuda_fail(e, "peer scatter workspace");
    int64_t* before = ctx->pr_delta.as<int64_t>();
    uint64_t* coltot = reinterpret_cast<uint64_t*>(before + static_cast<uint64_t>(p) * radix);
    uint64_t* dstart = coltot + radix;
    int64_t* gd = reinterpret_cast<int64_t*>(dstart + radix);
    uint64_t* colchunk = reinterpret_cast<uint64_t*>(gd + radix);
    PeerTable tab{};
    for (int w = 0; w < p; ++w) {
        if (!peer_blocks[w] && bsg_partition_size_of(n, p, w)) return fail(BSG_EINVAL, "peer scatter: null peer block");
        tab.blocks[w] = peer_blocks[w];
        tab.offset[w] = bsg_partition_offset_of(n, p, w);
    }
    tab.offset[p] = n;
    uint32_t* flag = nullptr;
    if (int rc = proto_begin(ctx, st, &flag)) return rc;
    {
        TimedScope ts(3 /*BSG_K_PR*/, st);
        if (check_count_rows(counts_all, p, radix, n, flag, st) < 0) return cuda_fail(cudaGetLastError(), "peer scatter check");
        pr_plan_col_kernel<<<chunks, kDigChunk, 0, st>>>(counts_all, p, radix, before, coltot, colchunk);
        pr_digit_start_kernel<<<chunks, kDigChunk, 0, st>>>(coltot, colchunk, radix, dstart);
        pr_peer_gd_kernel<<<chunks, kDigChunk, 0, st>>>(counts_all + static_cast<uint64_t>(me) * radix,
                                                        before + static_cast<uint64_t>(me) * radix, dstart, radix, gd);
        ctx->launches += 3;
        if (len) {
            const uint64_t want = (len + kScatterThreads * kScatterItems - 1) / (kScatterThreads * kScatterItems);
            const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, kSmCountB200 * 8)));
            pr_peer_scatter_kernel<<<grid, kScatterThreads, 0, st>>>(sorted, len, round * radix_log2,
                                                                     static_cast<uint32_t>(radix - 1), gd, p, tab);
            ctx->launches += 1;
        }
    }
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail(cudaGetLastError(), "peer scatter launch");
    return proto_end(ctx, st, "bsp_error: a worker's exchanged digit counts do not sum to its block size");
}

// A whole PR round fused with its exchange (see bsg.h).
extern "C" int bsg_pr_fused_round(bsg_ctx* ctx, const uint32_t* block, uint64_t len, const uint64_t* counts_all,
                                  uint64_t n, int p, int me, int round, int radix_log2, uint32_t* const* peer_blocks,
                                  void* stream) {
    using namespace bsg;
    if (!ctx) return fail(BSG_EINVAL, "null context");
    if (radix_log2 != 1 && radix_log2 != 2 && radix_log2 != 4 && radix_log2 != 8 && radix_log2 != 16)
        return fail(BSG_EINVAL, "radix must be a power of two whose bit width divides 32");
    if (p < 1 || p > kPeerMax || me < 0 || me >= p) return fail(BSG_EINVAL, "fused round: worker index out of range");
    if (round < 0 || round >= 32 / radix_log2) return fail(BSG_EINVAL, "round out of range");
    if (len != bsg_partition_size_of(n, p, me)) return fail(BSG_EINVAL, "fused round: block size != size_of(me)");
    if (!peer_blocks || !counts_all || (len && !block)) return fail(BSG_EINVAL, "null pointer");
    if (radix_log2 == 16) {
        cudaError_t e;
        {
            std::lock_guard<std::mutex> lock(ctx->mu);
            DeviceGuard dev(ctx->device);
            e = ctx->pr_sorted.ensure(std::max<uint64_t>(len, 4) * 4);
        }
        if (e != cudaSuccess) return cuda_fail(e, "fused round workspace");
        uint32_t* sorted = ctx->pr_sorted.as<uint32_t>();
        if (int rc = bsg_count_sort_round_u32(ctx, block, sorted, len, round, radix_log2, BSG_MEM_DEVICE, stream))
            return rc;
        return bsg_pr_peer_scatter(ctx, sorted, len, counts_all, n, p, me, round, radix_log2, peer_blocks, stream);
    }
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceGuard dev(ctx->device);
    TimerBinding bind(&ctx->timer);
    const int radix = 1 << radix_log2;
    const int chunks = (radix + kDigChunk - 1) / kDigChunk;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder order(ctx, st);
    const uint64_t words = static_cast<uint64_t>(p) * radix + 3ull * radix + chunks + 1; // + skew flag
    cudaError_t e = ctx->pr_delta.ensure(words * 8);
    if (e == cudaSuccess) e = ctx->status.ensure(onesweep_status_words(std::max<uint64_t>(len, 1)) * sizeof(uint32_t));
    if (e != cudaSuccess) return cuda_fail(e, "fused round workspace");
    int64_t* before = ctx->pr_delta.as<int64_t>();
    uint64_t* coltot = reinterpret_cast<uint64_t*>(before + static_cast<uint64_t>(p) * radix);
    uint64_t* dstart = coltot + radix;
    uint64_t* base = dstart + radix;
    uint64_t* colchunk = base + radix;
    uint32_t* skew = reinterpret_cast<uint32_t*>(colchunk + chunks); // heavy-digit flag of this round
    PeerTable tab{};
    for (int w = 0; w < p; ++w) {
        if (!peer_blocks[w] && bsg_partition_size_of(n, p, w)) return fail(BSG_EINVAL, "fused round: null peer block");
        tab.blocks[w] = peer_blocks[w];
        tab.offset[w] = bsg_partition_offset_of(n, p, w);
    }
    tab.offset[p] = n;
    uint32_t* flag = nullptr;
    if (int rc = proto_begin(ctx, st, &flag)) return rc;
    {
        TimedScope ts(3 /*BSG_K_PR*/, st);
        if (check_count_rows(counts_all, p, radix, n, flag, st) < 0) return cuda_fail(cudaGetLastError(), "fused round check");
        if ((e = cudaMemsetAsync(skew, 0, sizeof(uint32_t), st)) != cudaSuccess) return cuda_fail(e, "fused round plan");
        pr_plan_col_kernel<<<chunks, kDigChunk, 0, st>>>(counts_all, p, radix, before, coltot, colchunk, skew, n);
        pr_digit_start_kernel<<<chunks, kDigChunk, 0, st>>>(coltot, colchunk, radix, dstart);
        pr_fused_base_kernel<<<(radix + 255) / 256, 256, 0, st>>>(dstart, before + static_cast<uint64_t>(me) * radix,
                                                                 radix, base);
        ctx->launches += 3;
    }
    const int l = launch_onesweep_peer(block, len, radix_log2, round * radix_log2, base, ctx->status.as<uint32_t>(),
                                       tab, p, st, skew, n);
    if (l < 0) return cuda_fail(cudaGetLastError(), "fused round launch");
    ctx->launches += static_cast<uint64_t>(l) + 1;
    if ((e = cudaPeekAtLastError()) != cudaSuccess) return cuda_fail(cudaGetLastError(), "fused round launch");
    return proto_end(ctx, st, "bsp_error: a worker's exchanged digit counts do not sum to its block size");
}

// ===========================================================================
// Multi-GPU group (one process, G GPUs): bsg_ctx_create_group and
// bsg_pr_group_sort_u32 (include/bsg.h).  Member g owns the worker group
// Partition(p, G) block g, i.e. a contiguous key range; its workers' blocks
// are Partition(len_g, p_g) of that range (the big blocks of Partition(n, p)
// come first), so every in-process segmented kernel applies per member.
// ===========================================================================
namespace bsg {

// NCCL is resolved at run time (dlopen), so libbsg.so loads without it and a
// process that already holds libnccl.so.2 (torch) shares that one copy.
struct NcclApi {
    decltype(&ncclCommInitAll) commInitAll = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGetErrorString) errStr = nullptr;
    bool ok = false;
    std::string why;
};

static NcclApi& nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return a;
        }
        a.commInitAll = reinterpret_cast<decltype(a.commInitAll)>(dlsym(h, "ncclCommInitAll"));
        a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.groupStart = reinterpret_cast<decltype(a.groupStart)>(dlsym(h, "ncclGroupStart"));
        a.groupEnd = reinterpret_cast<decltype(a.groupEnd)>(dlsym(h, "ncclGroupEnd"));
        a.send = reinterpret_cast<decltype(a.send)>(dlsym(h, "ncclSend"));
        a.recv = reinterpret_cast<decltype(a.recv)>(dlsym(h, "ncclRecv"));
        a.errStr = reinterpret_cast<decltype(a.errStr)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.commInitAll && a.commDestroy && a.groupStart && a.groupEnd && a.send && a.recv && a.errStr;
        if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
        return a;
    }();
    return api;
}

struct NcclGroup {
    std::vector<ncclComm_t> comms;
};

static int nccl_fail(ncclResult_t r, const char* what) {
    const NcclApi& a = nccl_api();
    return fail(BSG_ENCCL, std::string(what) + ": " + (a.errStr ? a.errStr(r) : "nccl error"));
}

void destroy_group_nccl(bsg_ctx* grp) {
    auto* ng = static_cast<NcclGroup*>(grp->nccl);
    if (!ng) return;
    if (nccl_api().ok)
        for (ncclComm_t c : ng->comms)
            if (c) nccl_api().commDestroy(c);
    delete ng;
    grp->nccl = nullptr;
}

// Host restatement of the routing for RunStats / remote-byte accounting:
// slice[v][w] = keys of worker v landing in worker w's partition (the
// messages of sort_and_scatter, radix.hpp:151-179), from the p x r matrix.
static void host_slices(const std::vector<uint64_t>& cnt, uint64_t n, int p, int radix,
                        std::vector<uint64_t>& slice) {
    slice.assign(static_cast<size_t>(p) * p, 0);
    std::vector<uint64_t> dstart(radix), before(radix, 0);
    uint64_t run = 0;
    for (int d = 0; d < radix; ++d) {
        dstart[d] = run;
        for (int v = 0; v < p; ++v) run += cnt[static_cast<size_t>(v) * radix + d];
    }
    for (int v = 0; v < p; ++v)
        for (int d = 0; d < radix; ++d) {
            const uint64_t c = cnt[static_cast<size_t>(v) * radix + d];
            if (!c) continue;
            const uint64_t np = dstart[d] + before[d];
            before[d] += c;
            int w = bsg_partition_owner_of(n, p, np);
            uint64_t pos = np, end = np + c;
            while (pos < end) {
                const uint64_t hi = bsg_partition_offset_of(n, p, w) + bsg_partition_size_of(n, p, w);
                const uint64_t take = std::min(end, hi) - pos;
                slice[static_cast<size_t>(v) * p + w] += take;
                pos += take;
                ++w;
            }
        }
}

struct GroupMember {
    bsg_ctx* c = nullptr;
    cudaStream_t s = nullptr;
    int wlo = 0, pw = 0;       // workers [wlo, wlo + pw)
    uint64_t off = 0, len = 0; // key range
    uint32_t* cur = nullptr;
    uint32_t* nxt = nullptr;
    cudaEvent_t ev = nullptr;
    cudaEvent_t t[6] = {};
};

uint64_t group_range_offset(uint64_t n, int p, int G, int g) {
    const int wlo = static_cast<int>(bsg_partition_offset_of(static_cast<uint64_t>(p), G, g));
    return bsg_partition_offset_of(n, p, wlo);
}

int run_parallel_radix_group(bsg_ctx* grp, uint32_t* const* blocks, uint64_t n, int p, int bits, int rounds,
                             int variant, bsg_run_stats* stats, bsg_pr_timing* timing) {
    const int G = static_cast<int>(grp->members.size());
    if (G < 1) return fail(BSG_EINVAL, "not a group context");
    if (G > kPeerMax) return fail(BSG_EINVAL, "group: at most 64 members");
    if (p > kMaxP) return fail(BSG_EINVAL, "parallel radix sort: p must be <= 1024");
    if (variant != BSG_PR_PEER && variant != BSG_PR_NCCL) return fail(BSG_EINVAL, "group sort: unknown variant");
    if (variant == BSG_PR_PEER && !grp->peer_ok)
        return fail(BSG_ECUDA, "group sort: member GPUs lack peer access (use BSG_PR_NCCL)");
    if (variant == BSG_PR_NCCL && p != G) return fail(BSG_EINVAL, "group sort: BSG_PR_NCCL needs p == group size");
    const int radix = 1 << bits;
    const uint32_t mask = static_cast<uint32_t>(radix - 1);
    const uint64_t pp = static_cast<uint64_t>(p) * p;
    std::vector<GroupMember> M(G);
    cudaError_t e;
    for (int g = 0; g < G; ++g) {
        GroupMember& m = M[g];
        m.c = grp->members[g];
        m.s = grp->member_streams[g];
        m.wlo = static_cast<int>(bsg_partition_offset_of(static_cast<uint64_t>(p), G, g));
        m.pw = static_cast<int>(bsg_partition_size_of(static_cast<uint64_t>(p), G, g));
        m.off = bsg_partition_offset_of(n, p, m.wlo);
        m.len = bsg_partition_offset_of(n, p, m.wlo + m.pw) - m.off;
        m.cur = blocks[g];
        if (m.len && !m.cur) return fail(BSG_EINVAL, "group sort: null member block");
    }
    // workspace + events per member
    for (GroupMember& m : M) {
        DeviceGuard dg(m.c->device);
        bsg_ctx* c = m.c;
        const uint64_t L = std::max<uint64_t>(m.len, 4);
        if ((e = c->pr_block.ensure(L * 4)) != cudaSuccess) return cuda_fail(e, "group workspace");
        if ((e = c->pr_counts.ensure(static_cast<uint64_t>(p) * (radix + 1) * 8)) != cudaSuccess)
            return cuda_fail(e, "group workspace");
        if ((e = c->pr_delta.ensure(static_cast<uint64_t>(p) * radix * 8)) != cudaSuccess)
            return cuda_fail(e, "group workspace");
        if ((e = c->pr_misc.ensure(static_cast<uint64_t>(radix) * 16 + 128 * 8 + pp * 8 + 64)) != cudaSuccess)
            return cuda_fail(e, "group workspace");
        if ((e = c->status.ensure(onesweep_seg_status_words(L, std::max(m.pw, 1)) * sizeof(uint32_t))) != cudaSuccess)
            return cuda_fail(e, "group workspace");
        if (bits == 16 || variant == BSG_PR_NCCL) {
            if ((e = c->pr_sorted.ensure(L * 4)) != cudaSuccess) return cuda_fail(e, "group workspace");
            if ((e = c->stage_b.ensure(L * 4)) != cudaSuccess) return cuda_fail(e, "group workspace");
            const uint64_t chunks = (static_cast<uint64_t>(radix) + 1023) / 1024;
            const uint64_t plan_words = static_cast<uint64_t>(p) * (1 + chunks) + 2ull * radix + chunks;
            if ((e = c->pr_recv.ensure(std::max<uint64_t>(4ull * std::max(m.pw, 1) * 256 + 64, plan_words) * 8)) != cudaSuccess)
                return cuda_fail(e, "group workspace");
        }
        m.nxt = c->pr_block.as<uint32_t>();
        if ((e = cudaEventCreateWithFlags(&m.ev, cudaEventDisableTiming)) != cudaSuccess)
            return cuda_fail(e, "group events");
        if (timing)
            for (auto& t : m.t)
                if ((e = cudaEventCreate(&t)) != cudaSuccess) return cuda_fail(e, "group events");
    }
    struct EvFree {
        std::vector<GroupMember>& M;
        ~EvFree() {
            for (auto& m : M) {
                DeviceGuard dg(m.c->device);
                if (m.ev) cudaEventDestroy(m.ev);
                for (auto& t : m.t)
                    if (t) cudaEventDestroy(t);
            }
        }
    } evfree{M};
    auto all_wait_all = [&]() -> int {
        for (auto& m : M) {
            DeviceGuard dg(m.c->device);
            if ((e = cudaEventRecord(m.ev, m.s)) != cudaSuccess) return cuda_fail(e, "group barrier");
        }
        for (auto& m : M) {
            DeviceGuard dg(m.c->device);
            for (auto& o : M)
                if (&o != &m && (e = cudaStreamWaitEvent(m.s, o.ev, 0)) != cudaSuccess)
                    return cuda_fail(e, "group barrier");
        }
        return BSG_OK;
    };
    auto mark = [&](int k) {
        if (!timing) return;
        for (auto& m : M) {
            DeviceGuard dg(m.c->device);
            cudaEventRecord(m.t[k], m.s);
        }
    };
    // per-phase accumulation (ms, max over members per phase per round)
    double t_count = 0, t_exch = 0, t_local = 0;
    uint64_t remote = 0;
    auto phase_ms = [&](int a, int b) -> double {
        double mx = 0;
        for (auto& m : M) {
            DeviceGuard dg(m.c->device);
            cudaEventSynchronize(m.t[b]);
            float f = 0;
            cudaEventElapsedTime(&f, m.t[a], m.t[b]);
            mx = std::max(mx, static_cast<double>(f));
        }
        return mx;
    };
    // the caller's work on member streams is ordered by the synchronous call
    if (int rc = all_wait_all()) return rc;
    cudaEvent_t t_begin[kPeerMax] = {}, t_end[kPeerMax] = {};
    if (timing)
        for (int g = 0; g < G; ++g) {
            DeviceGuard dg(M[g].c->device);
            cudaEventCreate(&t_begin[g]);
            cudaEventCreate(&t_end[g]);
            cudaEventRecord(t_begin[g], M[g].s);
        }
    bsg_run_stats st{};
    std::vector<uint64_t> h_cnt, h_slice;
    uint64_t launches = 0;
    auto add = [&](int l) -> bool {
        if (l < 0) return false;
        launches += static_cast<uint64_t>(l);
        return true;
    };
    // pull the other members' rows of a [p][row] uint64 table into every member's copy
    auto exchange_rows = [&](auto table_of, uint64_t row) -> int {
        if (int rc = all_wait_all()) return rc;
        for (auto& m : M) {
            DeviceGuard dg(m.c->device);
            for (auto& o : M) {
                if (&o == &m || o.pw == 0) continue;
                const uint64_t b = static_cast<uint64_t>(o.pw) * row * 8;
                if ((e = cudaMemcpyAsync(table_of(m) + static_cast<uint64_t>(o.wlo) * row,
                                         table_of(o) + static_cast<uint64_t>(o.wlo) * row, b, cudaMemcpyDefault, m.s)) !=
                    cudaSuccess)
                    return cuda_fail(e, "group count exchange");
            }
        }
        return BSG_OK;
    };
    auto counts_of = [](GroupMember& m) { return m.c->pr_counts.as<uint64_t>(); };
    PeerTable tab{};
    for (int g = 0; g < G; ++g) tab.offset[g] = M[g].off;
    tab.offset[G] = n;
    NcclApi& api = nccl_api();
    if (variant == BSG_PR_NCCL && n) {
        if (!api.ok) return fail(BSG_ENCCL, "BSG_PR_NCCL: " + api.why);
        if (!grp->nccl) {
            auto* ng = new NcclGroup();
            ng->comms.resize(G);
            std::vector<int> devs(G);
            for (int g = 0; g < G; ++g) devs[g] = M[g].c->device;
            ncclResult_t r = api.commInitAll(ng->comms.data(), G, devs.data());
            if (r != ncclSuccess) {
                delete ng;
                return nccl_fail(r, "ncclCommInitAll");
            }
            grp->nccl = ng;
        }
    }
    for (int round = 0; round < rounds && n; ++round) {
        const int shift = round * bits;
        mark(0);
        if (variant == BSG_PR_PEER) {
            if (bits <= 8) {
                // count_digits of every local worker (radix.hpp:127-132), then the
                // count-matrix exchange (the reference's send-to-all of counts)
                for (auto& m : M) {
                    DeviceGuard dg(m.c->device);
                    TimerBinding tb(&m.c->timer);
                    if (m.pw && !add(launch_pr_seg_count(m.cur, m.len, m.pw, bits, shift,
                                                         counts_of(m) + static_cast<uint64_t>(m.wlo) * radix, m.s)))
                        return cuda_fail(cudaGetLastError(), "group count");
                }
                if (int rc = exchange_rows(counts_of, radix)) return rc;
                mark(1);
                for (auto& m : M) {
                    DeviceGuard dg(m.c->device);
                    TimerBinding tb(&m.c->timer);
                    uint64_t* counts = counts_of(m);
                    int64_t* base = m.c->pr_delta.as<int64_t>();
                    uint64_t* coltot = m.c->pr_misc.as<uint64_t>();
                    uint64_t* dstart = coltot + radix;
                    uint64_t* colchunk = dstart + radix;
                    uint32_t* skew = reinterpret_cast<uint32_t*>(colchunk + 64);
                    const int chunks = (radix + kDigChunk - 1) / kDigChunk;
                    if ((e = cudaMemsetAsync(skew, 0, sizeof(uint32_t), m.s)) != cudaSuccess) return cuda_fail(e, "group plan");
                    pr_plan_col_kernel<<<chunks, kDigChunk, 0, m.s>>>(counts, p, radix, base, coltot, colchunk, skew, n);
                    pr_digit_start_kernel<<<chunks, kDigChunk, 0, m.s>>>(coltot, colchunk, radix, dstart);
                    const uint64_t pr = static_cast<uint64_t>(p) * radix;
                    pr_add_dstart_kernel<<<static_cast<unsigned>((pr + 255) / 256), 256, 0, m.s>>>(base, dstart, p, radix);
                    launches += 3;
                    PeerTable t = tab;
                    for (int g = 0; g < G; ++g) t.blocks[g] = M[g].nxt;
                    // the whole round of every local worker as ONE pass: keys
                    // stored at their global positions in the owners' buffers
                    if (m.pw && !add(launch_onesweep_seg_peer(
                                    m.cur, m.len, m.pw, bits, shift,
                                    reinterpret_cast<const uint64_t*>(base) + static_cast<uint64_t>(m.wlo) * radix,
                                    m.c->status.as<uint32_t>(), m.s, skew, t, G, n)))
                        return cuda_fail(cudaGetLastError(), "group fused pass");
                }
            } else {
                // r = 2^16: local pass of every worker (two segmented byte
                // sub-passes, segment-local bases), run starts, starts exchange,
                // then one peer scatter to the global positions
                for (auto& m : M) {
                    if (!m.pw) continue;
                    DeviceGuard dg(m.c->device);
                    TimerBinding tb(&m.c->timer);
                    uint64_t* scratch = m.c->pr_recv.as<uint64_t>();
                    uint64_t* cA = scratch;
                    uint64_t* cB = cA + static_cast<uint64_t>(m.pw) * 256;
                    int64_t* bA = reinterpret_cast<int64_t*>(cB + static_cast<uint64_t>(m.pw) * 256);
                    int64_t* bB = bA + static_cast<uint64_t>(m.pw) * 256;
                    uint32_t* skew = reinterpret_cast<uint32_t*>(bB + static_cast<uint64_t>(m.pw) * 256);
                    uint32_t* mid = m.c->stage_b.as<uint32_t>();
                    uint32_t* S = m.c->pr_sorted.as<uint32_t>();
                    if (!add(launch_pr_seg_count(m.cur, m.len, m.pw, 8, shift, cA, m.s)) ||
                        !add(launch_pr_seg_count(m.cur, m.len, m.pw, 8, shift + 8, cB, m.s)))
                        return cuda_fail(cudaGetLastError(), "group local count");
                    if ((e = cudaMemsetAsync(skew, 0, 2 * sizeof(uint32_t), m.s)) != cudaSuccess)
                        return cuda_fail(e, "group local count");
                    pr_local_base_kernel<<<m.pw, 256, 0, m.s>>>(cA, m.len, m.pw, bA, skew);
                    pr_local_base_kernel<<<m.pw, 256, 0, m.s>>>(cB, m.len, m.pw, bB, skew + 1);
                    launches += 2;
                    if (!add(launch_onesweep_seg(m.cur, mid, m.len, m.pw, 8, shift, reinterpret_cast<const uint64_t*>(bA),
                                                 m.c->status.as<uint32_t>(), m.s, skew)) ||
                        !add(launch_onesweep_seg(mid, S, m.len, m.pw, 8, shift + 8, reinterpret_cast<const uint64_t*>(bB),
                                                 m.c->status.as<uint32_t>(), m.s, skew + 1)))
                        return cuda_fail(cudaGetLastError(), "group local pass");
                    pr_run_starts_kernel<<<dim3((radix + 1 + 255) / 256, m.pw), 256, 0, m.s>>>(
                        S, m.len, m.pw, shift, mask, radix, counts_of(m) + static_cast<uint64_t>(m.wlo) * (radix + 1));
                    ++launches;
                }
                if (int rc = exchange_rows(counts_of, static_cast<uint64_t>(radix) + 1)) return rc;
                mark(1);
                for (auto& m : M) {
                    DeviceGuard dg(m.c->device);
                    TimerBinding tb(&m.c->timer);
                    int64_t* gd = m.c->pr_delta.as<int64_t>();
                    uint64_t* coltot = m.c->pr_misc.as<uint64_t>();
                    uint64_t* dstart = coltot + radix;
                    uint64_t* colchunk = dstart + radix;
                    const int chunks = (radix + kDigChunk - 1) / kDigChunk;
                    pr_col_prefix_kernel<<<chunks, kDigChunk, 0, m.s>>>(counts_of(m), p, radix, gd, coltot, colchunk);
                    pr_digit_start_kernel<<<chunks, kDigChunk, 0, m.s>>>(coltot, colchunk, radix, dstart);
                    launches += 2;
                    if (!m.pw) continue;
                    PeerTable t = tab;
                    for (int g = 0; g < G; ++g) t.blocks[g] = M[g].nxt;
                    const uint64_t max_len = m.len / m.pw + 1;
                    const uint64_t want = (max_len + kScatterThreads * kScatterItems - 1) / (kScatterThreads * kScatterItems);
                    const unsigned gx = static_cast<unsigned>(std::max<uint64_t>(
                        1, std::min<uint64_t>(want, std::max<uint64_t>(1, kSmCountB200 * 8 / static_cast<uint64_t>(m.pw)))));
                    pr_scatter_peer_kernel<<<dim3(gx, m.pw), kScatterThreads, 0, m.s>>>(
                        m.c->pr_sorted.as<uint32_t>(), m.len, m.pw, m.wlo, shift, mask, radix, dstart, gd, t, G);
                    ++launches;
                }
            }
            mark(2);
            if (int rc = all_wait_all()) return rc; // every owner's next block is complete
            for (auto& m : M) std::swap(m.cur, m.nxt);
            if (timing) {
                t_count += phase_ms(0, 1);
                t_exch += phase_ms(1, 2);
            }
        } else {
            // ---- BSG_PR_NCCL: p == G, member g = worker g ----
            std::vector<uint64_t> h_send(pp), h_recv(pp);
            for (auto& m : M) {
                DeviceGuard dg(m.c->device);
                TimerBinding tb(&m.c->timer);
                uint64_t* counts = counts_of(m);
                if (!add(launch_pr_count(m.c, m.cur, m.len, round, bits, counts + static_cast<uint64_t>(m.wlo) * radix, m.s)))
                    return cuda_fail(cudaGetLastError(), "group count");
            }
            if (int rc = exchange_rows(counts_of, radix)) return rc;
            mark(1);
            for (int g = 0; g < G; ++g) {
                GroupMember& m = M[g];
                DeviceGuard dg(m.c->device);
                TimerBinding tb(&m.c->timer);
                uint64_t* scratch = m.c->pr_recv.as<uint64_t>();
                uint64_t* send = m.c->pr_misc.as<uint64_t>() + 2 * radix + 128; // [p]
                uint64_t* recv = send + p;                                         // [p]
                if ((e = cudaMemsetAsync(send, 0, 2ull * p * 8, m.s)) != cudaSuccess) return cuda_fail(e, "group plan");
                const int l = launch_pr_plan(counts_of(m), n, p, g, bits, send, recv, m.c->pr_delta.as<int64_t>(), m.s,
                                             scratch);
                if (!add(l)) return cuda_fail(cudaGetLastError(), "group plan");
                // local stable pass of sort_and_scatter (radix.hpp:151-179)
                RadixWorkspace ws;
                if (int rc = m.c->radix_ws(std::max<uint64_t>(m.len, 1), &ws)) return rc;
                uint32_t* S = m.c->pr_sorted.as<uint32_t>();
                if (m.len) {
                    if (bits <= 8) {
                        if (!add(launch_count_pass(m.cur, S, m.len, bits, shift, ws, m.s, true)))
                            return cuda_fail(cudaGetLastError(), "group local pass");
                    } else {
                        uint32_t* mid = m.c->stage_b.as<uint32_t>();
                        if (!add(launch_count_pass(m.cur, mid, m.len, 8, shift, ws, m.s, true)) ||
                            !add(launch_count_pass(mid, S, m.len, 8, shift + 8, ws, m.s, true)))
                            return cuda_fail(cudaGetLastError(), "group local pass");
                    }
                }
                if ((e = cudaMemcpyAsync(h_send.data() + static_cast<uint64_t>(g) * p, send, p * 8, cudaMemcpyDeviceToHost,
                                         m.s)) != cudaSuccess ||
                    (e = cudaMemcpyAsync(h_recv.data() + static_cast<uint64_t>(g) * p, recv, p * 8, cudaMemcpyDeviceToHost,
                                         m.s)) != cudaSuccess)
                    return cuda_fail(e, "group plan");
            }
            for (auto& m : M) {
                DeviceGuard dg(m.c->device);
                if ((e = cudaStreamSynchronize(m.s)) != cudaSuccess) return cuda_fail(e, "group plan");
            }
            // bsp_error checks of gather_slices (radix.hpp:207-220, 283-286)
            for (int g = 0; g < G; ++g) {
                uint64_t in_sum = 0, out_sum = 0;
                for (int h = 0; h < G; ++h) {
                    in_sum += h_recv[static_cast<uint64_t>(g) * p + h];
                    out_sum += h_send[static_cast<uint64_t>(g) * p + h];
                    if (h_send[static_cast<uint64_t>(g) * p + h] != h_recv[static_cast<uint64_t>(h) * p + g])
                        return fail(BSG_EPROTO, "bsp_error: send/receive counts disagree between workers");
                }
                if (in_sum != M[g].len || out_sum != M[g].len)
                    return fail(BSG_EPROTO, "bsp_error: received slices do not fill the worker's partition");
            }
            mark(2);
            // all-to-all-v of the contiguous slices over NCCL
            auto* ng = static_cast<NcclGroup*>(grp->nccl);
            ncclResult_t r = api.groupStart();
            if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
            for (int g = 0; g < G; ++g) {
                GroupMember& m = M[g];
                const uint32_t* S = m.c->pr_sorted.as<uint32_t>();
                uint32_t* R = m.c->stage_b.as<uint32_t>();
                uint64_t so = 0, ro = 0;
                for (int h = 0; h < G; ++h) {
                    const uint64_t sc = h_send[static_cast<uint64_t>(g) * p + h];
                    const uint64_t rc = h_recv[static_cast<uint64_t>(g) * p + h];
                    if (h != g) remote += sc * 4;
                    if (sc && (r = api.send(S + so, sc, ncclUint32, h, ng->comms[g], m.s)) != ncclSuccess) {
                        api.groupEnd();
                        return nccl_fail(r, "ncclSend");
                    }
                    if (rc && (r = api.recv(R + ro, rc, ncclUint32, h, ng->comms[g], m.s)) != ncclSuccess) {
                        api.groupEnd();
                        return nccl_fail(r, "ncclRecv");
                    }
                    so += sc;
                    ro += rc;
                }
            }
            if ((r = api.groupEnd()) != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
            mark(3);
            // gather_slices: stable digit scatter of the source-major buffer
            for (int g = 0; g < G; ++g) {
                GroupMember& m = M[g];
                DeviceGuard dg(m.c->device);
                TimerBinding tb(&m.c->timer);
                uint64_t* recv = m.c->pr_misc.as<uint64_t>() + 2 * radix + 128 + p;
                if (!add(launch_pr_rebuild(m.c->stage_b.as<uint32_t>(), m.len, bits, shift, m.c->pr_delta.as<int64_t>(),
                                           m.cur, m.s, recv, p, nullptr)))
                    return cuda_fail(cudaGetLastError(), "group rebuild");
            }
            mark(4);
            if (timing) {
                t_count += phase_ms(0, 1);
                t_local += phase_ms(1, 2) + phase_ms(3, 4);
                t_exch += phase_ms(2, 3);
            }
        }
        if (stats || (timing && variant == BSG_PR_PEER)) {
            // RunStats (and the remote bytes of the peer rounds) from member
            // 0's copy of this round's count matrix
            GroupMember& m0 = M[0];
            DeviceGuard dg(m0.c->device);
            const uint64_t row = (variant == BSG_PR_PEER && bits == 16) ? radix + 1 : radix;
            std::vector<uint64_t> raw(static_cast<size_t>(p) * row);
            if ((e = cudaMemcpyAsync(raw.data(), counts_of(m0), raw.size() * 8, cudaMemcpyDeviceToHost, m0.s)) != cudaSuccess ||
                (e = cudaStreamSynchronize(m0.s)) != cudaSuccess)
                return cuda_fail(e, "group stats");
            h_cnt.assign(static_cast<size_t>(p) * radix, 0);
            for (int v = 0; v < p; ++v)
                for (int d = 0; d < radix; ++d)
                    h_cnt[static_cast<size_t>(v) * radix + d] =
                        row == static_cast<uint64_t>(radix) ? raw[static_cast<size_t>(v) * row + d]
                                                            : raw[static_cast<size_t>(v) * row + d + 1] -
                                                                  raw[static_cast<size_t>(v) * row + d];
            host_slices(h_cnt, n, p, radix, h_slice);
            uint64_t nz = 0;
            for (uint64_t i = 0; i < pp; ++i) nz += h_slice[i] ? 1 : 0;
            st.messages_sent += pp + nz;
            st.words_sent += pp * static_cast<uint64_t>(radix) + n;
            if (variant == BSG_PR_PEER)
                for (int v = 0; v < p; ++v)
                    for (int w = 0; w < p; ++w) {
                        const int gv = static_cast<int>(std::upper_bound(M.begin(), M.end(), v, [](int x, const GroupMember& m) {
                                           return x < m.wlo + m.pw;
                                       }) - M.begin());
                        const int gw = static_cast<int>(std::upper_bound(M.begin(), M.end(), w, [](int x, const GroupMember& m) {
                                           return x < m.wlo + m.pw;
                                       }) - M.begin());
                        if (gv != gw) remote += h_slice[static_cast<size_t>(v) * p + w] * 4;
                    }
        }
    }
    // results back into the callers' blocks
    for (auto& m : M) {
        DeviceGuard dg(m.c->device);
        if (m.len && m.cur != blocks[&m - M.data()] &&
            (e = cudaMemcpyAsync(blocks[&m - M.data()], m.cur, m.len * 4, cudaMemcpyDeviceToDevice, m.s)) != cudaSuccess)
            return cuda_fail(e, "group copy out");
    }
    if (timing)
        for (int g = 0; g < G; ++g) {
            DeviceGuard dg(M[g].c->device);
            cudaEventRecord(t_end[g], M[g].s);
        }
    for (auto& m : M) {
        DeviceGuard dg(m.c->device);
        if ((e = cudaStreamSynchronize(m.s)) != cudaSuccess) return cuda_fail(e, "group sort");
    }
    grp->launches += launches;
    if (timing) {
        double tot = 0;
        for (int g = 0; g < G; ++g) {
            DeviceGuard dg(M[g].c->device);
            float f = 0;
            cudaEventElapsedTime(&f, t_begin[g], t_end[g]);
            tot = std::max(tot, static_cast<double>(f));
            cudaEventDestroy(t_begin[g]);
            cudaEventDestroy(t_end[g]);
        }
        timing->total_ms = tot;
        timing->count_ms = t_count;
        timing->exchange_ms = t_exch;
        timing->local_ms = t_local;
        timing->remote_bytes = remote;
    }
    if (stats) {
        if (n == 0) {
            st.messages_sent = static_cast<uint64_t>(rounds) * pp;
            st.words_sent = static_cast<uint64_t>(rounds) * pp * radix;
        }
        st.supersteps = 2 * rounds + 1;
        st.messages_delivered = st.messages_sent;
        st.words_delivered = st.words_sent;
        *stats = st;
    }
    return BSG_OK;
}

} // namespace bsg

extern "C" uint64_t bsg_group_range_offset(uint64_t n, int p, int G, int g) {
    if (p < 1 || G < 1 || g < 0) return 0;
    if (g >= G) return n;
    return bsg::group_range_offset(n, p, G, g);
}
extern "C" uint64_t bsg_group_range_size(uint64_t n, int p, int G, int g) {
    if (p < 1 || G < 1 || g < 0 || g >= G) return 0;
    return bsg::group_range_offset(n, p, G, g + 1) - bsg::group_range_offset(n, p, G, g);
}

extern "C" int bsg_pr_group_sort_u32(bsg_ctx* grp, uint32_t* const* blocks, uint64_t n, int p, int radix_log2,
                                     int rounds_limit, int variant, bsg_run_stats* stats, bsg_pr_timing* timing,
                                     void* const* streams) {
    using namespace bsg;
    if (!grp) return fail(BSG_EINVAL, "null context");
    if (grp->members.empty()) return fail(BSG_EINVAL, "bsg_pr_group_sort_u32 needs a group context (bsg_ctx_create_group)");
    if (p < 1) return fail(BSG_EINVAL, "parallel radix sort: p must be >= 1");
    if (radix_log2 != 1 && radix_log2 != 2 && radix_log2 != 4 && radix_log2 != 8 && radix_log2 != 16)
        return fail(BSG_EINVAL, "radix must be a power of two whose bit width divides 32");
    if (n && !blocks) return fail(BSG_EINVAL, "null block table");
    const int all_rounds = 32 / radix_log2;
    const int rounds = (rounds_limit >= 0 && rounds_limit < all_rounds) ? rounds_limit : all_rounds;
    std::lock_guard<std::mutex> lock(grp->mu);
    // order the callers' work on the blocks before the members' streams
    const int G = static_cast<int>(grp->members.size());
    for (int g = 0; g < G; ++g) {
        DeviceGuard dg(grp->members[g]->device);
        cudaError_t e;
        if (streams) {
            cudaEvent_t ev;
            if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess ||
                (e = cudaEventRecord(ev, static_cast<cudaStream_t>(streams[g]))) != cudaSuccess ||
                (e = cudaStreamWaitEvent(grp->member_streams[g], ev, 0)) != cudaSuccess)
                return cuda_fail(e, "group sort: caller stream ordering");
            cudaEventDestroy(ev);
        } else if ((e = cudaDeviceSynchronize()) != cudaSuccess) {
            return cuda_fail(e, "group sort: device synchronize");
        }
    }
    return run_parallel_radix_group(grp, blocks, n, p, radix_log2, rounds, variant, stats, timing);
}
