// radix.cu -- stable LSD radix sort of uint32 keys for sm_100a.
//
// Restates the count-sort round of radix.hpp:44-65 (histogram, exclusive
// scan, stable forward scatter) and serial_radix_sort (radix.hpp:69-90) as
// three kernels:
//   K1 hist_kernel      -- one read of the keys (16-byte loads), per-CTA
//                          shared-memory histograms of every digit with a
//                          private copy of every counter per lane (no bank
//                          conflicts for uniform and all-equal keys alike),
//                          reduced into per-chunk global bins.
//   K2 scan_plan_kernel -- exclusive digit scans -> per-chunk output bases, and
//                          a device-resident PassPlan that skips identity
//                          passes (one digit value holds all n keys) and picks
//                          the ping-pong buffers so the result lands in `out`
//                          with no host round trip.
//   K3 onesweep_kernel  -- one stable pass over persistent CTAs: TMA bulk
//                          load of a 12288-key tile into shared memory (double
//                          buffered), per-warp digit counts, early publication
//                          of the tile aggregate, decoupled look-back across
//                          tiles per digit, warp-striped stable ranking by a
//                          bit-serial ballot multisplit straight into the
//                          staged tile (original order inside a warp =
//                          item-major, lane-minor), digit runs written out
//                          coalesced.
// Inside a FULL keys-only sort, whose intermediate states nobody sees:
//   K3f first_pass_kernel -- pass 0: no order inside a digit run (shared-memory
//                          cursors per lane quad, global run reservations, no
//                          ballots, no look-back);
//   K3r onesweep_kernel<...,4> -- passes over long runs of equal low bits:
//                          value-stable ranking by one shared-memory atomic
//                          per key, ballots only where a warp item straddles
//                          a run boundary (rank_stage).
// All counts/positions are 64-bit at the chunk level (a chunk is <= 2^29
// keys so the 30-bit look-back payload never overflows).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "radix.cuh"
#include "timer.cuh"

#ifndef BSG_LB_WIN
#define BSG_LB_WIN 12
#endif
#ifndef BSG_CLAIM_AT
#define BSG_CLAIM_AT 0 // where a one-sweep CTA claims its next tile: 0 loop top, 1 after staging, 2 after look-back
#endif
#ifndef BSG_OS_DBG_MASK
#define BSG_OS_DBG_MASK 0 // development builds: -DBSG_OS_DBG_MASK=31 enables the BSG_OS_DBG timing switches
#endif
#ifndef BSG_SCAN_NBAR
#define BSG_SCAN_NBAR 1 // named barrier among the scan warps instead of a CTA barrier (-0.6%)
#endif
#ifndef BSG_COUNT_FAST
#define BSG_COUNT_FAST 1 // byte-digit counting: LOP3 row offset + IMAD increment (7 instead of 9 per key)
#endif
#ifndef BSG_LB_FAST
#define BSG_LB_FAST 1 // look-back rounds whose words are all published aggregates take a branch-free sum
#endif
#ifndef BSG_RANGE_CACHE
#define BSG_RANGE_CACHE 1 // every pass: the claiming thread computes a tile's range once (shared memory)
#endif
#ifndef BSG_HIST_LOADS
#define BSG_HIST_LOADS 4 // 16-byte loads in flight per thread in the histogram kernel (2 or 4)
#endif
#ifndef BSG_EARLY_WIDE
#define BSG_EARLY_WIDE 1 // the early count also in the segmented (PR) and 64-bit-row passes
#endif
#ifndef BSG_EARLY_COUNT
#define BSG_EARLY_COUNT 2 // count-then-rank: the upper half of the warps counts the next tile during the
                          // look-back (1: their own keys, 2: all keys)
#endif
#ifndef BSG_LB_FIRST
#define BSG_LB_FIRST 0 // wider first look-back round (predecessors), 0 = same as the window
#endif
#ifndef BSG_LB_WIN_SMALL
#define BSG_LB_WIN_SMALL 4
#endif
namespace bsg {

namespace {

constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kValMask = (1u << 30) - 1;

// Look-back status word: 2-bit flag (aggregate / inclusive) + count.  32-bit
// words (30-bit counts) while a pass covers <= 2^29 keys; 64-bit words
// (62-bit counts) above, so one pass is always one look-back domain.
template <bool WIDE>
struct StatusWord {
    using T = uint32_t;
    static constexpr T AGG = 1u << 30, INC = 2u << 30, VAL = (1u << 30) - 1;
};
template <>
struct StatusWord<true> {
    using T = unsigned long long;
    static constexpr T AGG = 1ull << 62, INC = 2ull << 62, VAL = (1ull << 62) - 1;
};
constexpr int kScanThreads = 256;

// ---------------------------------------------------------------------------
// K1: digit histograms.  NDIG digits of BITS bits starting at first_shift.
// Every lane owns a private copy of every counter (counter c of lane l lives
// at word c*32 + l, i.e. in bank l), so a warp's 32 shared-memory atomics
// never conflict -- for uniform and for all-equal keys alike.  One persistent
// CTA per SM streams 128-bit loads; copies are reduced once at the end.
// ---------------------------------------------------------------------------
constexpr int kHist2Threads = 1024;

template <int BITS, int NDIG>
__global__ void __launch_bounds__(kHist2Threads)
    hist_kernel(const uint32_t* __restrict__ in, uint64_t n, int first_shift, uint32_t* __restrict__ hist,
                const uint32_t* __restrict__ gate) {
    if (gate && *gate == 0) return; // another route already produced the result (msd.cu)
    constexpr int RADIX = 1 << BITS;
    constexpr uint32_t MASK = RADIX - 1;
    constexpr int COUNTERS = NDIG * RADIX;
    extern __shared__ uint32_t sh[]; // COUNTERS * 32
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < COUNTERS * 32; i += kHist2Threads) sh[i] = 0;
    __syncthreads();
    uint32_t* mine = sh + lane;
    // byte digits: one PRMT per digit and one IMAD for the lane-private
    // counter's byte offset (d * 128 + lane * 4; digit j's table at j * 32 KiB)
    const uint32_t sel = 0x4440u | static_cast<uint32_t>(first_shift >> 3);
    const uint32_t lane4 = static_cast<uint32_t>(lane) * 4u;
    auto count_key = [&](uint32_t key) {
#pragma unroll
        for (int j = 0; j < NDIG; ++j) {
            if constexpr (BITS == 8) {
                const uint32_t d = __byte_perm(key, 0u, sel + static_cast<uint32_t>(j));
                atomicAdd(reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(sh) + (d * 128u + lane4) +
                                                      j * RADIX * 128),
                          1u);
            } else {
                const uint32_t d = (key >> (first_shift + j * BITS)) & MASK;
                atomicAdd(mine + (j * RADIX + d) * 32, 1u);
            }
        }
    };
    const uint64_t mis = (reinterpret_cast<uintptr_t>(in) >> 2) & 3;
    uint64_t head = mis ? 4 - mis : 0;
    if (head > n) head = n;
    const uint4* body = reinterpret_cast<const uint4*>(in + head);
    const uint64_t nvec = (n - head) / 4;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kHist2Threads;
    uint64_t v = static_cast<uint64_t>(blockIdx.x) * kHist2Threads + threadIdx.x;
#if BSG_HIST_LOADS >= 4
    for (; v + 3 * stride < nvec; v += 4 * stride) { // four independent 16-byte loads in flight
        const uint4 a = ldg_stream_v4(body + v);
        const uint4 b = ldg_stream_v4(body + v + stride);
        const uint4 c = ldg_stream_v4(body + v + 2 * stride);
        const uint4 e = ldg_stream_v4(body + v + 3 * stride);
        count_key(a.x); count_key(a.y); count_key(a.z); count_key(a.w);
        count_key(b.x); count_key(b.y); count_key(b.z); count_key(b.w);
        count_key(c.x); count_key(c.y); count_key(c.z); count_key(c.w);
        count_key(e.x); count_key(e.y); count_key(e.z); count_key(e.w);
    }
#endif
    for (; v + stride < nvec; v += 2 * stride) { // two independent 16-byte loads in flight
        const uint4 a = ldg_stream_v4(body + v);
        const uint4 b = ldg_stream_v4(body + v + stride);
        count_key(a.x); count_key(a.y); count_key(a.z); count_key(a.w);
        count_key(b.x); count_key(b.y); count_key(b.z); count_key(b.w);
    }
    for (; v < nvec; v += stride) {
        const uint4 a = ldg_stream_v4(body + v);
        count_key(a.x); count_key(a.y); count_key(a.z); count_key(a.w);
    }
    if (blockIdx.x == 0) {
        for (uint64_t i = threadIdx.x; i < head; i += kHist2Threads) count_key(in[i]);
        for (uint64_t i = head + nvec * 4 + threadIdx.x; i < n; i += kHist2Threads) count_key(in[i]);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < COUNTERS; c += kHist2Threads) {
        uint32_t s = 0;
#pragma unroll 8
        for (int l = 0; l < 32; ++l) s += sh[c * 32 + ((l + c) & 31)]; // rotate: conflict-free
        if (s) atomicAdd(&hist[c], s);
    }
}

template <int BITS, int NDIG>
void launch_hist(const uint32_t* in, uint64_t n, int first_shift, uint32_t* hist, cudaStream_t stream,
                 const uint32_t* gate = nullptr) {
    constexpr size_t smem = sizeof(uint32_t) * NDIG * (1 << BITS) * 32;
    static PerDeviceOccupancy occ;
    auto kern = hist_kernel<BITS, NDIG>;
    const int per_sm = std::max(1, kernel_occupancy(occ, kern, kHist2Threads, smem));
    const int sms = current_sm_count();
    const uint64_t want = (n / 4 + kHist2Threads - 1) / kHist2Threads;
    const unsigned grid = static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, sms * per_sm)));
    kern<<<grid, kHist2Threads, smem, stream>>>(in, n, first_shift, hist, gate);
}

// ---------------------------------------------------------------------------
// K2: digit scans + pass plan.  hist/base layout [chunk][pass][radix].
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kScanThreads)
    scan_plan_kernel(const uint32_t* __restrict__ hist, int chunks, int passes, int radix,
                     uint64_t n, uint64_t* __restrict__ base, PassPlan* __restrict__ plan,
                     const uint32_t* in, uint32_t* out, uint32_t* tmp, int allow_skip,
                     const uint32_t* __restrict__ gate = nullptr) {
    __shared__ uint64_t s_warp[kScanThreads / 32];
    __shared__ int s_active[kMaxPasses];
    __shared__ int s_skew[kMaxPasses];
    const int d = threadIdx.x;
    const int lane = d & 31, warp = d >> 5;
    if (gate && *gate == 0) {
        // another route already produced the result in `out` (msd.cu): no
        // pass runs and nothing is copied
        if (d == 0) {
            PassPlan pl;
            for (int p = 0; p < kMaxPasses; ++p) {
                pl.src[p] = nullptr;
                pl.dst[p] = nullptr;
                pl.active[p] = 0;
                pl.skew[p] = 0;
            }
            pl.executed = 0;
            pl.need_copy = 0;
            pl.final_buf = out;
            *plan = pl;
        }
        return;
    }
    for (int p = 0; p < passes; ++p) {
        uint64_t total = 0;
        if (d < radix)
            for (int c = 0; c < chunks; ++c) total += hist[(static_cast<uint64_t>(c) * passes + p) * radix + d];
        const int ident = __syncthreads_or(d < radix && total == n);
        const int skew = __syncthreads_or(d < radix && total * 16 > n);
        const uint64_t incl = warp_inclusive_scan(total);
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        uint64_t excl = incl - total;
        for (int w = 0; w < warp; ++w) excl += s_warp[w];
        __syncthreads();
        if (d < radix) {
            uint64_t run = excl;
            for (int c = 0; c < chunks; ++c) {
                const uint64_t idx = (static_cast<uint64_t>(c) * passes + p) * radix + d;
                base[idx] = run;
                run += hist[idx];
            }
        }
        if (d == 0) {
            s_active[p] = (n > 0) && !(allow_skip && ident);
            s_skew[p] = skew;
        }
    }
    __syncthreads();
    if (d != 0) return;
    int m = 0;
    for (int p = 0; p < passes; ++p) m += s_active[p];
    PassPlan pl;
    for (int p = 0; p < kMaxPasses; ++p) {
        pl.src[p] = nullptr;
        pl.dst[p] = nullptr;
        pl.active[p] = p < passes ? s_active[p] : 0;
        pl.skew[p] = p < passes ? s_skew[p] : 0;
    }
    pl.executed = m;
    if (m == 0) {
        pl.final_buf = in;
        pl.need_copy = (in != out) && n > 0;
    } else {
        const bool forward = (in == out) && (m % 2 == 1);
        const uint32_t* cur = in;
        int j = 0;
        for (int p = 0; p < passes; ++p) {
            if (!s_active[p]) continue;
            uint32_t* dst;
            if (forward) dst = (j % 2 == 0) ? tmp : out;
            else dst = ((m - 1 - j) % 2 == 0) ? out : tmp;
            pl.src[p] = cur;
            pl.dst[p] = dst;
            cur = dst;
            ++j;
        }
        pl.final_buf = cur;
        pl.need_copy = cur != out;
    }
    *plan = pl;
}

__global__ void final_copy_kernel(const PassPlan* __restrict__ plan, uint32_t* out, uint64_t n) {
    if (!plan->need_copy) return;
    const uint32_t* src = plan->final_buf;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    if (vec) {
        const uint64_t nv = n / 4;
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
        uint4* o4 = reinterpret_cast<uint4*>(out);
        for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nv; i += stride)
            o4[i] = ldg_stream_v4(s4 + i);
        for (uint64_t i = nv * 4 + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
            out[i] = src[i];
    } else {
        for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
            out[i] = src[i];
    }
}

// ---------------------------------------------------------------------------
// K3: one-sweep stable pass (ranking + decoupled look-back + staged scatter).
// Persistent CTAs: while tile k is ranked/scattered, the TMA engine already
// streams tile k+1 into the other shared-memory buffer.
// ---------------------------------------------------------------------------
// The same byte digit computed on the FMA pipe (two IMADs) instead of the
// integer ALU pipe: (k << (24 - shift)) then the high word of (x * 256).
// `mul` = 1 << (24 - shift) is a runtime value so ptxas keeps the IMADs.
__device__ __forceinline__ uint32_t digit8_fma(uint32_t k, uint32_t mul) {
    return __umulhi(k * mul, 256u);
}

template <int BITS>
__device__ __forceinline__ uint32_t digit_of_key(uint32_t k, int shift) {
    if constexpr (BITS == 8) {
        return __byte_perm(k, 0u, 0x4440u | static_cast<uint32_t>(shift >> 3)); // one PRMT
    } else {
        return (k >> shift) & ((1u << BITS) - 1u);
    }
}

// Lanes of the warp holding the same digit (bit-serial ballot multisplit):
// per bit one predicate test, one VOTE, a predicated invert and an AND.
// `neg1` is a runtime -1 (kernel argument) so that ptxas keeps the
// conditional complement ~v = v*(-1) + (-1) as an IMAD on the FMA pipe instead
// of an IADD3/LOP3 on the (half-rate, saturated) integer ALU pipe.
template <int NBITS>
__device__ __forceinline__ uint32_t peers_ballot(uint32_t d, int32_t neg1) {
    uint32_t m[NBITS];
#pragma unroll
    for (int b = 0; b < NBITS; ++b) {
        asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
            "and.b32 t, %1, %2;\n\t"
            "setp.ne.u32 p, t, 0;\n\t"
            "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
            "@!p mad.lo.s32 %0, %0, %3, %3;\n\t}"
            : "=r"(m[b])
            : "r"(d), "r"(1u << b), "r"(neg1));
    }
    // AND-reduce the masks with 3-input LOP3s
    uint32_t peers = m[0];
    int b = 1;
#pragma unroll
    for (; b + 1 < NBITS; b += 2) asm("lop3.b32 %0, %0, %1, %2, 0x80;" : "+r"(peers) : "r"(m[b]), "r"(m[b + 1]));
    if (b < NBITS) peers &= m[b];
    return peers;
}

// Phase-cycle instrumentation (dbg bit 8): thread 0 of every CTA accumulates
// clock64 deltas per phase.  Development aid only.
__device__ unsigned long long g_phase_cycles[16]; // [0..7] thread 0, [8..15] thread 256 (an early-count warp)
#ifndef BSG_LB_STATS
#define BSG_LB_STATS 0 // development: look-back round/predecessor/stall counts (g_lb_stats)
#endif
__device__ unsigned long long g_lb_stats[4]; // rounds, predecessors consumed, unpublished stops, tiles

template <int BITS, int THREADS, int ITEMS, bool WIDE>
struct OnesweepSmem {
    static constexpr int RADIX = 1 << BITS;
    static constexpr int WARPS = THREADS / 32;
    static constexpr int TILE = THREADS * ITEMS;
    static_assert(TILE <= 65536, "16-bit tile offsets");
    using Off = typename std::conditional<WIDE, uint64_t, uint32_t>::type;
    static constexpr size_t in_off = 0;                                          // 2 x TILE u32
    static constexpr size_t wcnt_off = in_off + sizeof(uint32_t) * 2 * TILE;     // WARPS*RADIX u16
    static constexpr size_t delta_off = wcnt_off + sizeof(uint16_t) * WARPS * RADIX; // RADIX Off
    static constexpr size_t excl_off = delta_off + sizeof(uint64_t) * RADIX;     // RADIX u32
    static constexpr size_t tcnt_off = excl_off + sizeof(uint32_t) * RADIX;      // RADIX u32
    static constexpr size_t scan_off = tcnt_off + sizeof(uint32_t) * RADIX;      // 32 u32
    static constexpr size_t misc_off = scan_off + sizeof(uint32_t) * 32;         // 2 tile ids
    static constexpr size_t bar_off = misc_off + 16;                              // 2 mbarriers
    static constexpr size_t range_off = bar_off + 16;                             // 2 x 32 B tile ranges (SEG)
    static constexpr size_t bytes = range_off + 64;
};

// dbg bits (timing experiments only; output is wrong when set):
//   1 = skip look-back waits, 2 = trivial ranks, 4 = skip the write-out,
//   8 = per-phase clock64 accumulation (bsg_debug_phase_cycles), 16 = skip staging.
// One stable pass over chunk_n keys of src (tiles claimed dynamically from
// *tile_counter) into dst; digit_base[d] = destination index of digit d's
// first key of the chunk.  `bar_parity` carries the two mbarriers' phase
// parities across calls (the fused small-n sort runs several passes in one
// launch); `init_bars` initialises them on the first call.
// Segmented pass (the p worker blocks of an in-process PR round in ONE
// launch): segment w = Partition(n, p) block w, nbig blocks of small+1 keys
// then p-nbig of small keys; each segment is its own look-back domain with
// its own digit bases (base table [p][radix]).  tiles are numbered segment
// by segment, so tile -> (segment, start) is a closed form.
struct SegDesc {
    uint64_t small;       // n / p
    uint32_t p, nbig;     // nbig = n % p
    uint32_t tiles_big;   // ceil((small + 1) / TILE)
    uint32_t tiles_small; // ceil(small / TILE)
    uint64_t mbig, msmall; // ceil(2^64 / tiles_*): x / d = umul64hi(x, m) for 32-bit x (d > 1)
    void set_magic() {
        mbig = tiles_big > 1 ? ~0ull / tiles_big + 1 : 0;
        msmall = tiles_small > 1 ? ~0ull / tiles_small + 1 : 0;
    }
};
// x / d for 32-bit x without a division sequence (m = ceil(2^64 / d); exact
// because x * (m * d - 2^64) < 2^64)
__device__ __forceinline__ uint32_t div_magic(uint32_t x, uint32_t d, uint64_t m) {
    return d > 1 ? static_cast<uint32_t>(__umul64hi(static_cast<uint64_t>(x), m)) : x;
}
struct SegTile {
    uint32_t seg, first; // segment and its first tile id
    uint64_t start, end; // key range of the segment
};
template <int TILE>
__device__ __forceinline__ SegTile seg_of_tile(const SegDesc& sd, uint32_t tile) {
    SegTile r;
    const uint32_t big_tiles = sd.nbig * sd.tiles_big;
    if (tile < big_tiles) {
        r.seg = div_magic(tile, sd.tiles_big, sd.mbig);
        r.first = r.seg * sd.tiles_big;
    } else {
        r.seg = sd.nbig + (sd.tiles_small ? div_magic(tile - big_tiles, sd.tiles_small, sd.msmall) : 0u);
        r.first = big_tiles + (r.seg - sd.nbig) * sd.tiles_small;
    }
    r.start = static_cast<uint64_t>(r.seg) * sd.small + (r.seg < sd.nbig ? r.seg : sd.nbig);
    r.end = r.start + sd.small + (r.seg < sd.nbig ? 1 : 0);
    return r;
}

// Keys before the first 16-byte boundary at p (at most 3, at most valid).
__device__ __forceinline__ uint32_t head_words(const uint32_t* p, uint32_t valid) {
    const uint32_t hw = (4u - static_cast<uint32_t>((reinterpret_cast<uintptr_t>(p) >> 2) & 3u)) & 3u;
    return hw < valid ? hw : valid;
}

// Output sinks of the write-out: one array, or the owners' blocks of a PR round.
struct PlainSink {
    uint32_t* __restrict__ dst;
    template <typename Off>
    __device__ __forceinline__ void store(Off pos, uint32_t key) const {
        dst[pos] = key;
    }
};
struct PeerSink {
    const PeerTable* tab; // kernel parameter space
    int p;
    template <typename Off>
    __device__ __forceinline__ void store(Off pos, uint32_t key) const {
        const uint64_t g = static_cast<uint64_t>(pos);
        if (g >= tab->offset[p]) return; // inconsistent count matrix (reported by the caller's row check)
        int w = 0;
        for (int j = 1; j < p; ++j) w += g >= tab->offset[j] ? 1 : 0; // owner: p compares, no division
        tab->blocks[w][g - tab->offset[w]] = key;
    }
};

// Look-back window (predecessors per round trip), measured per configuration:
// 1024-thread CTAs (one per SM) 12; 512-thread CTAs (two per SM, twice the
// tiles in flight) 4 -- a wider window costs more than the extra round trips.
template <int THREADS>
constexpr int default_lb_window() {
    return THREADS <= 512 ? BSG_LB_WIN_SMALL : BSG_LB_WIN;
}

template <int BITS, int THREADS, int ITEMS, bool WIDE, int RANK, typename Sink = PlainSink,
          int LBW = default_lb_window<THREADS>(), bool SEG = false, bool RELAX = false>
__device__ __forceinline__ void onesweep_tiles(uint8_t* __restrict__ smem, const uint32_t* __restrict__ src,
                                               Sink dst, uint64_t chunk_n, int shift,
                                               const uint64_t* __restrict__ digit_base, uint32_t* __restrict__ status,
                                               uint32_t* __restrict__ tile_counter, int use_tma, int dbg,
                                               int32_t neg1, bool init_bars, uint32_t& bar_parity,
                                               const SegDesc sd = SegDesc{}) {
    using L = OnesweepSmem<BITS, THREADS, ITEMS, WIDE>;
    using Off = typename L::Off;
    dbg &= BSG_OS_DBG_MASK; // timing switches exist only in development builds
    constexpr int RADIX = L::RADIX;
    constexpr int WARPS = L::WARPS;
    constexpr int TILE = L::TILE;
    static_assert(ITEMS % 2 == 0, "ranks are packed in pairs");
    static_assert(RADIX <= THREADS, "one thread per digit");
    uint32_t* s_in = reinterpret_cast<uint32_t*>(smem + L::in_off);
    uint16_t* s_wcnt = reinterpret_cast<uint16_t*>(smem + L::wcnt_off); // tile offsets < 2^16
    Off* s_delta = reinterpret_cast<Off*>(smem + L::delta_off);
    uint32_t* s_excl = reinterpret_cast<uint32_t*>(smem + L::excl_off);
    uint32_t* s_tcnt = reinterpret_cast<uint32_t*>(smem + L::tcnt_off);
    uint32_t* s_scan = reinterpret_cast<uint32_t*>(smem + L::scan_off);
    uint32_t* s_tile = reinterpret_cast<uint32_t*>(smem + L::misc_off);
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + L::bar_off);

    const uint32_t ntiles = SEG ? sd.nbig * sd.tiles_big + (sd.p - sd.nbig) * sd.tiles_small
                                : static_cast<uint32_t>((chunk_n + TILE - 1) / TILE);
    // tile -> key range [start, start+valid), look-back floor, digit-base row
    auto tile_range = [&](uint32_t tile, uint64_t& start, uint32_t& valid, uint32_t& first, uint32_t& seg) {
        if constexpr (SEG) {
            const SegTile st = seg_of_tile<TILE>(sd, tile);
            start = st.start + static_cast<uint64_t>(tile - st.first) * TILE;
            valid = static_cast<uint32_t>(min(static_cast<uint64_t>(TILE), st.end - start));
            first = st.first;
            seg = st.seg;
        } else {
            start = static_cast<uint64_t>(tile) * TILE;
            valid = static_cast<uint32_t>(min(static_cast<uint64_t>(TILE), chunk_n - start));
            first = 0;
            seg = 0;
        }
    };
    using SW = StatusWord<WIDE>;
    using Stat = typename SW::T;
    Stat* __restrict__ stat = reinterpret_cast<Stat*>(status);

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;

    // Segmented passes: the tile -> (segment, key range) map is computed once
    // per tile by the claiming thread and read by the others from shared
    // memory (s_range[buffer]: start, valid, first tile, segment)
    uint64_t* s_range = reinterpret_cast<uint64_t*>(smem + L::range_off);
    constexpr bool RCACHE = SEG || BSG_RANGE_CACHE;
    auto buffer_range = [&](uint32_t tile, int b, uint64_t& start, uint32_t& valid, uint32_t& first, uint32_t& seg,
                            uint32_t& hw, uint32_t& body) {
        if constexpr (RCACHE) {
            (void)tile;
            start = s_range[4 * b];
            const uint64_t vf = s_range[4 * b + 1];
            valid = static_cast<uint32_t>(vf);
            first = static_cast<uint32_t>(vf >> 32);
            const uint64_t sh = s_range[4 * b + 2];
            seg = static_cast<uint32_t>(sh);
            const uint32_t hb = static_cast<uint32_t>(sh >> 32); // head words (2 bits) | TMA body << 2
            hw = hb & 3u;
            body = hb >> 2;
        } else {
            tile_range(tile, start, valid, first, seg);
            hw = head_words(src + start, valid);
            body = use_tma ? ((valid - hw) & ~3u) : 0u;
        }
    };
    // Issues the load of `tile` into buffer b (TMA for the 16B-aligned body).
    auto issue = [&](uint32_t tile, int b) {
        if (tile >= ntiles) return;
        uint64_t start;
        uint32_t valid, first_unused, seg_unused;
        tile_range(tile, start, valid, first_unused, seg_unused);
        if constexpr (RCACHE) {
            const uint32_t h = head_words(src + start, valid);
            const uint32_t bd = use_tma ? ((valid - h) & ~3u) : 0u;
            s_range[4 * b] = start;
            s_range[4 * b + 1] = static_cast<uint64_t>(valid) | (static_cast<uint64_t>(first_unused) << 32);
            s_range[4 * b + 2] = static_cast<uint64_t>(seg_unused) | (static_cast<uint64_t>(h | (bd << 2)) << 32);
        }
        // TMA moves the tile's 16-byte-aligned body; the <= 3 head and <= 3
        // tail keys are read with plain loads by the ranking threads
        const uint32_t hw = head_words(src + start, valid);
        const uint32_t body = use_tma ? ((valid - hw) & ~3u) : 0u;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&s_bar[b], body * 4);
        if (body) tma_bulk_g2s(s_in + b * TILE, src + start + hw, body * 4, &s_bar[b]);
    };

    if (tid == 0) {
        if (init_bars) {
            mbar_init(&s_bar[0], 1);
            mbar_init(&s_bar[1], 1);
            fence_mbar_init();
        }
        const uint32_t t0 = atomicAdd(tile_counter, 1u);
        s_tile[0] = t0;
        issue(t0, 0);
    }
    for (int i = tid; i < WARPS * RADIX / 2; i += THREADS) reinterpret_cast<uint32_t*>(s_wcnt)[i] = 0;

    const uint32_t lt = lanemask_lt();
    const uint32_t gt = ~(lt | (1u << lane));
    // per-warp 16-bit digit counters (count-then-rank): +1 on half d & 1 of
    // word d >> 1 of the warp's row.  Byte digits: the word's byte offset as
    // one LOP3 over the 512-byte row base and the increment (1 or 0x10000)
    // as one IMAD on the FMA pipe.
    const uint32_t wrow_bytes = static_cast<uint32_t>(warp) * (RADIX * 2);
    const uint32_t ffff = static_cast<uint32_t>(-neg1) * 0xFFFFu; // runtime 0xFFFF keeps the IMAD
    auto count_digit_row = [&](uint32_t d, uint32_t row_bytes) {
        if constexpr (BITS == 8 && BSG_COUNT_FAST) {
            uint32_t boff, inc;
            asm("lop3.b32 %0, %1, 0x1FC, %2, 0xEA;" : "=r"(boff) : "r"(d << 1), "r"(row_bytes)); // (a & b) | c
            asm("mad.lo.u32 %0, %1, %2, 1;" : "=r"(inc) : "r"(d & 1u), "r"(ffff));
            atomicAdd(reinterpret_cast<uint32_t*>(smem + L::wcnt_off + boff), inc);
        } else {
            atomicAdd(reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(s_wcnt) + row_bytes) + (d >> 1),
                      1u << ((d & 1u) * 16u));
        }
    };
    auto count_digit = [&](uint32_t d) { count_digit_row(d, wrow_bytes); };
    uint32_t lbs_rounds = 0, lbs_used = 0, lbs_stops = 0, lbs_tiles = 0;
    const uint32_t dmul = static_cast<uint32_t>(-neg1) << (BITS == 8 ? (24 - shift) : 0);
    uint32_t keys[ITEMS];
    // Early count (count-then-rank only): while warps [0, WARPS/2) walk the
    // look-back of tile k, warps [WARPS/2, WARPS) already load their keys of
    // tile k+1 (TMA-delivered to the other buffer) and count them into their
    // own (reset) counter rows; in iteration k+1 they skip the count phase.
    constexpr bool EARLY = RANK == 3 && BSG_EARLY_COUNT && BITS == 8 && THREADS == 512 && ITEMS >= 20 &&
                           (BSG_EARLY_WIDE || (!WIDE && !SEG));
    // EARLY2: the early warps also count their partner lower warps' keys of
    // the next tile, so no warp counts at the top of the next iteration
    constexpr bool EARLY2 = EARLY && BSG_EARLY_COUNT >= 2;
    const bool early_warp = EARLY && warp >= WARPS / 2;
    bool have_next = false; // this warp's keys and counts of the current tile are in place
    for (uint32_t k = 0;; ++k) {
        const int cur = k & 1;
        __syncthreads(); // s_tile[cur] visible; previous tile's buffer/counters free
        const uint32_t tile = s_tile[cur];
        if (tile >= ntiles) break;
        // claim the next tile and start its TMA load (buffer cur^1 is free:
        // its tile was written out before the barrier above)
        auto claim_next = [&]() {
            if (tid == 0) {
                const uint32_t nxt = atomicAdd(tile_counter, 1u);
                s_tile[cur ^ 1] = nxt;
                issue(nxt, cur ^ 1);
            }
        };
        if (BSG_CLAIM_AT == 0) claim_next();
        uint64_t tile_start;
        uint32_t valid, tfirst, seg, hw, body;
        buffer_range(tile, cur, tile_start, valid, tfirst, seg, hw, body);
        const bool full = valid == TILE;
        uint32_t* buf = s_in + cur * TILE;
        // non-TMA body / unaligned tail straight from global
        long long t_ph = (dbg & 8) ? clock64() : 0;
        auto phase = [&](int ph) {
            if ((dbg & 8) && (tid == 0 || tid == 256)) {
                const long long now = clock64();
                atomicAdd(&g_phase_cycles[ph + (tid == 256 ? 8 : 0)], static_cast<unsigned long long>(now - t_ph));
                t_ph = now;
            }
        };
        const bool pre = early_warp && have_next; // keys + counts of this tile already in place
        // EARLY2: the lower warps' counts of this tile were taken by their
        // partner early warps as well; they only load their keys
        const bool precounted = EARLY2 && !early_warp && have_next;
        if (!pre) {
            mbar_wait_parity(&s_bar[cur], (bar_parity >> cur) & 1u);
            bar_parity ^= 1u << cur;
        }
        phase(0);

        // ---- warp-local stable ranks + per-warp digit counts --------------
        // Warp w owns keys [w*32*ITEMS, (w+1)*32*ITEMS); item i of lane l is
        // key w*32*ITEMS + i*32 + l: item-major, lane-minor = input order.
        const uint32_t wbase = warp * (32 * ITEMS);
        uint16_t* wc = s_wcnt + warp * RADIX;
        uint32_t packed[ITEMS / 2];
        auto rank_items = [&](auto full_tag, auto aligned_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
            constexpr bool ALIGNED = decltype(aligned_tag)::value;
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const uint32_t idx = wbase + i * 32 + lane;
                const uint32_t rel = idx - hw; // wraps for head keys
                if (FULL && ALIGNED) { // whole tile delivered by TMA
                    keys[i] = buf[idx];
                } else if (FULL) {
                    keys[i] = rel < body ? buf[rel] : __ldg(src + tile_start + idx);
                } else {
                    keys[i] = idx < valid ? (rel < body ? buf[rel] : __ldg(src + tile_start + idx)) : 0u;
                }
            }
            if constexpr (RANK == 3) {
                // count only: per-warp digit histogram by shared-memory
                // reductions (16-bit halves of a word; counts < 2^16)
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const uint32_t idx = wbase + i * 32 + lane;
                    if (FULL || idx < valid) {
                        const uint32_t d = digit_of_key<BITS>(keys[i], shift);
                        count_digit(d);
                    }
                }
                return;
            }
            // multisplit masks in batches of PB items (independent inside a
            // batch), then the per-warp running counts of the batch, item by
            // item (input order): every peer reads the same counter (a
            // broadcast), the highest peer alone stores the advanced count.
            constexpr int PB = ITEMS % 4 == 0 ? 4 : ITEMS;
#pragma unroll
            for (int i0 = 0; i0 < ITEMS; i0 += PB) {
                uint32_t peers[PB], dgt[PB];
#pragma unroll
                for (int ii = 0; ii < PB; ++ii) {
                    const int i = i0 + ii;
                    const uint32_t idx = wbase + i * 32 + lane;
                    const bool ok = FULL || idx < valid;
                    const uint32_t d = ok ? (BITS == 8 ? digit8_fma(keys[i], dmul) : digit_of_key<BITS>(keys[i], shift))
                                          : static_cast<uint32_t>(RADIX);
                    dgt[ii] = d;
                    if (dbg & 2) peers[ii] = 1u << lane;
                    else if (RANK == 1) peers[ii] = __match_any_sync(0xffffffffu, d);
                    else peers[ii] = peers_ballot<FULL ? BITS : BITS + 1>(d, neg1);
                }
#pragma unroll
                for (int ii = 0; ii < PB; ++ii) {
                    const int i = i0 + ii;
                    const uint32_t idx = wbase + i * 32 + lane;
                    const bool ok = FULL || idx < valid;
                    const uint32_t d = ok ? dgt[ii] : 0u;
                    const uint32_t before = ok ? wc[d] : 0u;
                    const bool leader = (peers[ii] & gt) == 0u; // highest peer: no peer above it
                    const uint32_t r = before + __popc(peers[ii] & lt);
                    // the highest peer's rank is before + (group size - 1)
                    if (leader && ok) wc[d] = static_cast<uint16_t>(r + 1);
                    __syncwarp();
                    if (i & 1) packed[i >> 1] = __byte_perm(packed[i >> 1], r, 0x5410);
                    else packed[i >> 1] = r;
                }
            }
        };
        // full TMA tiles rank straight from shared memory; partial tiles and
        // misaligned (non-TMA) bodies take the guarded path
        if (pre) {
            // counted during the previous tile's look-back
        } else if (precounted) {
            // counted by the partner early warp: keys only
            if (full && hw == 0 && body == static_cast<uint32_t>(TILE)) {
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) keys[i] = buf[wbase + i * 32 + lane];
            } else {
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const uint32_t idx = wbase + i * 32 + lane;
                    const uint32_t rel = idx - hw;
                    keys[i] = idx < valid ? (rel < body ? buf[rel] : __ldg(src + tile_start + idx)) : 0u;
                }
            }
        } else if (full && hw == 0 && body == static_cast<uint32_t>(TILE)) rank_items(std::true_type{}, std::true_type{});
        else if (full) rank_items(std::true_type{}, std::false_type{});
        else rank_items(std::false_type{}, std::false_type{});
        have_next = false;
        phase(1);
        __syncthreads();
        phase(2);

        // ---- per-digit: warp prefix, tile count, publish aggregate ---------
        // Thread t < RADIX/2 owns digits 2t, 2t+1: one 32-bit word holds both
        // 16-bit counters (counts and offsets < 2^16: packed adds never carry).
        uint32_t tile_cnt = 0; // digit tid's count, valid for tid < RADIX (see below)
        constexpr int PAIRS = RADIX / 2;
        uint32_t* wc32 = reinterpret_cast<uint32_t*>(s_wcnt);
        uint32_t run2 = 0;
        if (tid < PAIRS) {
#pragma unroll
            for (int w = 0; w < WARPS; ++w) {
                const uint32_t c2 = wc32[w * PAIRS + tid];
                wc32[w * PAIRS + tid] = run2;
                run2 += c2;
            }
            const uint32_t lo = run2 & 0xFFFFu, hi = run2 >> 16;
            const Stat flag = tile == tfirst ? SW::INC : SW::AGG;
            st_relaxed_gpu(&stat[static_cast<uint64_t>(tile) * RADIX + 2 * tid], flag | static_cast<Stat>(lo));
            st_relaxed_gpu(&stat[static_cast<uint64_t>(tile) * RADIX + 2 * tid + 1], flag | static_cast<Stat>(hi));
        }
        constexpr int SCAN_WARPS = (PAIRS + 31) / 32;
        uint32_t pair_incl = 0, pair_sum = 0;
        if (warp < SCAN_WARPS) {
            pair_sum = (run2 & 0xFFFFu) + (run2 >> 16);
            pair_incl = warp_inclusive_scan(pair_sum);
            if (lane == 31) s_scan[warp] = pair_incl;
        }
        if constexpr (BSG_SCAN_NBAR && PAIRS % 32 == 0 && SCAN_WARPS * 32 == PAIRS && PAIRS < THREADS) {
            // only the scan warps exchange partial sums: a named barrier among them
            if (tid < PAIRS) asm volatile("bar.sync 1, %0;" ::"n"(PAIRS) : "memory");
        } else {
            __syncthreads();
        }
        if (tid < PAIRS) {
            uint32_t excl = pair_incl - pair_sum;
#pragma unroll
            for (int w = 0; w < SCAN_WARPS; ++w)
                if (w < warp) excl += s_scan[w];
            const uint32_t excl_hi = excl + (run2 & 0xFFFFu);
            s_excl[2 * tid] = excl;
            s_excl[2 * tid + 1] = excl_hi;
            s_tcnt[2 * tid] = run2 & 0xFFFFu;
            s_tcnt[2 * tid + 1] = run2 >> 16;
            const uint32_t add2 = excl | (excl_hi << 16);
#pragma unroll
            for (int w = 0; w < WARPS; ++w) wc32[w * PAIRS + tid] += add2;
        }
        __syncthreads();
        if (tid < RADIX) tile_cnt = s_tcnt[tid];
        phase(3);

        // ---- stage the tile in digit order (in place: keys are in registers)
        if constexpr (RANK == 3) {
            // rank against the warp's final digit offsets (the counter rows
            // now hold tile offset + warp prefix) and scatter at once
            auto rank_stage = [&](auto full_tag) {
                constexpr bool FULL = decltype(full_tag)::value;
                constexpr int PB = ITEMS % 4 == 0 ? 4 : ITEMS;
                // PB items ranked by the ballot multisplit (input order kept)
                auto ballot_batch = [&](int i0) {
                    uint32_t peers[PB], dgt[PB];
#pragma unroll
                    for (int ii = 0; ii < PB; ++ii) {
                        const int i = i0 + ii;
                        const uint32_t idx = wbase + i * 32 + lane;
                        const bool ok = FULL || idx < valid;
                        const uint32_t d = ok ? (BITS == 8 ? digit8_fma(keys[i], dmul) : digit_of_key<BITS>(keys[i], shift))
                                              : static_cast<uint32_t>(RADIX);
                        dgt[ii] = d;
                        peers[ii] = peers_ballot<FULL ? BITS : BITS + 1>(d, neg1);
                    }
#pragma unroll
                    for (int ii = 0; ii < PB; ++ii) {
                        const int i = i0 + ii;
                        const uint32_t idx = wbase + i * 32 + lane;
                        const bool ok = FULL || idx < valid;
                        const uint32_t d = ok ? dgt[ii] : 0u;
                        const uint32_t before = ok ? wc[d] : 0u;
                        const bool leader = (peers[ii] & gt) == 0u;
                        const uint32_t r = before + __popc(peers[ii] & lt);
                        if (leader && ok) wc[d] = static_cast<uint16_t>(r + 1);
                        __syncwarp();
                        if (ok) buf[r] = keys[i];
                    }
                };
                if constexpr (RELAX && FULL && BITS == 8) {
                    // Value-stable ranking (passes k > 0 of a full keys-only
                    // sort): the input is ordered by the low `shift` bits, and
                    // keys equal in those bits AND in the digit may leave the
                    // pass in any order (later passes and the final array
                    // cannot tell them apart).  A run of items whose first and
                    // last key agree in the low bits holds one low-bits value,
                    // so its keys take their slots by one shared-memory atomic
                    // each on the warp's offset row -- no ballots.  Items are
                    // still ranked in item order, warps and tiles by the scan
                    // and the look-back as in the stable pass.
                    const uint32_t lowmask = (1u << shift) - 1u;
                    auto atomic_item = [&](int i) {
                        const uint32_t key = keys[i];
                        const uint32_t d = digit_of_key<BITS>(key, shift);
                        uint32_t boff, inc, sel;
                        asm("lop3.b32 %0, %1, 0x1FC, %2, 0xEA;" : "=r"(boff) : "r"(d << 1), "r"(wrow_bytes));
                        asm("mad.lo.u32 %0, %1, %2, 1;" : "=r"(inc) : "r"(d & 1u), "r"(ffff));
                        const uint32_t old = atomicAdd(reinterpret_cast<uint32_t*>(smem + L::wcnt_off + boff), inc);
                        asm("mad.lo.u32 %0, %1, 0x22, 0x4410;" : "=r"(sel) : "r"(d & 1u)); // half d & 1 of the word
                        buf[__byte_perm(old, 0u, sel)] = key;
                    };
                    const uint32_t kf = __shfl_sync(0xffffffffu, keys[0], 0);
                    const uint32_t kl = __shfl_sync(0xffffffffu, keys[ITEMS - 1], 31);
                    if (((kf ^ kl) & lowmask) == 0u) {
                        // the warp's whole chunk holds one low-bits value
#pragma unroll
                        for (int i = 0; i < ITEMS; ++i) atomic_item(i);
                        return;
                    }
#pragma unroll
                    for (int i0 = 0; i0 < ITEMS; i0 += PB) {
                        const uint32_t a = __shfl_sync(0xffffffffu, keys[i0], 0);
                        const uint32_t b = __shfl_sync(0xffffffffu, keys[i0 + PB - 1], 31);
                        if (((a ^ b) & lowmask) == 0u) {
#pragma unroll
                            for (int ii = 0; ii < PB; ++ii) atomic_item(i0 + ii);
                            __syncwarp(); // the next batch ranks after these slots are taken
                        } else {
                            ballot_batch(i0);
                        }
                    }
                    return;
                }
#pragma unroll
                for (int i0 = 0; i0 < ITEMS; i0 += PB) ballot_batch(i0);
            };
            if (full) rank_stage(std::true_type{});
            else rank_stage(std::false_type{});
            const uint32_t nxt = s_tile[cur ^ 1];
            if (EARLY2 && !early_warp && nxt < ntiles) {
                // this warp is done with its counter row: the partner early
                // warp may reset it and count this warp's keys of the next tile
                asm volatile("bar.arrive %0, 64;" ::"r"(2 + warp) : "memory");
            }
            if (early_warp) {
                if (nxt < ntiles) {
                    uint64_t nstart;
                    uint32_t nvalid, nfirst, nseg;
                    uint32_t nhw, nbody;
                    buffer_range(nxt, cur ^ 1, nstart, nvalid, nfirst, nseg, nhw, nbody);
                    // own counter row: this tile's ranks are done with it
                    uint32_t* row = reinterpret_cast<uint32_t*>(wc);
                    for (int i = lane; i < RADIX / 2; i += 32) row[i] = 0;
                    const uint32_t pwarp = warp - WARPS / 2; // partner lower warp
                    if (EARLY2) {
                        asm volatile("bar.sync %0, 64;" ::"r"(2 + pwarp) : "memory");
                        uint32_t* prow = reinterpret_cast<uint32_t*>(s_wcnt + pwarp * RADIX);
                        for (int i = lane; i < RADIX / 2; i += 32) prow[i] = 0;
                    }
                    __syncwarp();
                    mbar_wait_parity(&s_bar[cur ^ 1], (bar_parity >> (cur ^ 1)) & 1u);
                    bar_parity ^= 1u << (cur ^ 1);
                    const uint32_t* nbuf = s_in + (cur ^ 1) * TILE;
                    const uint32_t pbase = pwarp * (32 * ITEMS);
                    const uint32_t prow_bytes = pwarp * (RADIX * 2);
                    if (nbody == static_cast<uint32_t>(TILE)) {
                        // whole tile delivered by TMA (full, 16-byte aligned): no guards
#pragma unroll
                        for (int i = 0; i < ITEMS; ++i) keys[i] = nbuf[wbase + i * 32 + lane];
#pragma unroll
                        for (int i = 0; i < ITEMS; ++i) count_digit(digit_of_key<BITS>(keys[i], shift));
                        if (EARLY2) {
#pragma unroll
                            for (int i = 0; i < ITEMS; ++i)
                                count_digit_row(digit_of_key<BITS>(nbuf[pbase + i * 32 + lane], shift), prow_bytes);
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < ITEMS; ++i) {
                            const uint32_t idx = wbase + i * 32 + lane;
                            const uint32_t rel = idx - nhw;
                            keys[i] = idx < nvalid ? (rel < nbody ? nbuf[rel] : __ldg(src + nstart + idx)) : 0u;
                        }
#pragma unroll
                        for (int i = 0; i < ITEMS; ++i) {
                            const uint32_t idx = wbase + i * 32 + lane;
                            if (idx < nvalid) count_digit(digit_of_key<BITS>(keys[i], shift));
                        }
                        if (EARLY2) {
#pragma unroll
                            for (int i = 0; i < ITEMS; ++i) {
                                const uint32_t idx = pbase + i * 32 + lane;
                                const uint32_t rel = idx - nhw;
                                if (idx < nvalid) {
                                    const uint32_t k2 = rel < nbody ? nbuf[rel] : __ldg(src + nstart + idx);
                                    count_digit_row(digit_of_key<BITS>(k2, shift), prow_bytes);
                                }
                            }
                        }
                    }
                }
            }
            have_next = EARLY && nxt < ntiles;
        } else if (dbg & 16) {
            // timing experiment only: skip staging
        } else if (full) { // every item valid: no per-item guards
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const uint32_t r = (packed[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu;
                buf[wc[digit_of_key<BITS>(keys[i], shift)] + r] = keys[i];
            }
        } else {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const uint32_t idx = wbase + i * 32 + lane;
                if (idx < valid) {
                    const uint32_t r = (packed[i >> 1] >> ((i & 1) * 16)) & 0xFFFFu;
                    buf[wc[digit_of_key<BITS>(keys[i], shift)] + r] = keys[i];
                }
            }
        }

        if (BSG_CLAIM_AT == 1) claim_next();
        phase(4);
        // ---- decoupled look-back: LB_WIN predecessors per round trip ------
        // (each warp's load covers 32 consecutive digits of one predecessor:
        // one coalesced 128-byte request per predecessor per warp)
        if (tid < RADIX) {
            constexpr int LB_WIN = LBW;
            constexpr int LB_FIRST = BSG_LB_FIRST > LBW ? BSG_LB_FIRST : LBW;
            Stat prefix = 0;
            // one round trip: W predecessors from t down; consumes the
            // published ones up to the first inclusive (done) or unpublished
            auto lb_round = [&](auto wtag, int32_t& t, bool& done) {
                constexpr int W = decltype(wtag)::value;
                Stat sv[W];
                const Stat* p = stat + static_cast<uint64_t>(static_cast<uint32_t>(t)) * RADIX + tid;
                const int32_t avail = t - static_cast<int32_t>(tfirst); // predecessors t .. t-avail exist
#pragma unroll
                for (int j = 0; j < W; ++j) sv[j] = (j <= avail) ? ld_relaxed_gpu(p - j * RADIX) : SW::INC;
                if constexpr (BSG_LB_FAST) {
                    // common case: W published aggregates -- consume them all
                    Stat all = sv[0], any = sv[0], sum = sv[0];
#pragma unroll
                    for (int j = 1; j < W; ++j) {
                        all &= sv[j];
                        any |= sv[j];
                        sum += sv[j];
                    }
                    if ((all & SW::AGG) && !(any & SW::INC)) {
                        prefix += sum - static_cast<Stat>(W) * SW::AGG; // each word carries the AGG bit once
                        if (BSG_LB_STATS) {
                            ++lbs_rounds;
                            lbs_used += W;
                        }
                        t -= W;
                        return;
                    }
                }
                int used = 0;
                bool stop = false;
#pragma unroll
                for (int j = 0; j < W; ++j) {
                    if (!stop) {
                        if ((sv[j] & ~SW::VAL) == 0) {
                            stop = true;
                        } else {
                            prefix += sv[j] & SW::VAL;
                            ++used;
                            if (sv[j] & SW::INC) done = stop = true;
                        }
                    }
                }
                if (BSG_LB_STATS) {
                    ++lbs_rounds;
                    lbs_used += used;
                    lbs_stops += (!done && used < W) ? 1 : 0;
                }
                t -= used;
            };
            if (tile > tfirst && !(dbg & 1)) {
                int32_t t = static_cast<int32_t>(tile) - 1;
                bool done = false;
                if constexpr (LB_FIRST > LB_WIN) lb_round(std::integral_constant<int, LB_FIRST>{}, t, done);
                while (!done) lb_round(std::integral_constant<int, LB_WIN>{}, t, done);
            }
            if (BSG_LB_STATS) ++lbs_tiles;
            if (tile > tfirst)
                st_relaxed_gpu(&stat[static_cast<uint64_t>(tile) * RADIX + tid],
                               SW::INC | (prefix + static_cast<Stat>(tile_cnt)));
            s_delta[tid] = static_cast<Off>(digit_base[static_cast<uint64_t>(seg) * RADIX + tid] + prefix -
                                            s_excl[tid]);
        }
        phase(7);
        __syncthreads();

        if (BSG_CLAIM_AT == 2) claim_next();
        phase(5);
        // ---- write digit runs (coalesced within each run); reset counters --
        if (EARLY2) {
            // every counter row of the next tile was reset and filled by the early warps
        } else if (EARLY) {
            if (!early_warp) // early warps hold the next tile's counts already
                for (int i = lane; i < RADIX / 2; i += 32) reinterpret_cast<uint32_t*>(wc)[i] = 0;
        } else {
            for (int i = tid; i < WARPS * RADIX / 2; i += THREADS) reinterpret_cast<uint32_t*>(s_wcnt)[i] = 0;
        }
        if (dbg & 4) {
            // timing experiment only: skip the write-out
        } else if (full) {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) {
                const uint32_t i = j * THREADS + tid;
                const uint32_t key = buf[i];
                dst.store(static_cast<Off>(s_delta[digit_of_key<BITS>(key, shift)] + i), key);
            }
        } else {
            for (uint32_t i = tid; i < valid; i += THREADS) {
                const uint32_t key = buf[i];
                dst.store(static_cast<Off>(s_delta[digit_of_key<BITS>(key, shift)] + i), key);
            }
        }
        phase(6);
    }
    if (BSG_LB_STATS && tid < RADIX && lane == 0) {
        atomicAdd(&g_lb_stats[0], static_cast<unsigned long long>(lbs_rounds));
        atomicAdd(&g_lb_stats[1], static_cast<unsigned long long>(lbs_used));
        atomicAdd(&g_lb_stats[2], static_cast<unsigned long long>(lbs_stops));
        atomicAdd(&g_lb_stats[3], static_cast<unsigned long long>(lbs_tiles));
    }
}

// ---------------------------------------------------------------------------
// K3f: the first pass of a full keys-only sort (pass 0 of bsg_radix_sort_u32).
// An LSD sort needs pass k to leave the keys ordered by their low 8(k+1) bits.
// For k > 0 that takes a stable pass (keys with equal digit k keep the order
// of their lower digits); for the first pass nothing below the digit exists,
// so keys with equal digit 0 may land in any order inside their digit run and
// the final sorted array is unchanged (keys equal in every byte are equal).
// The single count-sort round (bsg_count_sort_round_u32, radix.hpp:44-65),
// whose output is observable, always takes the stable K3.  Here:
//   - no ballots: a key's slot inside its tile run is an atomicAdd on a
//     shared-memory cursor; counters are private to a lane quad (counter
//     (d, q) at word d*8 + q, q = lane/4: bank 8*(d&3) + q), so only lanes of
//     one quad can meet in a bank -- about 2 wavefronts per 32 keys instead of
//     ~3.5 for a warp-shared row, and at most 4 for any skew;
//   - no look-back: a tile reserves its slice of digit d's output run with one
//     global atomicAdd per digit (runs are filled in claim order, not tile
//     order).  Status words are not used.
// Tiles, TMA double buffering and the coalesced write-out are K3's.
// ---------------------------------------------------------------------------
constexpr int kFirstGroups = 8; // counter copies per digit (lane quads)

template <int THREADS, int ITEMS, bool WIDE>
struct FirstPassSmem {
    static constexpr int TILE = THREADS * ITEMS;
    using Off = typename std::conditional<WIDE, uint64_t, uint32_t>::type;
    static constexpr size_t in_off = 0;                                           // 2 x TILE u32
    static constexpr size_t cnt_off = in_off + sizeof(uint32_t) * 2 * TILE;       // 256 x 8 u32
    static constexpr size_t delta_off = cnt_off + sizeof(uint32_t) * 256 * kFirstGroups; // 256 Off
    static constexpr size_t scan_off = delta_off + sizeof(uint64_t) * 256;       // 8 u32
    static constexpr size_t misc_off = scan_off + sizeof(uint32_t) * 8;          // 2 tile ids, 2 (head, body)
    static constexpr size_t bar_off = misc_off + 16;                               // 2 mbarriers
    static constexpr size_t bytes = bar_off + 16;
};

template <int THREADS, int ITEMS, bool WIDE>
__global__ void __launch_bounds__(THREADS, 2)
    first_pass_kernel(const PassPlan* __restrict__ plan, uint64_t n, const uint64_t* __restrict__ digit_base,
                      unsigned long long* __restrict__ reserve, uint32_t* __restrict__ tile_counter, int use_tma) {
    using L = FirstPassSmem<THREADS, ITEMS, WIDE>;
    using Off = typename L::Off;
    constexpr int TILE = L::TILE;
    constexpr int WARPS = THREADS / 32;
    static_assert(THREADS >= 256, "one thread per digit in the scan");
    extern __shared__ __align__(128) uint8_t smem[];
    if (!plan->active[0]) return;
    const uint32_t* __restrict__ src = plan->src[0];
    uint32_t* __restrict__ dst = plan->dst[0];
    uint32_t* s_in = reinterpret_cast<uint32_t*>(smem + L::in_off);
    uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem + L::cnt_off);
    Off* s_delta = reinterpret_cast<Off*>(smem + L::delta_off);
    uint32_t* s_scan = reinterpret_cast<uint32_t*>(smem + L::scan_off);
    uint32_t* s_tile = reinterpret_cast<uint32_t*>(smem + L::misc_off); // [0..1] tile ids, [2..3] head | body << 2
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + L::bar_off);
    const uint32_t ntiles = static_cast<uint32_t>((n + TILE - 1) / TILE);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    auto issue = [&](uint32_t tile, int b) {
        if (tile >= ntiles) return;
        const uint64_t start = static_cast<uint64_t>(tile) * TILE;
        const uint32_t valid = static_cast<uint32_t>(min(static_cast<uint64_t>(TILE), n - start));
        const uint32_t hw = head_words(src + start, valid);
        const uint32_t body = use_tma ? ((valid - hw) & ~3u) : 0u;
        s_tile[2 + b] = hw | (body << 2);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&s_bar[b], body * 4);
        if (body) tma_bulk_g2s(s_in + b * TILE, src + start + hw, body * 4, &s_bar[b]);
    };
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_mbar_init();
        const uint32_t t0 = atomicAdd(tile_counter, 1u);
        s_tile[0] = t0;
        issue(t0, 0);
    }
    for (int i = tid; i < 256 * kFirstGroups; i += THREADS) s_cnt[i] = 0;

    // counter (d, q) byte offset: d * 32 + q * 4 = ((key << 5) & 0x1FE0) | q4
    const uint32_t q4 = static_cast<uint32_t>(lane >> 2) * 4u;
    auto cnt_off = [&](uint32_t key) {
        uint32_t o;
        asm("lop3.b32 %0, %1, 0x1FE0, %2, 0xEA;" : "=r"(o) : "r"(key << 5), "r"(q4)); // (a & b) | c
        return o;
    };
    uint8_t* cnt_base = smem + L::cnt_off;
    uint32_t parity = 0;
    uint32_t keys[ITEMS];
    for (uint32_t k = 0;; ++k) {
        const int cur = k & 1;
        __syncthreads(); // s_tile[cur] visible; the previous tile's buffer, counters and deltas are free
        const uint32_t tile = s_tile[cur];
        if (tile >= ntiles) break;
        if (tid == 0) {
            const uint32_t nxt = atomicAdd(tile_counter, 1u);
            s_tile[cur ^ 1] = nxt;
            issue(nxt, cur ^ 1);
        }
        const uint64_t start = static_cast<uint64_t>(tile) * TILE;
        const uint32_t valid = static_cast<uint32_t>(min(static_cast<uint64_t>(TILE), n - start));
        const uint32_t hb = s_tile[2 + cur];
        const uint32_t hw = hb & 3u, body = hb >> 2;
        uint32_t* buf = s_in + cur * TILE;
        mbar_wait_parity(&s_bar[cur], (parity >> cur) & 1u);
        parity ^= 1u << cur;
        const bool fast = body == static_cast<uint32_t>(TILE); // full tile, all of it delivered by TMA
        const uint32_t wbase = warp * (32 * ITEMS);

        // ---- load + count (4 bytes per key: counters hold byte offsets) ----
        if (fast) {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) keys[i] = buf[wbase + i * 32 + lane];
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) atomicAdd(reinterpret_cast<uint32_t*>(cnt_base + cnt_off(keys[i])), 4u);
        } else {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const uint32_t idx = wbase + i * 32 + lane;
                const uint32_t rel = idx - hw; // wraps for head keys
                keys[i] = idx < valid ? (rel < body ? buf[rel] : __ldg(src + start + idx)) : 0u;
            }
#pragma unroll
            for (int i = 0; i < ITEMS; ++i)
                if (wbase + i * 32 + lane < valid)
                    atomicAdd(reinterpret_cast<uint32_t*>(cnt_base + cnt_off(keys[i])), 4u);
        }
        __syncthreads();

        // ---- digit d = tid: quad prefixes -> cursors, tile run start, reservation
        uint32_t total = 0, excl = 0;
        unsigned long long reserved = 0;
        if (tid < 256) {
            uint4* row = reinterpret_cast<uint4*>(s_cnt + tid * kFirstGroups);
            const uint4 a = row[0], b = row[1];
            uint32_t c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            uint32_t run = 0;
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                const uint32_t v = c[g];
                c[g] = run;
                run += v;
            }
            total = run; // bytes
            if (total) reserved = atomicAdd(&reserve[tid], static_cast<unsigned long long>(total >> 2));
            const uint32_t incl = warp_inclusive_scan(total);
            if (lane == 31) s_scan[warp] = incl;
            asm volatile("bar.sync 1, 256;" ::: "memory");
            excl = incl - total;
#pragma unroll
            for (int w = 0; w < 8; ++w)
                if (w < warp) excl += s_scan[w];
            row[0] = make_uint4(c[0] + excl, c[1] + excl, c[2] + excl, c[3] + excl);
            row[1] = make_uint4(c[4] + excl, c[5] + excl, c[6] + excl, c[7] + excl);
        }
        __syncthreads();

        // ---- slot per key, staged in digit order in place ------------------
        uint8_t* bufb = reinterpret_cast<uint8_t*>(buf);
        if (fast) {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                const uint32_t pos = atomicAdd(reinterpret_cast<uint32_t*>(cnt_base + cnt_off(keys[i])), 4u);
                *reinterpret_cast<uint32_t*>(bufb + pos) = keys[i];
            }
        } else {
#pragma unroll
            for (int i = 0; i < ITEMS; ++i)
                if (wbase + i * 32 + lane < valid) {
                    const uint32_t pos = atomicAdd(reinterpret_cast<uint32_t*>(cnt_base + cnt_off(keys[i])), 4u);
                    *reinterpret_cast<uint32_t*>(bufb + pos) = keys[i];
                }
        }
        if (tid < 256) {
            // the tile's run of digit d starts at staged index excl/4 and at
            // output index digit_base[d] + reserved
            s_delta[tid] = static_cast<Off>(digit_base[tid] + reserved - (excl >> 2));
        }
        __syncthreads();
        if (tid < 256) {
            uint4* row = reinterpret_cast<uint4*>(s_cnt + tid * kFirstGroups);
            row[0] = make_uint4(0, 0, 0, 0);
            row[1] = make_uint4(0, 0, 0, 0);
        }

        // ---- write digit runs (coalesced within each run) ------------------
        if (valid == static_cast<uint32_t>(TILE)) {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) {
                const uint32_t i = j * THREADS + tid;
                const uint32_t key = buf[i];
                dst[static_cast<Off>(s_delta[key & 0xFFu] + i)] = key;
            }
        } else {
            for (uint32_t i = tid; i < valid; i += THREADS) {
                const uint32_t key = buf[i];
                dst[static_cast<Off>(s_delta[key & 0xFFu] + i)] = key;
            }
        }
    }
    (void)WARPS;
}

#ifndef BSG_OS_MINB16
#define BSG_OS_MINB16 2 // CTAs per SM the 512 x 16 row is compiled for
#endif
#ifndef BSG_OS_MINB256
#define BSG_OS_MINB256 2 // CTAs per SM the 256-thread rows are compiled for
#endif
template <int THREADS, int ITEMS>
constexpr int onesweep_min_blocks() {
    return THREADS <= 256 ? BSG_OS_MINB256 : (THREADS <= 512 ? (ITEMS <= 16 ? BSG_OS_MINB16 : 2) : 1);
}

template <int BITS, int THREADS, int ITEMS, bool WIDE, int RANK>
__global__ void __launch_bounds__(THREADS, (onesweep_min_blocks<THREADS, ITEMS>()))
    onesweep_kernel(const PassPlan* __restrict__ plan, int pass, uint64_t chunk_off, uint64_t chunk_n,
                    int shift, const uint64_t* __restrict__ digit_base, uint32_t* __restrict__ status,
                    uint32_t* __restrict__ tile_counter, int use_tma, int dbg, int32_t neg1) {
    extern __shared__ __align__(128) uint8_t smem[];
    if (!plan->active[pass]) return;
    uint32_t parity = 0;
    // RANK 4 = count-then-rank (3) with value-stable ranking (see rank_stage)
    constexpr int R = RANK == 4 ? 3 : RANK;
    if constexpr (R == 3) {
        // skewed digit distribution (a digit holds > n/16 keys): the counting
        // reductions would serialise on that digit's counter; rank first
        // (warp-aggregated by the ballot multisplit) instead.  (Two kernels
        // launched back to back, one exiting at once, measured 1.6% slower:
        // an empty 296-CTA launch per pass costs ~13 us.)
        if (plan->skew[pass]) {
            onesweep_tiles<BITS, THREADS, ITEMS, WIDE, 0>(smem, plan->src[pass] + chunk_off,
                                                          PlainSink{plan->dst[pass]}, chunk_n, shift, digit_base,
                                                          status, tile_counter, use_tma, dbg, neg1, true, parity);
            return;
        }
    }
    onesweep_tiles<BITS, THREADS, ITEMS, WIDE, R, PlainSink, default_lb_window<THREADS>(), false, RANK == 4>(
        smem, plan->src[pass] + chunk_off, PlainSink{plan->dst[pass]}, chunk_n, shift, digit_base, status,
        tile_counter, use_tma, dbg, neg1, true, parity);
}

constexpr int kMinTile = 4096;

// 0 = auto by n; otherwise a fixed THREADS x ITEMS row (see launch_onesweep_pass).
// Initialised from BSG_OS_CFG (development builds only); bsg_debug_set_onesweep_cfg
// overrides it (tests).
inline int& onesweep_cfg_ref() {
    static int cfg = dev_knob("BSG_OS_CFG", 0);
    return cfg;
}
inline int onesweep_cfg() { return onesweep_cfg_ref(); }
inline int onesweep_dbg() {
    static int d = dev_knob("BSG_OS_DBG", 0);
    return d;
}

// K3f for the first pass of full sorts (bsg_debug_set_first_pass toggles it:
// tests compare both paths)
inline int& first_pass_ref() {
    static int on = dev_knob("BSG_FIRST_PASS", 1);
    return on;
}
inline bool first_pass_enabled() { return first_pass_ref() != 0; }

// Value-stable ranking in passes k > 0 of full sorts (bsg_debug_set_relaxed_passes
// toggles it: tests compare both paths).  A pass qualifies when the runs of equal
// low bits it meets are long for uniformly distributed low bits: n >> shift keys
// per run, at least kRelaxMinRun (a warp item is 32 keys).
inline int& relaxed_passes_ref() {
    static int on = dev_knob("BSG_RELAXED", 1);
    return on;
}
constexpr uint64_t kRelaxMinRun = 512;
// below 2^24 keys the sort is latency-bound and the ranking is not what it
// waits for (measured 2^22-2^23: +0.4 / +1.9% with the relaxation, 2^24: -0.5%,
// 2^25-2^28: -3.2 .. -4.5%)
constexpr uint64_t kRelaxMinKeys = uint64_t{1} << 24;
inline bool relaxed_pass(uint64_t n, int shift) {
    return relaxed_passes_ref() != 0 && n >= kRelaxMinKeys && shift > 0 && shift < 32 &&
           (n >> shift) >= kRelaxMinRun;
}

inline int onesweep_rank_mode() {
    static int r = dev_knob("BSG_OS_RANK", 0);
    return r;
}

template <int BITS, int THREADS, int ITEMS, bool WIDE, int RANK>
int launch_onesweep_cfg_r(const PassPlan* plan, int pass, uint64_t n, int shift, const uint64_t* base_for_pass,
                          int passes_stride, uint32_t* status, cudaStream_t stream, bool use_tma) {
    using L = OnesweepSmem<BITS, THREADS, ITEMS, WIDE>;
    constexpr int RADIX = 1 << BITS;
    auto kern = onesweep_kernel<BITS, THREADS, ITEMS, WIDE, RANK>;
    static PerDeviceOccupancy occ;
    const int per_sm = std::max(1, kernel_occupancy(occ, kern, THREADS, L::bytes));
    const int sms = current_sm_count();
    // one look-back domain per pass: [tile counter (32 words)] [tiles * RADIX status words]
    const uint32_t tiles = static_cast<uint32_t>((n + L::TILE - 1) / L::TILE);
    const uint32_t grid = std::min<uint32_t>(tiles, static_cast<uint32_t>(sms * per_sm));
    const uint64_t stat_words = static_cast<uint64_t>(tiles) * RADIX * (WIDE ? 2 : 1);
    (void)passes_stride; // digit bases: chunk row 0 of [chunk][pass][radix] = global starts
    if (cudaMemsetAsync(status, 0, (32 + stat_words) * sizeof(uint32_t), stream) != cudaSuccess) return -1;
    TimedScope ts(RANK == 4 ? 5 /*BSG_K_RELAXED_PASS*/ : 0 /*BSG_K_ONESWEEP*/, stream);
    kern<<<grid, THREADS, L::bytes, stream>>>(plan, pass, 0, n, shift, base_for_pass, status + 32, status,
                                               use_tma ? 1 : 0, onesweep_dbg(), -1);
    return 1;
}

template <int BITS, int THREADS, int ITEMS, bool WIDE, bool CAN_RELAX = false>
int launch_onesweep_cfg(const PassPlan* plan, int pass, uint64_t n, int shift, const uint64_t* base_for_pass,
                        int passes_stride, uint32_t* status, cudaStream_t stream, bool use_tma, bool relaxed = false) {
    // RANK 3 = per-warp count by shared-memory reductions, then ballot-multisplit
    // ranks against the final offsets with the scatter (default, BSG_OS_RANK=0);
    // 0 = rank first, stage after the scan (BSG_OS_RANK=2, +3.4% per sort);
    // 1 = match-any ranks (~40 SM-cycles per warp-item on B200)
    if constexpr (BITS == 8) {
        switch (onesweep_rank_mode()) {
        case 1:
            return launch_onesweep_cfg_r<BITS, THREADS, ITEMS, WIDE, 1>(plan, pass, n, shift, base_for_pass,
                                                                        passes_stride, status, stream, use_tma);
        case 2:
            return launch_onesweep_cfg_r<BITS, THREADS, ITEMS, WIDE, 0>(plan, pass, n, shift, base_for_pass,
                                                                        passes_stride, status, stream, use_tma);
        default:
            break;
        }
        // RANK 4: value-stable ranking for passes k > 0 of a full sort
        if constexpr (CAN_RELAX) {
            if (relaxed)
                return launch_onesweep_cfg_r<BITS, THREADS, ITEMS, WIDE, 4>(plan, pass, n, shift, base_for_pass,
                                                                            passes_stride, status, stream, use_tma);
        }
    }
    (void)relaxed;
    return launch_onesweep_cfg_r<BITS, THREADS, ITEMS, WIDE, 3>(plan, pass, n, shift, base_for_pass, passes_stride,
                                                                status, stream, use_tma);
}

template <int BITS>
int launch_onesweep_pass(const PassPlan* plan, int pass, uint64_t n, int shift, const uint64_t* base_for_pass,
                         int passes_stride, uint32_t* status, cudaStream_t stream, bool use_tma,
                         bool relaxed = false) {
    const bool wide = n > kChunkKeys;
    if (wide) // n > 2^29: 64-bit status words and positions, the large-n rows
        return launch_onesweep_cfg<BITS, 512, 24, true, BITS == 8>(plan, pass, n, shift, base_for_pass,
                                                                   passes_stride, status, stream, use_tma, relaxed);
    if constexpr (BITS != 8)
        return launch_onesweep_cfg<BITS, 1024, 16, false>(plan, pass, n, shift, base_for_pass, passes_stride, status,
                                                         stream, use_tma);
    int cfg = onesweep_cfg();
    // measured on B200 with the count-then-rank kernels
    // (profiles/r01_onesweep_cfg_sweep.txt): 512x16 up to 2^25 keys (8192-key
    // tiles, two CTAs per SM; 2^22-2^24: 7% faster than 1024x16), 512x24
    // beyond (12288-key tiles, 4-wide look-back)
    if (cfg == 0) cfg = n <= (uint64_t{1} << 25) ? 1 : 6;
    switch (cfg) {
    case 3: // 256 x 16: 4096-key tiles so small inputs still fill 148 SMs
        return launch_onesweep_cfg<BITS, 256, 16, false>(plan, pass, n, shift, base_for_pass, passes_stride, status,
                                                         stream, use_tma);
    case 1:
        return launch_onesweep_cfg<BITS, 512, 16, false, BITS == 8>(plan, pass, n, shift, base_for_pass,
                                                                    passes_stride, status, stream, use_tma, relaxed);
    case 4:
        return launch_onesweep_cfg<BITS, 1024, 24, false>(plan, pass, n, shift, base_for_pass, passes_stride, status,
                                                          stream, use_tma);
    case 5:
        return launch_onesweep_cfg<BITS, 1024, 20, false>(plan, pass, n, shift, base_for_pass, passes_stride, status,
                                                          stream, use_tma);
    case 6:
        return launch_onesweep_cfg<BITS, 512, 24, false, BITS == 8>(plan, pass, n, shift, base_for_pass,
                                                                    passes_stride, status, stream, use_tma, relaxed);
    case 7:
        return launch_onesweep_cfg<BITS, 256, 24, false>(plan, pass, n, shift, base_for_pass, passes_stride, status,
                                                         stream, use_tma);
#if BSG_DEV_KNOBS
    case 8: // development rows: other tile heights at two CTAs per SM
        return launch_onesweep_cfg<BITS, 512, 22, false>(plan, pass, n, shift, base_for_pass, passes_stride, status,
                                                         stream, use_tma);
    case 9:
        return launch_onesweep_cfg<BITS, 512, 20, false>(plan, pass, n, shift, base_for_pass, passes_stride, status,
                                                         stream, use_tma);
#endif
    default: // 1024 threads x 16 keys: 16384-key tiles, one CTA per SM
        return launch_onesweep_cfg<BITS, 1024, 16, false>(plan, pass, n, shift, base_for_pass, passes_stride, status,
                                                          stream, use_tma);
    }
}

// First pass of a full sort (K3f): [tile counter (32 words)][256 x u64 run
// reservations].  Returns 1 (launches) or -1.
template <int THREADS, int ITEMS, bool WIDE>
int launch_first_pass_cfg(const PassPlan* plan, uint64_t n, const uint64_t* base_for_pass, uint32_t* status,
                          cudaStream_t stream, bool use_tma) {
    using L = FirstPassSmem<THREADS, ITEMS, WIDE>;
    auto kern = first_pass_kernel<THREADS, ITEMS, WIDE>;
    static PerDeviceOccupancy occ; // one per instantiation: the smem attribute is per kernel and device
    const int per_sm = std::max(1, kernel_occupancy(occ, kern, THREADS, L::bytes));
    const uint32_t tiles = static_cast<uint32_t>((n + L::TILE - 1) / L::TILE);
    const uint32_t grid = std::min<uint32_t>(tiles, static_cast<uint32_t>(current_sm_count() * per_sm));
    if (cudaMemsetAsync(status, 0, (32 + 512) * sizeof(uint32_t), stream) != cudaSuccess) return -1;
    TimedScope ts(4 /*BSG_K_FIRST_PASS*/, stream);
    kern<<<grid, THREADS, L::bytes, stream>>>(plan, n, base_for_pass, reinterpret_cast<unsigned long long*>(status + 32),
                                               status, use_tma ? 1 : 0);
    return 1;
}

int launch_first_pass(const PassPlan* plan, uint64_t n, const uint64_t* base_for_pass, uint32_t* status,
                      cudaStream_t stream, bool use_tma) {
    if (n > kChunkKeys) return launch_first_pass_cfg<512, 24, true>(plan, n, base_for_pass, status, stream, use_tma);
    if (n <= (uint64_t{1} << 25))
        return launch_first_pass_cfg<512, 16, false>(plan, n, base_for_pass, status, stream, use_tma);
    return launch_first_pass_cfg<512, 24, false>(plan, n, base_for_pass, status, stream, use_tma);
}

template <int BITS>
uint64_t status_words_for(uint64_t n) {
    constexpr int RADIX = 1 << BITS;
    if (n > kChunkKeys) // WIDE: 512 x 24 tiles, 64-bit status words
        return 32 + ((n + 12287) / 12288) * RADIX * 2;
    return 32 + ((n + kMinTile - 1) / kMinTile) * RADIX;
}


} // namespace

// ---------------------------------------------------------------------------
// Fused small-n SR4 (C1: latency, SURVEY §8(d) "CUDA Graph or persistent
// kernel"): one cooperative launch runs the 4-digit histogram, the digit
// scans + pass plan (computed redundantly by every CTA), and the four
// one-sweep passes, with grid barriers in between, instead of ~10 launches.
// Workspace (zeroed by one memset): hist[4][256] | barrier word (+31 pad) |
// 4 x per-pass look-back regions [tile counter (+31)][tiles][256].
// ---------------------------------------------------------------------------
#ifndef BSG_SMALL_THREADS
#define BSG_SMALL_THREADS 512
#endif
constexpr int kSmallThreads = BSG_SMALL_THREADS, kSmallItems = 16;
constexpr uint64_t kSmallMaxKeys = uint64_t{1} << 21;
constexpr int kSmallHistCopies = 4;

uint64_t small_region_words(uint64_t n) {
    constexpr uint64_t tile = kSmallThreads * kSmallItems;
    return 32 + ((n + tile - 1) / tile) * 256;
}
uint64_t small_ws_words(uint64_t n) { return 1024 + 32 + 4 * small_region_words(n); }

__device__ __forceinline__ void grid_barrier(uint32_t* ctr, uint32_t target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        while (ld_acquire_gpu(ctr) < target) __nanosleep(64);
        __threadfence();
        fence_proxy_async_global(); // next pass's TMA loads read the previous pass's stores
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kSmallThreads, (kSmallThreads <= 512 ? 2 : 1))
    small_sort_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint32_t* __restrict__ tmp,
                      uint32_t n, uint32_t* __restrict__ ws, uint32_t region_words, int use_tma, int32_t neg1) {
    using L = OnesweepSmem<8, kSmallThreads, kSmallItems, false>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* s_base = reinterpret_cast<uint64_t*>(smem + L::bytes); // [4][256]
    __shared__ const uint32_t* s_src[4];
    __shared__ uint32_t* s_dst[4];
    __shared__ int s_active[4];
    __shared__ int s_skew[4];
    __shared__ const uint32_t* s_final;
    __shared__ int s_copy;
    __shared__ uint64_t s_warp[kSmallThreads / 32];
    uint32_t* g_hist = ws;
    uint32_t* g_bar = ws + 1024;
    uint32_t* regions = ws + 1056;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t G = gridDim.x;

    // ---- digit histograms of all four passes (replicated smem counters) --
    uint32_t* s_h = reinterpret_cast<uint32_t*>(smem); // aliases the tile buffers
    for (int i = tid; i < kSmallHistCopies * 1024; i += kSmallThreads) s_h[i] = 0;
    __syncthreads();
    {
        uint32_t* h = s_h + (warp % kSmallHistCopies) * 1024;
        const uint32_t stride = G * kSmallThreads;
        for (uint32_t i = blockIdx.x * kSmallThreads + tid; i < n; i += stride) {
            const uint32_t k = __ldg(in + i);
            atomicAdd(&h[k & 255u], 1u);
            atomicAdd(&h[256 + ((k >> 8) & 255u)], 1u);
            atomicAdd(&h[512 + ((k >> 16) & 255u)], 1u);
            atomicAdd(&h[768 + (k >> 24)], 1u);
        }
    }
    __syncthreads();
    for (int i = tid; i < 1024; i += kSmallThreads) {
        uint32_t v = 0;
#pragma unroll
        for (int c = 0; c < kSmallHistCopies; ++c) v += s_h[c * 1024 + i];
        if (v) atomicAdd(&g_hist[i], v);
    }
    uint32_t bar_target = G;
    grid_barrier(g_bar, bar_target);

    // ---- digit bases + pass plan (scan_plan_kernel's logic, per CTA) -------
    for (int p = 0; p < 4; ++p) {
        const uint32_t total = tid < 256 ? __ldcg(&g_hist[p * 256 + tid]) : 0u;
        const int ident = __syncthreads_or(tid < 256 && total == n);
        const int skew = __syncthreads_or(tid < 256 && static_cast<uint64_t>(total) * 16 > n);
        const uint64_t incl = warp_inclusive_scan(static_cast<uint64_t>(total));
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        uint64_t excl = incl - total;
        for (int w = 0; w < warp; ++w) excl += s_warp[w];
        if (tid < 256) s_base[p * 256 + tid] = excl;
        if (tid == 0) {
            s_active[p] = !ident;
            s_skew[p] = skew;
        }
        __syncthreads();
    }
    if (tid == 0) {
        int m = 0;
        for (int p = 0; p < 4; ++p) m += s_active[p];
        const bool forward = (in == out) && (m % 2 == 1);
        const uint32_t* cur = in;
        int j = 0;
        for (int p = 0; p < 4; ++p) {
            s_src[p] = nullptr;
            s_dst[p] = nullptr;
            if (!s_active[p]) continue;
            uint32_t* d = forward ? ((j % 2 == 0) ? tmp : out) : (((m - 1 - j) % 2 == 0) ? out : tmp);
            s_src[p] = cur;
            s_dst[p] = d;
            cur = d;
            ++j;
        }
        s_final = cur;
        s_copy = cur != out;
    }
    __syncthreads();

    // ---- the executed passes, one grid barrier after each ------------------
    uint32_t parity = 0;
    bool first = true;
    for (int p = 0; p < 4; ++p) {
        if (!s_active[p]) continue;
        uint32_t* region = regions + static_cast<uint64_t>(p) * region_words;
        // all tiles are in flight at once here: the wide window; count then
        // rank unless a digit holds > n/16 keys (then rank first)
        if (s_skew[p])
            onesweep_tiles<8, kSmallThreads, kSmallItems, false, 0, PlainSink, BSG_LB_WIN>(
                smem, s_src[p], PlainSink{s_dst[p]}, n, 8 * p, s_base + p * 256, region + 32, region, use_tma, 0,
                neg1, first, parity);
        else
            onesweep_tiles<8, kSmallThreads, kSmallItems, false, 3, PlainSink, BSG_LB_WIN>(
                smem, s_src[p], PlainSink{s_dst[p]}, n, 8 * p, s_base + p * 256, region + 32, region, use_tma, 0,
                neg1, first, parity);
        first = false;
        bar_target += G;
        grid_barrier(g_bar, bar_target);
    }
    if (s_copy) {
        const uint32_t* src = s_final;
        for (uint32_t i = blockIdx.x * kSmallThreads + tid; i < n; i += G * kSmallThreads) out[i] = __ldcg(src + i);
    }
}

int& small_sort_flag() {
    static int on = dev_knob("BSG_SMALL", 1);
    return on;
}
bool small_sort_enabled() { return small_sort_flag() != 0; }

// Returns launches (1) or 0 when the fused path does not apply, -1 on error.
int launch_small_sort(const uint32_t* in, uint32_t* out, uint64_t n, const RadixWorkspace& ws, cudaStream_t stream,
                      bool tma) {
    if (n == 0 || n > kSmallMaxKeys || !small_sort_enabled()) return 0;
    using L = OnesweepSmem<8, kSmallThreads, kSmallItems, false>;
    const size_t smem = L::bytes + 4 * 256 * sizeof(uint64_t);
    static PerDeviceOccupancy occ;
    const int per_sm = kernel_occupancy(occ, small_sort_kernel, kSmallThreads, smem);
    const int sms = current_sm_count();
    if (per_sm < 1) return 0;
    const uint64_t region = small_region_words(n);
    if (cudaMemsetAsync(ws.status, 0, small_ws_words(n) * sizeof(uint32_t), stream) != cudaSuccess) return -1;
    // grid: every tile gets a CTA, at least one CTA per SM for the histogram
    // (measured: 2^20 keys 56 us at 148 CTAs vs 59 us at all 296 resident)
    static const int gmin = dev_knob("BSG_SMALL_GRID", kSmCountB200);
    const uint64_t tiles = (n + kSmallThreads * kSmallItems - 1) / (kSmallThreads * kSmallItems);
    unsigned grid = static_cast<unsigned>(per_sm * sms);
    if (gmin > 0) grid = static_cast<unsigned>(std::min<uint64_t>(grid, std::max<uint64_t>(tiles, gmin)));
    const uint32_t* a_in = in;
    uint32_t* a_out = out;
    uint32_t* a_tmp = ws.tmp;
    uint32_t a_n = static_cast<uint32_t>(n);
    uint32_t* a_ws = ws.status;
    uint32_t a_region = static_cast<uint32_t>(region);
    int a_tma = tma ? 1 : 0;
    int32_t a_neg1 = -1;
    void* args[] = {&a_in, &a_out, &a_tmp, &a_n, &a_ws, &a_region, &a_tma, &a_neg1};
    TimedScope ts(0 /*BSG_K_ONESWEEP*/, stream);
    if (cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(small_sort_kernel), dim3(grid), dim3(kSmallThreads),
                                    args, smem, stream) != cudaSuccess)
        return -1;
    return 1;
}

// ---------------------------------------------------------------------------
// PR round fused with its exchange (launch_onesweep_peer, see radix.cuh).
// ---------------------------------------------------------------------------
template <int BITS, int THREADS, int ITEMS, bool WIDE>
__global__ void __launch_bounds__(THREADS, (THREADS <= 512 ? 2 : 1))
    onesweep_peer_kernel(const uint32_t* __restrict__ src, uint64_t len, int shift,
                         const uint64_t* __restrict__ digit_base, uint32_t* __restrict__ status,
                         uint32_t* __restrict__ tile_counter, int use_tma, int32_t neg1,
                         const __grid_constant__ PeerTable tab, int p, const uint32_t* __restrict__ skew) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t parity = 0;
    // count then rank unless the round's count matrix has a heavy digit
    if (BITS == 8 && skew && !*skew)
        onesweep_tiles<BITS, THREADS, ITEMS, WIDE, 3, PeerSink>(smem, src, PeerSink{&tab, p}, len, shift, digit_base,
                                                                  status, tile_counter, use_tma, 0, neg1, true, parity);
    else
        onesweep_tiles<BITS, THREADS, ITEMS, WIDE, 0, PeerSink>(smem, src, PeerSink{&tab, p}, len, shift, digit_base,
                                                                  status, tile_counter, use_tma, 0, neg1, true, parity);
    __threadfence_system(); // peer stores performed before the round's barrier
}

template <int BITS, int THREADS, int ITEMS, bool WIDE = false>
int launch_onesweep_peer_cfg(const uint32_t* block, uint64_t len, int shift, const uint64_t* digit_base,
                             uint32_t* status, const PeerTable& tab, int p, cudaStream_t stream,
                             const uint32_t* skew) {
    using L = OnesweepSmem<BITS, THREADS, ITEMS, WIDE>;
    auto kern = onesweep_peer_kernel<BITS, THREADS, ITEMS, WIDE>;
    static PerDeviceOccupancy occ;
    const int per_sm = std::max(1, kernel_occupancy(occ, kern, THREADS, L::bytes));
    const int sms = current_sm_count();
    constexpr int RADIX = 1 << BITS;
    const uint32_t tiles = static_cast<uint32_t>((len + L::TILE - 1) / L::TILE);
    const uint32_t grid = std::min<uint32_t>(tiles, static_cast<uint32_t>(sms * per_sm));
    if (cudaMemsetAsync(status, 0, (32 + static_cast<uint64_t>(tiles) * RADIX * (WIDE ? 2 : 1)) * sizeof(uint32_t),
                        stream) != cudaSuccess)
        return -1;
    const bool tma = true; // per-tile aligned bodies (head/tail keys via plain loads)
    TimedScope ts(3 /*BSG_K_PR*/, stream);
    kern<<<grid, THREADS, L::bytes, stream>>>(block, len, shift, digit_base, status + 32, status, tma ? 1 : 0, -1,
                                              tab, p, skew);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_onesweep_peer(const uint32_t* block, uint64_t len, int bits, int shift, const uint64_t* digit_base,
                         uint32_t* status, const PeerTable& tab, int p, cudaStream_t stream, const uint32_t* skew,
                         uint64_t n_total) {
    if (len == 0) return 0;
    // 64-bit status words and positions when the block exceeds a 30-bit
    // look-back count (config 5: 2^30-2^32 keys per GPU) OR when the global
    // positions the write-out computes (digit bases up to n_total) do not fit
    // in 32 bits -- e.g. 2^28 keys per GPU at p >= 17, or 2^33 keys at p = 16.
    if (len > kChunkKeys || n_total > 0xFFFFFFFFull) {
        switch (bits) {
        case 1: return launch_onesweep_peer_cfg<1, 512, 24, true>(block, len, shift, digit_base, status, tab, p, stream, skew);
        case 2: return launch_onesweep_peer_cfg<2, 512, 24, true>(block, len, shift, digit_base, status, tab, p, stream, skew);
        case 4: return launch_onesweep_peer_cfg<4, 512, 24, true>(block, len, shift, digit_base, status, tab, p, stream, skew);
        case 8: return launch_onesweep_peer_cfg<8, 512, 24, true>(block, len, shift, digit_base, status, tab, p, stream, skew);
        default: return -1;
        }
    }
    const uint32_t n = static_cast<uint32_t>(len);
    switch (bits) {
    case 1: return launch_onesweep_peer_cfg<1, 1024, 16>(block, n, shift, digit_base, status, tab, p, stream, skew);
    case 2: return launch_onesweep_peer_cfg<2, 1024, 16>(block, n, shift, digit_base, status, tab, p, stream, skew);
    case 4: return launch_onesweep_peer_cfg<4, 1024, 16>(block, n, shift, digit_base, status, tab, p, stream, skew);
    case 8:
        if (len > (uint64_t{1} << 23))
            return launch_onesweep_peer_cfg<8, 512, 24>(block, n, shift, digit_base, status, tab, p, stream, skew);
        return launch_onesweep_peer_cfg<8, 512, 16>(block, n, shift, digit_base, status, tab, p, stream, skew);
    default: return -1;
    }
}

// ---------------------------------------------------------------------------
// Segmented pass: all worker blocks of an in-process PR round in one launch.
// ---------------------------------------------------------------------------
// WIDE: 64-bit status words and positions (segments above 2^29 keys or
// arrays above 2^32 keys, e.g. BASELINE config 5's n = 2^33 with p <= 8).
// RELAX: value-stable ranking (rank_stage) -- the rounds of a full in-process
// PR run, whose worker blocks are ordered by the low `shift` bits (round 0:
// shift = 0, every key qualifies).
template <int BITS, int THREADS, int ITEMS, bool WIDE, bool RELAX>
__global__ void __launch_bounds__(THREADS, (THREADS <= 512 ? 2 : 1))
    onesweep_seg_kernel(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, const SegDesc sd, int shift,
                        const uint64_t* __restrict__ base_table, uint32_t* __restrict__ status,
                        uint32_t* __restrict__ tile_counter, int32_t neg1, const uint32_t* __restrict__ skew) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t parity = 0;
    // count then rank unless the caller flags a heavy digit (or gives no flag)
    if (BITS == 8 && skew && !*skew)
        onesweep_tiles<BITS, THREADS, ITEMS, WIDE, 3, PlainSink, default_lb_window<THREADS>(), true, RELAX>(
            smem, src, PlainSink{dst}, 0, shift, base_table, status, tile_counter, 1, 0, neg1, true, parity, sd);
    else
        onesweep_tiles<BITS, THREADS, ITEMS, WIDE, 0, PlainSink, default_lb_window<THREADS>(), true>(
            smem, src, PlainSink{dst}, 0, shift, base_table, status, tile_counter, 1, 0, neg1, true, parity, sd);
}

template <int BITS, int THREADS, int ITEMS, bool WIDE = false, bool RELAX = false>
int launch_onesweep_seg_cfg(const uint32_t* src, uint32_t* dst, uint64_t n, int p, int shift,
                            const uint64_t* base_table, uint32_t* status, cudaStream_t stream,
                            const uint32_t* skew) {
    using L = OnesweepSmem<BITS, THREADS, ITEMS, WIDE>;
    constexpr int RADIX = 1 << BITS;
    auto kern = onesweep_seg_kernel<BITS, THREADS, ITEMS, WIDE, RELAX>;
    static PerDeviceOccupancy occ;
    const int per_sm = std::max(1, kernel_occupancy(occ, kern, THREADS, L::bytes));
    const int sms = current_sm_count();
    SegDesc sd;
    sd.small = n / static_cast<uint64_t>(p);
    sd.p = static_cast<uint32_t>(p);
    sd.nbig = static_cast<uint32_t>(n % static_cast<uint64_t>(p));
    sd.tiles_big = static_cast<uint32_t>((sd.small + 1 + L::TILE - 1) / L::TILE);
    sd.tiles_small = static_cast<uint32_t>((sd.small + L::TILE - 1) / L::TILE);
    sd.set_magic();
    const uint64_t tiles = static_cast<uint64_t>(sd.nbig) * sd.tiles_big +
                           static_cast<uint64_t>(sd.p - sd.nbig) * sd.tiles_small;
    if (tiles == 0) return 0;
    const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(tiles, static_cast<uint64_t>(sms) * per_sm));
    if (cudaMemsetAsync(status, 0, (32 + tiles * RADIX * (WIDE ? 2 : 1)) * sizeof(uint32_t), stream) != cudaSuccess)
        return -1;
    TimedScope ts(0 /*BSG_K_ONESWEEP*/, stream);
    kern<<<grid, THREADS, L::bytes, stream>>>(src, dst, sd, shift, base_table, status + 32, status, -1, skew);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_onesweep_seg(const uint32_t* src, uint32_t* dst, uint64_t n, int p, int bits, int shift,
                        const uint64_t* base_table, uint32_t* status, cudaStream_t stream, const uint32_t* skew,
                        bool full_run) {
    if (n == 0) return 0;
    // rounds of a full run may rank value-stably (round 0: nothing below the digit)
    const bool relaxed = full_run && bits == 8 && relaxed_passes_ref() != 0 && n >= kRelaxMinKeys &&
                         (shift == 0 || relaxed_pass(n, shift));
    if (n / static_cast<uint64_t>(p) + 1 > kChunkKeys || n > 0xFFFFFFFFull) {
        // 64-bit status words and positions
        if (bits != 8) return -1;
        if (relaxed)
            return launch_onesweep_seg_cfg<8, 512, 24, true, true>(src, dst, n, p, shift, base_table, status, stream,
                                                                   skew);
        return launch_onesweep_seg_cfg<8, 512, 24, true>(src, dst, n, p, shift, base_table, status, stream, skew);
    }
    if (relaxed) // n >= 2^24: the 12288-key tile row
        return launch_onesweep_seg_cfg<8, 512, 24, false, true>(src, dst, n, p, shift, base_table, status, stream,
                                                                skew);
    switch (bits) {
    case 1: return launch_onesweep_seg_cfg<1, 512, 16>(src, dst, n, p, shift, base_table, status, stream, skew);
    case 2: return launch_onesweep_seg_cfg<2, 512, 16>(src, dst, n, p, shift, base_table, status, stream, skew);
    case 4: return launch_onesweep_seg_cfg<4, 512, 16>(src, dst, n, p, shift, base_table, status, stream, skew);
    case 8:
        if (n > (uint64_t{1} << 23))
            return launch_onesweep_seg_cfg<8, 512, 24>(src, dst, n, p, shift, base_table, status, stream, skew);
        return launch_onesweep_seg_cfg<8, 512, 16>(src, dst, n, p, shift, base_table, status, stream, skew);
    default: return -1;
    }
}

// Segmented pass whose write-out goes through a PeerTable: the member of a
// multi-GPU group runs its workers' blocks as segments; key positions are
// global and land in the owning member's next-round buffer (local or a peer
// GPU's, NVLink stores).  G = members in the table.
template <int BITS, int THREADS, int ITEMS, bool WIDE>
__global__ void __launch_bounds__(THREADS, (THREADS <= 512 ? 2 : 1))
    onesweep_seg_peer_kernel(const uint32_t* __restrict__ src, const SegDesc sd, int shift,
                             const uint64_t* __restrict__ base_table, uint32_t* __restrict__ status,
                             uint32_t* __restrict__ tile_counter, int32_t neg1, const uint32_t* __restrict__ skew,
                             const __grid_constant__ PeerTable tab, int G) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint32_t parity = 0;
    if (BITS == 8 && skew && !*skew)
        onesweep_tiles<BITS, THREADS, ITEMS, WIDE, 3, PeerSink, default_lb_window<THREADS>(), true>(
            smem, src, PeerSink{&tab, G}, 0, shift, base_table, status, tile_counter, 1, 0, neg1, true, parity, sd);
    else
        onesweep_tiles<BITS, THREADS, ITEMS, WIDE, 0, PeerSink, default_lb_window<THREADS>(), true>(
            smem, src, PeerSink{&tab, G}, 0, shift, base_table, status, tile_counter, 1, 0, neg1, true, parity, sd);
    __threadfence_system(); // peer stores performed before the round's cross-GPU barrier
}

template <int BITS, int THREADS, int ITEMS, bool WIDE = false>
int launch_onesweep_seg_peer_cfg(const uint32_t* src, uint64_t n, int p, int shift, const uint64_t* base_table,
                                 uint32_t* status, cudaStream_t stream, const uint32_t* skew, const PeerTable& tab,
                                 int G) {
    using L = OnesweepSmem<BITS, THREADS, ITEMS, WIDE>;
    constexpr int RADIX = 1 << BITS;
    auto kern = onesweep_seg_peer_kernel<BITS, THREADS, ITEMS, WIDE>;
    static PerDeviceOccupancy occ;
    const int per_sm = std::max(1, kernel_occupancy(occ, kern, THREADS, L::bytes));
    const int sms = current_sm_count();
    SegDesc sd;
    sd.small = n / static_cast<uint64_t>(p);
    sd.p = static_cast<uint32_t>(p);
    sd.nbig = static_cast<uint32_t>(n % static_cast<uint64_t>(p));
    sd.tiles_big = static_cast<uint32_t>((sd.small + 1 + L::TILE - 1) / L::TILE);
    sd.tiles_small = static_cast<uint32_t>((sd.small + L::TILE - 1) / L::TILE);
    sd.set_magic();
    const uint64_t tiles = static_cast<uint64_t>(sd.nbig) * sd.tiles_big +
                           static_cast<uint64_t>(sd.p - sd.nbig) * sd.tiles_small;
    if (tiles == 0) return 0;
    const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(tiles, static_cast<uint64_t>(sms) * per_sm));
    if (cudaMemsetAsync(status, 0, (32 + tiles * RADIX * (WIDE ? 2 : 1)) * sizeof(uint32_t), stream) != cudaSuccess)
        return -1;
    TimedScope ts(3 /*BSG_K_PR*/, stream);
    kern<<<grid, THREADS, L::bytes, stream>>>(src, sd, shift, base_table, status + 32, status, -1, skew, tab, G);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_onesweep_seg_peer(const uint32_t* src, uint64_t n, int p, int bits, int shift, const uint64_t* base_table,
                             uint32_t* status, cudaStream_t stream, const uint32_t* skew, const PeerTable& tab, int G,
                             uint64_t n_total) {
    if (n == 0) return 0;
    // 64-bit rows when a segment exceeds a 30-bit look-back count or global
    // positions exceed 32 bits
    if (n / static_cast<uint64_t>(p) + 1 > kChunkKeys || n_total > 0xFFFFFFFFull) {
        switch (bits) {
        case 1: return launch_onesweep_seg_peer_cfg<1, 512, 24, true>(src, n, p, shift, base_table, status, stream, skew, tab, G);
        case 2: return launch_onesweep_seg_peer_cfg<2, 512, 24, true>(src, n, p, shift, base_table, status, stream, skew, tab, G);
        case 4: return launch_onesweep_seg_peer_cfg<4, 512, 24, true>(src, n, p, shift, base_table, status, stream, skew, tab, G);
        case 8: return launch_onesweep_seg_peer_cfg<8, 512, 24, true>(src, n, p, shift, base_table, status, stream, skew, tab, G);
        default: return -1;
        }
    }
    switch (bits) {
    case 1: return launch_onesweep_seg_peer_cfg<1, 512, 16>(src, n, p, shift, base_table, status, stream, skew, tab, G);
    case 2: return launch_onesweep_seg_peer_cfg<2, 512, 16>(src, n, p, shift, base_table, status, stream, skew, tab, G);
    case 4: return launch_onesweep_seg_peer_cfg<4, 512, 16>(src, n, p, shift, base_table, status, stream, skew, tab, G);
    case 8:
        if (n > (uint64_t{1} << 23))
            return launch_onesweep_seg_peer_cfg<8, 512, 24>(src, n, p, shift, base_table, status, stream, skew, tab, G);
        return launch_onesweep_seg_peer_cfg<8, 512, 16>(src, n, p, shift, base_table, status, stream, skew, tab, G);
    default: return -1;
    }
}

uint64_t onesweep_seg_status_words(uint64_t n, int p) {
    // 8192-key tiles at the smallest: one extra partial tile per segment
    // (64-bit words for the large segments of the WIDE rows)
    return 32 + (n / 8192 + static_cast<uint64_t>(p) + 1) * 256 * 2;
}

uint64_t onesweep_status_words(uint64_t n) {
    const uint64_t w = status_words_for<8>(n);
    return n <= kSmallMaxKeys ? std::max<uint64_t>(w, small_ws_words(n)) : w;
}


int launch_radix_sort8(const uint32_t* in, uint32_t* out, uint64_t n, const RadixWorkspace& ws,
                       cudaStream_t stream, bool allow_tma, const uint32_t* gate) {
    return launch_byte_passes(in, out, n, 0, 4, ws, stream, allow_tma, gate);
}

// `passes` stable 8-bit passes over bytes first_byte .. first_byte+passes-1:
// ONE histogram read for all of them (digit histograms are properties of the
// multiset, so every pass's bases come from the input), one scan/plan, the
// passes ping-ponging through ws.tmp.  passes = 4: the full sort (SR4, and
// the r = 2^16 sort as 2 rounds x 2 byte sub-passes); passes = 2: one
// r = 2^16 count-sort round (radix.hpp:44-65 at r = 65536) at 20 B/key.
int launch_byte_passes(const uint32_t* in, uint32_t* out, uint64_t n, int first_byte, int passes,
                       const RadixWorkspace& ws, cudaStream_t stream, bool allow_tma, const uint32_t* gate) {
    constexpr int RADIX = 256;
    const uint64_t chunks = n ? (n + kChunkKeys - 1) / kChunkKeys : 1;
    int launches = 0;
    if (passes == 4 && first_byte == 0) {
        const bool tma = allow_tma; // tiles TMA their 16-byte-aligned bodies at any alignment
        const int l = gate ? 0 : launch_small_sort(in, out, n, ws, stream, tma);
        if (l != 0) return l;
    }
    if (passes < 1 || passes > 4 || first_byte + passes > 4) return -1;
    if (cudaMemsetAsync(ws.hist, 0, chunks * passes * RADIX * sizeof(uint32_t), stream) != cudaSuccess) return -1;
    for (uint64_t c = 0; c < chunks && n; ++c) {
        const uint64_t off = c * kChunkKeys;
        const uint64_t len = std::min<uint64_t>(kChunkKeys, n - off);
        TimedScope ts(1 /*BSG_K_HIST*/, stream);
        uint32_t* h = ws.hist + c * passes * RADIX;
        switch (passes) {
        case 1: launch_hist<8, 1>(in + off, len, 8 * first_byte, h, stream, gate); break;
        case 2: launch_hist<8, 2>(in + off, len, 8 * first_byte, h, stream, gate); break;
        case 3: launch_hist<8, 3>(in + off, len, 8 * first_byte, h, stream, gate); break;
        default: launch_hist<8, 4>(in + off, len, 8 * first_byte, h, stream, gate); break;
        }
        ++launches;
    }
    scan_plan_kernel<<<1, kScanThreads, 0, stream>>>(ws.hist, static_cast<int>(chunks), passes, RADIX, n, ws.base,
                                                     ws.plan, in, out, ws.tmp, 1, gate);
    ++launches;
    const bool tma = allow_tma; // tiles TMA their 16-byte-aligned bodies at any alignment
    // a full sort's first pass needs no order inside a digit run (K3f)
    const bool first_free = passes == 4 && first_byte == 0 && first_pass_enabled();
    for (int p = 0; p < passes && n; ++p) {
        if (p == 0 && first_free) {
            const int l = launch_first_pass(ws.plan, n, ws.base, ws.status, stream, tma);
            if (l < 0) return -1;
            launches += l;
            continue;
        }
        // passes k > 0 of a full sort read keys ordered by their low 8k bits
        // and need keep only that order (value-stable ranking)
        const bool relaxed = passes == 4 && first_byte == 0 && p > 0 && relaxed_pass(n, 8 * p);
        const int l = launch_onesweep_pass<8>(ws.plan, p, n, 8 * (first_byte + p), ws.base + p * RADIX, passes,
                                              ws.status, stream, tma, relaxed);
        if (l < 0) return -1;
        launches += l;
    }
    final_copy_kernel<<<kSmCountB200 * 4, 256, 0, stream>>>(ws.plan, out, n);
    ++launches;
    if (cudaGetLastError() != cudaSuccess) return -1;
    return launches;
}

int launch_count_pass(const uint32_t* in, uint32_t* out, uint64_t n, int bits, int shift,
                      const RadixWorkspace& ws, cudaStream_t stream, bool allow_tma) {
    const int radix = 1 << bits;
    const uint64_t chunks = n ? (n + kChunkKeys - 1) / kChunkKeys : 1;
    int launches = 0;
    if (cudaMemsetAsync(ws.hist, 0, chunks * radix * sizeof(uint32_t), stream) != cudaSuccess) return -1;
    for (uint64_t c = 0; c < chunks && n; ++c) {
        const uint64_t off = c * kChunkKeys;
        const uint64_t len = std::min<uint64_t>(kChunkKeys, n - off);
        uint32_t* h = ws.hist + c * radix;
        switch (bits) {
        case 1: launch_hist<1, 1>(in + off, len, shift, h, stream); break;
        case 2: launch_hist<2, 1>(in + off, len, shift, h, stream); break;
        case 4: launch_hist<4, 1>(in + off, len, shift, h, stream); break;
        case 8: launch_hist<8, 1>(in + off, len, shift, h, stream); break;
        default: return -1;
        }
        ++launches;
    }
    // The reference always performs the pass (no identity skip), but an
    // identity pass is a copy either way; skipping keeps the result identical.
    scan_plan_kernel<<<1, kScanThreads, 0, stream>>>(ws.hist, static_cast<int>(chunks), 1, radix, n, ws.base, ws.plan,
                                                     in, out, ws.tmp, 1);
    ++launches;
    const bool tma = allow_tma; // tiles TMA their 16-byte-aligned bodies at any alignment
    if (n) {
        uint64_t sw = 0;
        switch (bits) {
        case 1: sw = status_words_for<1>(n); break;
        case 2: sw = status_words_for<2>(n); break;
        case 4: sw = status_words_for<4>(n); break;
        default: sw = status_words_for<8>(n); break;
        }
        (void)sw;
        int l1 = 0;
        switch (bits) {
        case 1: l1 = launch_onesweep_pass<1>(ws.plan, 0, n, shift, ws.base, 1, ws.status, stream, tma); break;
        case 2: l1 = launch_onesweep_pass<2>(ws.plan, 0, n, shift, ws.base, 1, ws.status, stream, tma); break;
        case 4: l1 = launch_onesweep_pass<4>(ws.plan, 0, n, shift, ws.base, 1, ws.status, stream, tma); break;
        default: l1 = launch_onesweep_pass<8>(ws.plan, 0, n, shift, ws.base, 1, ws.status, stream, tma); break;
        }
        if (l1 < 0) return -1;
        launches += l1;
    }
    final_copy_kernel<<<kSmCountB200 * 4, 256, 0, stream>>>(ws.plan, out, n);
    ++launches;
    if (cudaGetLastError() != cudaSuccess) return -1;
    return launches;
}

namespace {
__global__ void widen_counts_kernel(const uint32_t* __restrict__ c32, uint64_t* __restrict__ c64, int radix,
                                    int chunks) {
    for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < radix; d += gridDim.x * blockDim.x) {
        uint64_t s = 0;
        for (int c = 0; c < chunks; ++c) s += c32[static_cast<uint64_t>(c) * radix + d];
        c64[d] = s;
    }
}
} // namespace

int launch_digit_counts(const uint32_t* in, uint64_t n, int bits, int shift, uint64_t* counts, uint32_t* scratch32,
                        cudaStream_t stream) {
    const int radix = 1 << bits;
    const uint64_t chunks = n ? (n + kChunkKeys - 1) / kChunkKeys : 1;
    int launches = 0;
    if (cudaMemsetAsync(scratch32, 0, chunks * radix * sizeof(uint32_t), stream) != cudaSuccess) return -1;
    for (uint64_t c = 0; c < chunks && n; ++c) {
        const uint64_t off = c * kChunkKeys;
        const uint64_t len = std::min<uint64_t>(kChunkKeys, n - off);
        uint32_t* h = scratch32 + c * radix;
        switch (bits) {
        case 1: launch_hist<1, 1>(in + off, len, shift, h, stream); break;
        case 2: launch_hist<2, 1>(in + off, len, shift, h, stream); break;
        case 4: launch_hist<4, 1>(in + off, len, shift, h, stream); break;
        case 8: launch_hist<8, 1>(in + off, len, shift, h, stream); break;
        default: return -1;
        }
        ++launches;
    }
    widen_counts_kernel<<<(radix + 255) / 256, 256, 0, stream>>>(scratch32, counts, radix, static_cast<int>(chunks));
    ++launches;
    if (cudaGetLastError() != cudaSuccess) return -1;
    return launches;
}

} // namespace bsg

// Test aid: pins the one-sweep configuration (0 = auto, 1..7 fixed rows) so
// parity tests cover every instantiation; returns the previous value.
extern "C" int bsg_debug_set_onesweep_cfg(int cfg) {
    const int prev = bsg::onesweep_cfg_ref();
    bsg::onesweep_cfg_ref() = cfg;
    return prev;
}

// Test aid: enables/disables K3f for the first pass of full sorts (on < 0:
// query only); returns the previous setting.
extern "C" int bsg_debug_set_first_pass(int on) {
    const int prev = bsg::first_pass_ref();
    if (on >= 0) bsg::first_pass_ref() = on;
    return prev;
}

// Test aid: enables/disables value-stable ranking in passes k > 0 of full
// sorts (on < 0: query only); returns the previous setting.
extern "C" int bsg_debug_set_relaxed_passes(int on) {
    const int prev = bsg::relaxed_passes_ref();
    if (on >= 0) bsg::relaxed_passes_ref() = on;
    return prev;
}

// Test aid: enables/disables the fused small-n sort (n <= 2^21); returns the
// previous setting.
extern "C" int bsg_debug_set_small_sort(int on) {
    const int prev = bsg::small_sort_flag();
    bsg::small_sort_flag() = on;
    return prev;
}

// Development aid: reads (and optionally clears) the one-sweep phase-cycle
// accumulators filled when BSG_OS_DBG has bit 8 set.
extern "C" int bsg_debug_lb_stats(unsigned long long* out4, int reset) {
    cudaError_t e = cudaMemcpyFromSymbol(out4, bsg::g_lb_stats, sizeof(unsigned long long) * 4);
    if (e == cudaSuccess && reset) {
        unsigned long long z[4] = {0, 0, 0, 0};
        e = cudaMemcpyToSymbol(bsg::g_lb_stats, z, sizeof(z));
    }
    return e == cudaSuccess ? 0 : 3;
}

// (out16: [0..7] thread 0 of every CTA, [8..15] thread 256)
extern "C" int bsg_debug_phase_cycles(unsigned long long* out16, int reset) {
    cudaError_t e = cudaMemcpyFromSymbol(out16, bsg::g_phase_cycles, sizeof(unsigned long long) * 16);
    if (e == cudaSuccess && reset) {
        unsigned long long z[16] = {};
        e = cudaMemcpyToSymbol(bsg::g_phase_cycles, z, sizeof(z));
    }
    return e == cudaSuccess ? 0 : 3;
}
