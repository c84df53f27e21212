// msd.cu -- hybrid full sort for large, evenly spread inputs (keys only).
//
// bsg_radix_sort_u32 returns only the sorted array (radix.hpp:69-90), so a
// full sort may take ANY route to it.  For inputs a little above 2^28 keys
// (msd.cuh: the window it measured >= 5% faster in) whose top 16 bits spread
// evenly this route costs three passes over the keys instead of four and
// none of them ranks with ballots or walks a look-back:
//   H1  hist16: one read, histogram of the top 16 bits (65536 bins; packed
//       16-bit shared-memory counters per CTA, dumped and reduced)
//   H2  plan: bucket offsets (exclusive scan), level-1 digit bases, level-2
//       tile map, and the decision: every top-16-bit bucket <= kLocalCap keys
//   MA  partition by byte 3 (no order inside a digit run: K3f's scheme --
//       shared-memory cursors per lane quad, a global atomic per digit and
//       tile reserves the tile's slice of the digit's run)
//   MB  the same by byte 2 inside each of the 256 byte-3 buckets (tiles never
//       straddle a bucket; digit bases and reservations per (bucket, digit))
//   MC  local sort of each of the 65536 buckets by its low 16 bits in shared
//       memory: a table of 4-bit counters addressed by the 16-bit value
//       (one atomic per key), a prefix over the table, rank = prefix +
//       smaller values in the word + rank among equal keys.
// Anything the route cannot take (a bucket above kLocalCap, more than 15
// equal keys in one bucket, in == out) falls back to the LSD sort of radix.cu
// ON THE DEVICE: the plan or the local sort raise `need_lsd`, which the LSD
// path's histogram and plan kernels read (launch_byte_passes' gate); the
// input is never written, so the fallback re-sorts it from scratch.
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "msd.cuh"
#include "radix.cuh"
#include "timer.cuh"

namespace bsg {

namespace {

constexpr int kH16Threads = 1024;
constexpr int kPartThreads = 512;
constexpr int kPartItems = 24;
constexpr int kPartTile = kPartThreads * kPartItems; // 12288 keys
constexpr int kPartGroups = 8;                       // cursor copies per digit (lane quads)
constexpr int kLocalThreads = 512;
constexpr int kLocalItems = 12;
#ifndef BSG_MSD_LOCAL_CTAS
#define BSG_MSD_LOCAL_CTAS 3 // CTAs per SM the local sort is compiled for (register cap 42 at 3, 64 at 2)
#endif

// ---------------------------------------------------------------------------
// H1: histogram of key >> 16.  One persistent CTA per SM; 32768 words of
// packed 16-bit counters; a half that reaches 0x8000 is moved to the global
// 32-bit bins at once, so no count is ever lost to a carry.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kH16Threads)
    msd_hist16_kernel(const uint32_t* __restrict__ in, uint64_t n, uint32_t* __restrict__ dump,
                      uint32_t* __restrict__ extra) {
    extern __shared__ uint32_t h16[]; // 32768 words
    for (int i = threadIdx.x; i < 32768; i += kH16Threads) h16[i] = 0;
    __syncthreads();
    auto count_key = [&](uint32_t key) {
        const uint32_t d = key >> 16;
        const uint32_t sh = (d & 1u) * 16u;
        const uint32_t old = atomicAdd(&h16[d >> 1], 1u << sh);
        if (((old >> sh) & 0xFFFFu) == 0x7FFFu) { // this add made it 0x8000
            atomicSub(&h16[d >> 1], 0x8000u << sh);
            atomicAdd(&extra[d], 0x8000u);
        }
    };
    const uint64_t mis = (reinterpret_cast<uintptr_t>(in) >> 2) & 3;
    uint64_t head = mis ? 4 - mis : 0;
    if (head > n) head = n;
    const uint4* body = reinterpret_cast<const uint4*>(in + head);
    const uint64_t nvec = (n - head) / 4;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kH16Threads;
    uint64_t v = static_cast<uint64_t>(blockIdx.x) * kH16Threads + threadIdx.x;
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
    for (; v < nvec; v += stride) {
        const uint4 a = ldg_stream_v4(body + v);
        count_key(a.x); count_key(a.y); count_key(a.z); count_key(a.w);
    }
    if (blockIdx.x == 0) {
        for (uint64_t i = threadIdx.x; i < head; i += kH16Threads) count_key(in[i]);
        for (uint64_t i = head + nvec * 4 + threadIdx.x; i < n; i += kH16Threads) count_key(in[i]);
    }
    __syncthreads();
    uint4* out4 = reinterpret_cast<uint4*>(dump + static_cast<uint64_t>(blockIdx.x) * 32768);
    const uint4* h4 = reinterpret_cast<const uint4*>(h16);
    for (int i = threadIdx.x; i < 32768 / 4; i += kH16Threads) out4[i] = h4[i];
}

// counts[d] = sum over the CTAs' dumps + the bins moved out early
__global__ void msd_reduce16_kernel(const uint32_t* __restrict__ dump, int ctas, const uint32_t* __restrict__ extra,
                                    uint32_t* __restrict__ counts) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x; // word = bins 2w, 2w+1
    if (w >= 32768) return;
    uint32_t lo = 0, hi = 0;
    for (int c = 0; c < ctas; ++c) {
        const uint32_t x = dump[static_cast<uint64_t>(c) * 32768 + w];
        lo += x & 0xFFFFu;
        hi += x >> 16;
    }
    counts[2 * w] = lo + extra[2 * w];
    counts[2 * w + 1] = hi + extra[2 * w + 1];
}

// ---------------------------------------------------------------------------
// H2: plan.  One CTA of 1024 threads, 64 bins each.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024)
    msd_plan_kernel(const uint32_t* __restrict__ counts, uint64_t n, MsdPlan* __restrict__ plan) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_max[32];
    __shared__ uint32_t s_seg[257];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint4* c4 = reinterpret_cast<const uint4*>(counts) + tid * 16;
    uint32_t sum = 0, mx = 0;
#pragma unroll 8
    for (int j = 0; j < 16; ++j) {
        const uint4 c = c4[j];
        sum += c.x + c.y + c.z + c.w;
        mx = max(max(mx, max(c.x, c.y)), max(c.z, c.w));
    }
    const uint32_t incl = warp_inclusive_scan(sum);
    uint32_t wm = mx;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wm = max(wm, __shfl_xor_sync(0xffffffffu, wm, o));
    if (lane == 31) s_warp[warp] = incl;
    if (lane == 0) s_max[warp] = wm;
    __syncthreads();
    uint32_t excl = incl - sum;
    for (int w = 0; w < warp; ++w) excl += s_warp[w];
    uint32_t run = excl;
    uint4* o4 = reinterpret_cast<uint4*>(plan->bucket_off) + tid * 16;
#pragma unroll 4
    for (int j = 0; j < 16; ++j) { // second read of the counts (L2 hits) instead of 64 live registers
        const uint4 c = c4[j];
        uint4 o;
        o.x = run, run += c.x;
        o.y = run, run += c.y;
        o.z = run, run += c.z;
        o.w = run, run += c.w;
        o4[j] = o;
    }
    // thread t starts bucket row t / 4 (256 bins per byte-3 value = 4 threads)
    if ((tid & 3) == 0) {
        plan->base1[tid >> 2] = excl;
        s_seg[tid >> 2] = excl;
    }
    if (tid == 1023) {
        plan->bucket_off[65536] = run;
        s_seg[256] = run;
    }
    __syncthreads();
    // MB's tiles: inside byte-3 bucket s tile j covers positions
    // [A + j * TILE, A + (j + 1) * TILE) of the bucket, A = its start rounded
    // down to 4 keys, so every tile but a bucket's first starts 16-byte aligned
    uint32_t tiles = 0;
    if (tid < 256) {
        const uint32_t s0 = s_seg[tid], s1 = s_seg[tid + 1];
        tiles = s1 > s0 ? (s1 - (s0 & ~3u) + kPartTile - 1) / kPartTile : 0u;
    }
    const uint32_t tincl = warp_inclusive_scan(tiles);
    __syncthreads();
    if (tid < 256 && lane == 31) s_warp[warp] = tincl;
    __syncthreads();
    if (tid < 256) {
        uint32_t texcl = tincl - tiles;
        for (int w = 0; w < warp; ++w) texcl += s_warp[w];
        plan->seg_tile_first[tid] = texcl;
        if (tid == 255) {
            plan->seg_tile_first[256] = texcl + tiles;
            plan->ntiles2 = texcl + tiles;
        }
    }
    if (tid == 0) {
        uint32_t m = 0;
        for (int w = 0; w < 32; ++w) m = max(m, s_max[w]);
        plan->max_bucket = m;
        const uint32_t ok = (m <= static_cast<uint32_t>(kMsdLocalCap) && static_cast<uint64_t>(s_seg[256]) == n) ? 1u : 0u;
        plan->ok = ok;
        plan->need_lsd = ok ? 0u : 1u;
    }
}

// ---------------------------------------------------------------------------
// MA / MB: partition by one byte, no order inside a digit run (the scheme of
// radix.cu's K3f).  SEG = false: the whole array by byte 3 (digit bases
// plan->base1, reservations reserve[256]).  SEG = true: inside each byte-3
// bucket by byte 2: tile t belongs to segment s with seg_tile_first[s] <= t <
// seg_tile_first[s+1]; digit bases bucket_off[s*256 + d], reservations
// reserve[s*256 + d].
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t head_words16(const uint32_t* p, uint32_t valid) {
    const uint32_t hw = (4u - static_cast<uint32_t>((reinterpret_cast<uintptr_t>(p) >> 2) & 3u)) & 3u;
    return hw < valid ? hw : valid;
}

struct PartSmem {
    static constexpr size_t in_off = 0;                                                // 2 x TILE u32
    static constexpr size_t cnt_off = in_off + sizeof(uint32_t) * 2 * kPartTile;      // 256 x 8 u32
    static constexpr size_t delta_off = cnt_off + sizeof(uint32_t) * 256 * kPartGroups; // 256 u32
    static constexpr size_t scan_off = delta_off + sizeof(uint32_t) * 256;            // 8 u32
    static constexpr size_t misc_off = scan_off + sizeof(uint32_t) * 8;               // per buffer: tile, start, valid, seg, head|body
    static constexpr size_t bar_off = misc_off + 64;                                   // 2 mbarriers
    static constexpr size_t bytes = bar_off + 16;
};

template <bool SEG>
__global__ void __launch_bounds__(kPartThreads, 2)
    msd_partition_kernel(const MsdPlan* __restrict__ plan, const uint32_t* __restrict__ src,
                         uint32_t* __restrict__ dst, uint64_t n, uint32_t* __restrict__ reserve,
                         uint32_t* __restrict__ tile_counter) {
    using L = PartSmem;
    constexpr int TILE = kPartTile;
    constexpr int ITEMS = kPartItems;
    constexpr int THREADS = kPartThreads;
    extern __shared__ __align__(128) uint8_t smem[];
    if (!plan->ok) return;
    uint32_t* s_in = reinterpret_cast<uint32_t*>(smem + L::in_off);
    uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem + L::cnt_off);
    uint32_t* s_delta = reinterpret_cast<uint32_t*>(smem + L::delta_off);
    uint32_t* s_scan = reinterpret_cast<uint32_t*>(smem + L::scan_off);
    uint32_t* s_misc = reinterpret_cast<uint32_t*>(smem + L::misc_off); // [b*8 + {tile, start, valid, seg, hb}]
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + L::bar_off);
    const uint32_t ntiles = SEG ? plan->ntiles2 : static_cast<uint32_t>((n + TILE - 1) / TILE);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr uint32_t SEL = SEG ? 0x4442u : 0x4443u; // byte 2 / byte 3

    // claim + describe + start the load of the next tile into buffer b (thread 0)
    auto claim = [&](int b) {
        const uint32_t tile = atomicAdd(tile_counter, 1u);
        s_misc[b * 8] = tile;
        if (tile >= ntiles) return;
        uint32_t start, valid, seg = 0;
        if constexpr (SEG) {
            int lo = 0, hi = 256; // last s with seg_tile_first[s] <= tile
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (plan->seg_tile_first[mid] <= tile) lo = mid;
                else hi = mid;
            }
            seg = static_cast<uint32_t>(lo);
            const uint32_t s0 = plan->bucket_off[seg * 256], s1 = plan->bucket_off[seg * 256 + 256];
            const uint32_t j = tile - plan->seg_tile_first[seg];
            const uint32_t a = (s0 & ~3u) + j * TILE; // tiles after the first start 16-byte aligned
            start = max(a, s0);
            valid = min(a + static_cast<uint32_t>(TILE), s1) - start;
        } else {
            start = tile * TILE;
            valid = static_cast<uint32_t>(min(static_cast<uint64_t>(TILE), n - start));
        }
        const uint32_t hw = head_words16(src + start, valid);
        const uint32_t body = (valid - hw) & ~3u;
        s_misc[b * 8 + 1] = start;
        s_misc[b * 8 + 2] = valid;
        s_misc[b * 8 + 3] = seg;
        s_misc[b * 8 + 4] = hw | (body << 2);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&s_bar[b], body * 4);
        if (body) tma_bulk_g2s(s_in + b * TILE, src + start + hw, body * 4, &s_bar[b]);
    };
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        fence_mbar_init();
        claim(0);
    }
    for (int i = tid; i < 256 * kPartGroups; i += THREADS) s_cnt[i] = 0;

    // cursor (d, q) byte offset: d * 32 + q * 4
    const uint32_t q4 = static_cast<uint32_t>(lane >> 2) * 4u;
    constexpr int CSH = SEG ? 11 : 19; // digit * 32 = (key >> CSH) & 0x1FE0
    auto cnt_off = [&](uint32_t key) {
        uint32_t o;
        asm("lop3.b32 %0, %1, 0x1FE0, %2, 0xEA;" : "=r"(o) : "r"(key >> CSH), "r"(q4)); // (a & b) | c
        return o;
    };
    uint8_t* cnt_base = smem + L::cnt_off;
    uint32_t parity = 0;
    uint32_t keys[ITEMS];
    for (uint32_t k = 0;; ++k) {
        const int cur = k & 1;
        __syncthreads(); // s_misc[cur] visible; the previous tile's buffer, cursors and deltas are free
        const uint32_t tile = s_misc[cur * 8];
        if (tile >= ntiles) break;
        if (tid == 0) claim(cur ^ 1);
        const uint32_t start = s_misc[cur * 8 + 1];
        const uint32_t valid = s_misc[cur * 8 + 2];
        const uint32_t seg = s_misc[cur * 8 + 3];
        const uint32_t hb = s_misc[cur * 8 + 4];
        const uint32_t hw = hb & 3u, body = hb >> 2;
        uint32_t* buf = s_in + cur * TILE;
        mbar_wait_parity(&s_bar[cur], (parity >> cur) & 1u);
        parity ^= 1u << cur;
        const bool fast = body == static_cast<uint32_t>(TILE);
        const uint32_t wbase = warp * (32 * ITEMS);
        // digit d = tid's first output position (needed after the ranking: loaded early)
        uint32_t dbase = 0;
        if (tid < 256) dbase = SEG ? plan->bucket_off[seg * 256 + tid] : static_cast<uint32_t>(plan->base1[tid]);

        // ---- load + count (cursors hold byte offsets) ----------------------
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
        uint32_t total = 0, excl = 0, reserved = 0;
        if (tid < 256) {
            uint4* row = reinterpret_cast<uint4*>(s_cnt + tid * kPartGroups);
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
            if (total) reserved = atomicAdd(&reserve[seg * 256 + tid], total >> 2);
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
            // output index (digit base) + reserved
            s_delta[tid] = dbase + reserved - (excl >> 2);
        }
        __syncthreads();
        if (tid < 256) {
            uint4* row = reinterpret_cast<uint4*>(s_cnt + tid * kPartGroups);
            row[0] = make_uint4(0, 0, 0, 0);
            row[1] = make_uint4(0, 0, 0, 0);
        }

        // ---- write digit runs (coalesced within each run) ------------------
        if (valid == static_cast<uint32_t>(TILE)) {
#pragma unroll
            for (int j = 0; j < ITEMS; ++j) {
                const uint32_t i = j * THREADS + tid;
                const uint32_t key = buf[i];
                dst[s_delta[__byte_perm(key, 0u, SEL)] + i] = key;
            }
        } else {
            for (uint32_t i = tid; i < valid; i += THREADS) {
                const uint32_t key = buf[i];
                dst[s_delta[__byte_perm(key, 0u, SEL)] + i] = key;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// MC: every top-16-bit bucket (<= kMsdLocalCap keys) sorted by its low 16
// bits.  tab[v >> 3] holds eight 4-bit counters (values 8w .. 8w+7); a key's
// atomic returns how many equal keys came before it; pre[w] = keys with
// values below 8w.  rank = pre + smaller values inside the word + equal keys
// before.  A 16th equal key would carry into the next counter: the bucket
// raises need_lsd and the LSD path re-sorts the untouched input.
// ---------------------------------------------------------------------------
// sum of the eight 4-bit fields of w, added to acc (3 logic ops + one DP4A)
__device__ __forceinline__ uint32_t nibble_sum_add(uint32_t w, uint32_t acc) {
    const uint32_t x = (w & 0x0F0F0F0Fu) + ((w >> 4) & 0x0F0F0F0Fu);
    return __dp4a(x, 0x01010101u, acc);
}

struct LocalSmem {
    static constexpr size_t tab_off = 0;                                         // 8192 u32
    static constexpr size_t pre_off = tab_off + sizeof(uint32_t) * 8192;         // 8192 u16
    static constexpr size_t stage_off = pre_off + sizeof(uint16_t) * 8192;       // kMsdLocalCap u32
    static constexpr size_t scan_off = stage_off + sizeof(uint32_t) * kMsdLocalCap; // 16 u32
    static constexpr size_t bytes = scan_off + 64;
};

__global__ void __launch_bounds__(kLocalThreads, BSG_MSD_LOCAL_CTAS)
    msd_local_sort_kernel(MsdPlan* __restrict__ plan, const uint32_t* __restrict__ src, uint32_t* __restrict__ dst) {
    using L = LocalSmem;
    constexpr int THREADS = kLocalThreads;
    constexpr int ITEMS = kLocalItems;
    static_assert(THREADS * ITEMS == kMsdLocalCap, "one bucket per CTA iteration");
    extern __shared__ __align__(16) uint8_t smem[];
    if (!plan->ok) return;
    uint32_t* tab = reinterpret_cast<uint32_t*>(smem + L::tab_off);
    uint16_t* pre = reinterpret_cast<uint16_t*>(smem + L::pre_off);
    uint32_t* stage = reinterpret_cast<uint32_t*>(smem + L::stage_off);
    uint32_t* s_scan = reinterpret_cast<uint32_t*>(smem + L::scan_off);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t overflow = 0;
    uint4* tab4 = reinterpret_cast<uint4*>(tab);
#pragma unroll
    for (int k = 0; k < 4; ++k) tab4[k * THREADS + tid] = make_uint4(0, 0, 0, 0);
    for (uint32_t b = blockIdx.x; b < 65536u; b += gridDim.x) {
        const uint32_t off = plan->bucket_off[b];
        const uint32_t m = plan->bucket_off[b + 1] - off;
        if (m == 0) continue;
        // rows of THREADS keys the bucket fills (whole rows are skipped by uniform branches)
        const int rows = static_cast<int>((m + THREADS - 1) / THREADS);
        // ---- load, count, rank among equal keys ----------------------------
        uint32_t keys[ITEMS];
        uint32_t dup[(ITEMS + 7) / 8] = {0, 0};
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            if (i < rows) {
                const uint32_t idx = i * THREADS + tid;
                keys[i] = idx < m ? __ldg(src + off + idx) : 0u;
            }
        }
        __syncthreads(); // the table is clear and the staging area free (previous bucket done)
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            if (i < rows) {
                const uint32_t idx = i * THREADS + tid;
                if (idx < m) {
                    const uint32_t v = keys[i] & 0xFFFFu;
                    const uint32_t sh = (v & 7u) * 4u;
                    const uint32_t old = (atomicAdd(&tab[v >> 3], 1u << sh) >> sh) & 15u;
                    overflow |= old + 1u; // bit 4 set = a 16th equal key
                    dup[i >> 3] |= old << ((i & 7) * 4);
                }
            }
        }
        __syncthreads();
        // ---- prefix over the table: thread t owns words [16t, 16t + 16) -----
        // (measured and dropped: plane-major ownership, rotated chunk loads and
        // a conflict-free physical layout all remove the 4-way bank conflicts
        // of these loads but cost registers -- the kernel is capped at 42 --
        // and instructions: 1.35-1.48 ms against 1.24)
        {
            const uint4* t4 = reinterpret_cast<const uint4*>(tab + tid * 16);
            uint32_t w[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 x = t4[q];
                w[q * 4] = x.x, w[q * 4 + 1] = x.y, w[q * 4 + 2] = x.z, w[q * 4 + 3] = x.w;
            }
            uint32_t p[17];
            p[0] = 0;
#pragma unroll
            for (int j = 0; j < 16; ++j) p[j + 1] = nibble_sum_add(w[j], p[j]);
            const uint32_t total = p[16];
            const uint32_t incl = warp_inclusive_scan(total);
            if (lane == 31) s_scan[warp] = incl;
            __syncthreads();
            uint32_t excl = incl - total;
#pragma unroll
            for (int ww = 0; ww < THREADS / 32; ++ww)
                if (ww < warp) excl += s_scan[ww];
            const uint32_t e2 = excl * 0x10001u; // both halves
            uint4* pre4 = reinterpret_cast<uint4*>(pre + tid * 16);
#pragma unroll
            for (int q = 0; q < 2; ++q)
                pre4[q] =
                    make_uint4((p[8 * q] | (p[8 * q + 1] << 16)) + e2, (p[8 * q + 2] | (p[8 * q + 3] << 16)) + e2,
                               (p[8 * q + 4] | (p[8 * q + 5] << 16)) + e2, (p[8 * q + 6] | (p[8 * q + 7] << 16)) + e2);
        }
        __syncthreads();
        // ---- rank and stage -------------------------------------------------
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            if (i < rows) {
                const uint32_t idx = i * THREADS + tid;
                if (idx < m) {
                    const uint32_t v = keys[i] & 0xFFFFu;
                    const uint32_t word = tab[v >> 3];
                    const uint32_t d4 = (dup[i >> 3] >> ((i & 7) * 4)) & 15u;
                    const uint32_t r = nibble_sum_add(word & ((1u << ((v & 7u) * 4u)) - 1u), pre[v >> 3] + d4);
                    stage[r < static_cast<uint32_t>(kMsdLocalCap) ? r : 0u] = keys[i];
                }
            }
        }
        __syncthreads();
        // ---- write the bucket; clear the table for the next one -------------
#pragma unroll
        for (int k = 0; k < 4; ++k) tab4[k * THREADS + tid] = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            if (i < rows) {
                const uint32_t idx = i * THREADS + tid;
                if (idx < m) dst[off + idx] = stage[idx];
            }
        }
        // (the barrier after the next bucket's loads orders these reads of the
        // staging area and the table stores before their next use)
    }
    if (overflow & 16u) atomicOr(&plan->need_lsd, 1u);
}

// 0 = auto (on for the sizes it was measured faster at), 1 = off, 2 = on for every n it can run at
int& msd_mode_ref() {
    static int mode = dev_knob("BSG_MSD", 0);
    return mode;
}

} // namespace

bool msd_sort_applies(const uint32_t* in, const uint32_t* out, uint64_t n) {
    const int mode = msd_mode_ref();
    if (mode == 1) return false;
    if (in == out) return false; // the fallback re-sorts the input: it must survive
    const uintptr_t a = reinterpret_cast<uintptr_t>(in), b = reinterpret_cast<uintptr_t>(out);
    if (a < b + n * 4 && b < a + n * 4) return false;
    if (mode == 2) return n >= 2 && n <= (uint64_t{1} << 29);
    return n > kMsdMinKeys && n <= kMsdMaxKeys;
}

size_t msd_workspace_bytes() {
    // [MsdPlan][counts 65536][extra 65536][reserve1 256][reserve2 65536][tile counters 64][dump ctas x 32768]
    return sizeof(MsdPlan) + sizeof(uint32_t) * (65536 * 3 + 256 + 64) +
           sizeof(uint32_t) * 32768 * static_cast<size_t>(kSmCountB200 + 8) + 256;
}

// Enqueues H1, H2, MA, MB, MC.  `tmp` holds n keys.  Returns launches or -1;
// *gate receives the device word the LSD fallback must test (nonzero = run).
int launch_msd_sort(const uint32_t* in, uint32_t* out, uint32_t* tmp, uint64_t n, void* workspace,
                    cudaStream_t stream, const uint32_t** gate) {
    uint8_t* w = static_cast<uint8_t*>(workspace);
    MsdPlan* plan = reinterpret_cast<MsdPlan*>(w);
    uint32_t* counts = reinterpret_cast<uint32_t*>(w + ((sizeof(MsdPlan) + 255) & ~size_t{255}));
    uint32_t* extra = counts + 65536;
    uint32_t* reserve1 = extra + 65536;
    uint32_t* reserve2 = reserve1 + 256;
    uint32_t* tile_ctr = reserve2 + 65536; // [0] level 1, [32] level 2
    uint32_t* dump = tile_ctr + 64;
    *gate = &plan->need_lsd;
    // extra .. tile counters are contiguous: one memset
    if (cudaMemsetAsync(extra, 0, sizeof(uint32_t) * (65536 + 256 + 65536 + 64), stream) != cudaSuccess) return -1;
    const int sms = current_sm_count();
    static PerDeviceOccupancy occ_h, occ_a, occ_b, occ_c;
    int launches = 0;
    {
        TimedScope ts(6 /*BSG_K_MSD_HIST*/, stream);
        (void)kernel_occupancy(occ_h, msd_hist16_kernel, kH16Threads, 32768 * 4);
        const int ctas = std::min(sms, kSmCountB200 + 8);
        msd_hist16_kernel<<<ctas, kH16Threads, 32768 * 4, stream>>>(in, n, dump, extra);
        msd_reduce16_kernel<<<32768 / 256, 256, 0, stream>>>(dump, ctas, extra, counts);
        msd_plan_kernel<<<1, 1024, 0, stream>>>(counts, n, plan);
        launches += 3;
    }
    {
        TimedScope ts(7 /*BSG_K_MSD_PARTITION*/, stream);
        const int pa = std::max(1, kernel_occupancy(occ_a, msd_partition_kernel<false>, kPartThreads, PartSmem::bytes));
        const int pb = std::max(1, kernel_occupancy(occ_b, msd_partition_kernel<true>, kPartThreads, PartSmem::bytes));
        const uint32_t tiles = static_cast<uint32_t>((n + kPartTile - 1) / kPartTile);
        msd_partition_kernel<false><<<std::min<uint32_t>(tiles, sms * pa), kPartThreads, PartSmem::bytes, stream>>>(
            plan, in, out, n, reserve1, tile_ctr);
        msd_partition_kernel<true><<<std::min<uint32_t>(tiles + 256, sms * pb), kPartThreads, PartSmem::bytes, stream>>>(
            plan, out, tmp, n, reserve2, tile_ctr + 32);
        launches += 2;
    }
    {
        TimedScope ts(8 /*BSG_K_MSD_LOCAL*/, stream);
        const int pc = std::max(1, kernel_occupancy(occ_c, msd_local_sort_kernel, kLocalThreads, LocalSmem::bytes));
        msd_local_sort_kernel<<<sms * pc, kLocalThreads, LocalSmem::bytes, stream>>>(plan, tmp, out);
        launches += 1;
    }
    if (cudaGetLastError() != cudaSuccess) return -1;
    return launches;
}

} // namespace bsg

// Test aid: 0 = auto, 1 = never, 2 = whenever it can run; returns the previous mode.
extern "C" int bsg_debug_set_msd(int mode) {
    const int prev = bsg::msd_mode_ref();
    if (mode >= 0) bsg::msd_mode_ref() = mode;
    return prev;
}
