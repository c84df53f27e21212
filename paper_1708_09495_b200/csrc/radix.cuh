// radix.cuh -- host-side launchers for the LSD radix kernels (radix.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bsg {

constexpr int kMaxPasses = 8;

// Device-resident plan of one sort: which digit passes execute and where each
// reads and writes.  Built on the device from the histograms (identity passes,
// where one digit value holds all n keys, are skipped without a host sync).
struct PassPlan {
    const uint32_t* src[kMaxPasses];
    uint32_t* dst[kMaxPasses];
    int32_t active[kMaxPasses];
    int32_t skew[kMaxPasses];  // a digit holds > n/16 keys: contention-free ranking path
    int32_t executed;          // number of active passes
    int32_t need_copy;         // result is not in `out` yet
    const uint32_t* final_buf; // buffer holding the result after the last pass
};

// Tile geometry of the one-sweep pass.
constexpr int kOnesweepThreads = 512;
constexpr int kOnesweepItems = 16;
constexpr int kOnesweepTile = kOnesweepThreads * kOnesweepItems; // 8192 keys
// Keys per look-back chunk: status words hold a 30-bit count.
constexpr uint64_t kChunkKeys = uint64_t{1} << 29;

struct RadixWorkspace {
    uint32_t* tmp = nullptr;     // ping-pong buffer, >= n keys
    uint32_t* status = nullptr;  // look-back status words + tile counters
    uint32_t* hist = nullptr;    // [chunks][passes][256]
    uint64_t* base = nullptr;    // [chunks][passes][256]
    PassPlan* plan = nullptr;
};

// Bytes of look-back status needed for one pass over min(n, kChunkKeys) keys.
uint64_t onesweep_status_words(uint64_t n);

// Full LSD sort of n keys with 8-bit passes over bits [0, 8*passes).
// Returns the number of kernel launches enqueued, or -1 on launch error.
// gate: optional device word; when it reads 0 at run time the whole sort is
// skipped on the device (another route already wrote `out`, msd.cu).
int launch_radix_sort8(const uint32_t* in, uint32_t* out, uint64_t n, const RadixWorkspace& ws,
                       cudaStream_t stream, bool allow_tma, const uint32_t* gate = nullptr);

// `passes` stable byte passes starting at byte `first_byte` with one
// histogram read and one plan (passes = 2, first_byte = 2*round: one r = 2^16
// count-sort round).  Returns launches or -1.
int launch_byte_passes(const uint32_t* in, uint32_t* out, uint64_t n, int first_byte, int passes,
                       const RadixWorkspace& ws, cudaStream_t stream, bool allow_tma, const uint32_t* gate = nullptr);

// One stable count-sort pass over the `bits`-wide digit at bit `shift`
// (bits in {1,2,4,8}).  Returns launches enqueued or -1.
int launch_count_pass(const uint32_t* in, uint32_t* out, uint64_t n, int bits, int shift,
                      const RadixWorkspace& ws, cudaStream_t stream, bool allow_tma);

// Digit histogram of one `bits`-wide digit into 64-bit counts (PR count_digits).
int launch_digit_counts(const uint32_t* in, uint64_t n, int bits, int shift, uint64_t* counts,
                        uint32_t* scratch32, cudaStream_t stream);

// Next-round blocks of all PR workers as seen from this process (own block
// local, others CUDA-IPC mapped over NVLink) and their Partition offsets.
constexpr int kPeerMax = 64;
struct PeerTable {
    uint32_t* blocks[kPeerMax];
    uint64_t offset[kPeerMax + 1]; // Partition(n, p).offset_of(w); offset[p] = n
};

// One PR round fused with its exchange (r <= 2^8): a one-sweep pass over the
// worker's block whose digit bases are the global positions of the block's
// first key per digit (digit_base, device [radix]); every key is stored at
// its final position in its owner's block.  len <= kChunkKeys.
// The stable pass of all p worker blocks (Partition(n, p)) of an in-process
// PR round in ONE launch: key i of block w with digit d goes to
// base_table[w][d] + (its rank among block w's digit-d keys).  Returns
// launches (0 or 1) or -1.
// skew: device flag (0 = no digit holds > 1/16 of a block: count-then-rank
// path); nullptr = always rank first.
// full_run: the pass is round shift / bits of a full PR run from round 0 whose
// intermediate states are not returned (value-stable ranking allowed).
int launch_onesweep_seg(const uint32_t* src, uint32_t* dst, uint64_t n, int p, int bits, int shift,
                        const uint64_t* base_table, uint32_t* status, cudaStream_t stream,
                        const uint32_t* skew = nullptr, bool full_run = false);
uint64_t onesweep_seg_status_words(uint64_t n, int p);

// launch_onesweep_seg whose write-out stores key position g into
// tab.blocks[m][g - tab.offset[m]] of the member m owning g (G members,
// tab.offset[G] = n_total): one multi-GPU group member's PR round.
int launch_onesweep_seg_peer(const uint32_t* src, uint64_t n, int p, int bits, int shift, const uint64_t* base_table,
                             uint32_t* status, cudaStream_t stream, const uint32_t* skew, const PeerTable& tab, int G,
                             uint64_t n_total);

int launch_onesweep_peer(const uint32_t* block, uint64_t len, int bits, int shift, const uint64_t* digit_base,
                         uint32_t* status, const PeerTable& tab, int p, cudaStream_t stream,
                         const uint32_t* skew, uint64_t n_total);

} // namespace bsg
