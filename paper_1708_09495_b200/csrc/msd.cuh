// msd.cuh -- hybrid MSD / local-sort route of full keys-only sorts (msd.cu).
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace bsg {

constexpr int kMsdLocalCap = 6144;                        // keys a top-16-bit bucket may hold
// Auto mode takes the route where it measured >= 5% faster than the LSD sort
// on uniform keys (1.125 x 2^28: -5.0%, 1.25 x 2^28: -8.8%; at 2^28 -3.5%, at
// 0.875 x 2^28 equal, at 0.75 x 2^28 +6.8%: a bucket's fixed cost -- clearing
// and scanning its 32 KB table -- is spread over fewer keys) and the largest
// bucket of a uniform input stays under kMsdLocalCap (a declined plan costs
// the 16-bit histogram: +8% at 1.5 x 2^28).
constexpr uint64_t kMsdMinKeys = (uint64_t{1} << 28) + (uint64_t{1} << 24);                        // 1.0625 x 2^28 < n
constexpr uint64_t kMsdMaxKeys = (uint64_t{1} << 28) + (uint64_t{1} << 26) + (uint64_t{1} << 24); // n <= 1.3125 x 2^28

// Device-resident plan of one hybrid sort.
struct MsdPlan {
    uint32_t ok;         // every bucket fits the local sort: MA, MB, MC run
    uint32_t need_lsd;   // the LSD path must (re-)sort the input: !ok, or MC met > 15 equal keys
    uint32_t ntiles2;    // tiles of MB
    uint32_t max_bucket;
    uint64_t base1[256];          // first output position of every byte-3 value
    uint32_t seg_tile_first[260]; // MB: first tile of every byte-3 bucket, [256] = ntiles2
    uint32_t bucket_off[65540];   // first position of every top-16-bit bucket, [65536] = n
};

// The route is tried for this call (size window, disjoint in/out).
bool msd_sort_applies(const uint32_t* in, const uint32_t* out, uint64_t n);
size_t msd_workspace_bytes();
// Enqueues the route (in -> out through tmp).  *gate = device word that is
// nonzero when the LSD sort must run afterwards.  Returns launches or -1.
int launch_msd_sort(const uint32_t* in, uint32_t* out, uint32_t* tmp, uint64_t n, void* workspace,
                    cudaStream_t stream, const uint32_t** gate);

} // namespace bsg
