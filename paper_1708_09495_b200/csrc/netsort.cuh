// netsort.cuh -- launchers for the batched BTN/OET block networks and the
// standalone merge_split (netsort.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bsg {

// Largest padded array (p * ceil(len/p) keys) a CTA keeps resident in
// shared memory (two ping-pong copies: 2 x 64 KiB).
constexpr uint64_t kNetMaxPadded = 16384;

// network: 0 = BTN, 1 = OET.  run_stages merge-split stages are executed;
// full => write the stripped len keys per array, else the padded states.
int launch_block_network(int network, const uint32_t* in, uint32_t* out, uint64_t num_arrays, uint32_t len, int p,
                         int run_stages, bool full, cudaStream_t stream);

// One merge-split stage of a global-memory block network (arrays larger than
// kNetMaxPadded): src/dst hold p blocks of L keys.
int launch_net_stage(const uint32_t* src, uint32_t* dst, int p, uint32_t L, int network, int s, cudaStream_t stream);

// netsort.hpp:30-51 merge_split on device arrays.
int launch_merge_split(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb, uint32_t* low, uint32_t* high,
                       cudaStream_t stream);

} // namespace bsg
