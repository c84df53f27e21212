// pr.cuh -- parallel radix sort (PR4 / PR2) step kernels and the in-process
// p-logical-worker orchestration (pr.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/bsg.h"

struct bsg_ctx;

namespace bsg {

// count_digits (radix.hpp:127-132) into uint64 counts[radix].
int launch_pr_count(bsg_ctx* ctx, const uint32_t* block, uint64_t len, int round, int bits, uint64_t* counts,
                    cudaStream_t stream);

// Routing plan of worker `me` from the p x r count matrix (radix.hpp:137-179).
// scratch: p(1 + c) + 2r + c uint64 words of device workspace, c = ceil(r /
// 1024) (split = the index in each source's sorted block where the slice for
// `me` begins, column totals, digit starts, chunk sums).
int launch_pr_plan(const uint64_t* counts, uint64_t n, int p, int me, int bits, uint64_t* send_counts,
                   uint64_t* recv_counts, int64_t* rebuild_delta, cudaStream_t stream, uint64_t* scratch);

// Protocol checks (bsp_error equivalent, radix.hpp:207-220 / 283-286): a flag
// word zeroed before a call's kernels and read back after them (one stream
// synchronisation) -> BSG_EPROTO; check_count_rows raises it when a row of an
// exchanged count matrix does not sum to its worker's block size.
int proto_begin(bsg_ctx* ctx, cudaStream_t st, uint32_t** flag);
int proto_end(bsg_ctx* ctx, cudaStream_t st, const char* what);
int check_count_rows(const uint64_t* counts, int p, int radix, uint64_t n, uint32_t* flag, cudaStream_t st);

// gather_slices (radix.hpp:184-222) as a stable scatter of the source-major
// receive buffer: block[delta[src][digit] + j] = recv[j].  Raises *proto
// (when given) if the received slices do not fill the block exactly; never
// stores outside [0, recv_len).
int launch_pr_rebuild(const uint32_t* recv, uint64_t recv_len, int bits, int shift, const int64_t* rebuild_delta,
                      uint32_t* block, cudaStream_t stream, const uint64_t* recv_counts, int p, uint32_t* proto);

// PR with p logical workers on the context's GPU.
int run_parallel_radix_local(bsg_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n, int p, int bits, int rounds,
                             bsg_run_stats* stats, cudaStream_t stream);

// Multi-GPU group (bsg_pr_group_sort_u32): p workers over the group's
// members; blocks[g] = member g's key range (device g), sorted in place.
int run_parallel_radix_group(bsg_ctx* grp, uint32_t* const* blocks, uint64_t n, int p, int bits, int rounds,
                             int variant, bsg_run_stats* stats, bsg_pr_timing* timing);
uint64_t group_range_offset(uint64_t n, int p, int G, int g);
void destroy_group_nccl(bsg_ctx* grp);

} // namespace bsg
