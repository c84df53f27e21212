/*
 * bsg.h -- C ABI of the B200-native integer-sorting hot path of
 * arXiv 1708.09495 (Gerbessiotis, "Integer sorting on multicores").
 *
 * The reference (/root/reference/proj/include/bspsort/, header-only C++20)
 * exposes no FFI; its "operator API" is a set of C++ free functions taking
 * std::vector<uint32_t>.  Each entry point below replaces one of them (cited
 * file:line), with plain pointers and sizes.  The C++ mirror of the reference
 * signatures is include/bspsort_b200/bspsort.hpp (header-only, calls this ABI);
 * the Python mirror is paper_1708_09495_b200/ (ctypes).
 *
 * Conventions
 *  - Every function returns BSG_OK (0) or a positive status; the thread-local
 *    message of the last failure is bsg_last_error().  BSG_EINVAL plays the
 *    role of the reference's std::invalid_argument, BSG_EPROTO of bsp::bsp_error.
 *  - mem_kind BSG_MEM_DEVICE: in/out are device pointers on the context's GPU;
 *    the call only enqueues work on `stream` (a cudaStream_t, NULL = legacy
 *    default stream) and returns.  BSG_MEM_HOST: in/out are host pointers
 *    (pinned for full PCIe speed); the call copies in, sorts, copies out and
 *    synchronises `stream` before returning -- the reference's synchronous
 *    by-value semantics (radix.hpp:69, netsort.hpp:157).
 *  - in == out is allowed everywhere (in-place); partially overlapping device
 *    inputs/outputs (e.g. merge_split's low == a, or a padded intermediate
 *    network state written over its own input) are staged through the
 *    context's workspace first, so any aliasing gives the non-aliased result.
 *  - One context may be used from several streams: each call is ordered
 *    after the context's previous call (an event on the previous stream), as
 *    all calls share the context's device workspace.
 *  - Keys are uint32; counts and positions are 64-bit everywhere (n may
 *    exceed 2^32 on one GPU), fixing the reference's uint32 count blocks
 *    (radix.hpp:127-132) which wrap at 2^32 keys per worker.
 *  - There is no CPU fallback: without a usable GPU every compute entry point
 *    fails with BSG_ECUDA.
 */
#ifndef BSG_H_
#define BSG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSG_ABI_VERSION 2

enum bsg_status {
    BSG_OK = 0,
    BSG_EINVAL = 1, /* invalid argument (reference: std::invalid_argument) */
    BSG_EPROTO = 2, /* protocol / consistency failure (reference: bsp::bsp_error) */
    BSG_ECUDA = 3,  /* CUDA runtime error or no GPU */
    BSG_ENOMEM = 4, /* device or host allocation failed */
    BSG_ENCCL = 5   /* NCCL failure (group contexts, BSG_PR_NCCL) */
};

enum bsg_mem_kind { BSG_MEM_HOST = 0, BSG_MEM_DEVICE = 1 };

/* core.hpp:24 enum class Algorithm { SR4, PR4, PR2, BTN, OET } (same order) */
enum bsg_algorithm { BSG_SR4 = 0, BSG_PR4 = 1, BSG_PR2 = 2, BSG_BTN = 3, BSG_OET = 4 };

/* netsort.hpp: BTN = bitonic_schedule (70-89), OET = odd_even_rounds (95-108) */
enum bsg_network { BSG_NET_BTN = 0, BSG_NET_OET = 1 };

/* bsp.hpp:86-92 RunStats, synthesised with the reference semantics. */
typedef struct bsg_run_stats {
    int32_t supersteps;
    uint64_t messages_sent;
    uint64_t messages_delivered;
    uint64_t words_sent;
    uint64_t words_delivered;
} bsg_run_stats;

typedef struct bsg_ctx bsg_ctx;

/* ---- library / context ------------------------------------------------ */
int bsg_abi_version(void);
const char* bsg_last_error(void);
/* Number of kernel launches this context has enqueued since creation. */
uint64_t bsg_ctx_launch_count(const bsg_ctx* ctx);

/* Binds a context to CUDA device `device`.  The context owns the cached
 * device workspace (so no cudaMalloc happens on a warm path).  A context
 * serialises its calls internally; use one per host thread for concurrency. */
int bsg_ctx_create(int device, bsg_ctx** out);
int bsg_ctx_destroy(bsg_ctx* ctx);
/* Frees the context's cached device workspace (after its last queued call
 * completes); the context stays usable and re-allocates on demand. */
int bsg_ctx_release(bsg_ctx* ctx);
/* Pre-sizes the workspace for sorts of up to n keys (optional). */
int bsg_ctx_reserve(bsg_ctx* ctx, uint64_t n);

/* Kernel-level timing on the launching stream (CUDA events around every
 * launch of the given class while enabled).  Classes: */
enum bsg_kernel_class {
    BSG_K_ONESWEEP = 0, /* one stable digit pass (radix.cu K3) */
    BSG_K_HIST = 1,     /* digit histograms (radix.cu K1) */
    BSG_K_NETWORK = 2,  /* batched BTN/OET block network (netsort.cu) */
    BSG_K_PR = 3,       /* parallel-radix plan/rebuild kernels (pr.cu) */
    BSG_K_FIRST_PASS = 4, /* first pass of a full sort, no order inside a digit run (radix.cu K3f) */
    BSG_K_RELAXED_PASS = 5, /* pass k > 0 of a full sort, value-stable ranking (radix.cu K3r) */
    BSG_K_MSD_HIST = 6,      /* hybrid route: 16-bit histogram + plan (msd.cu H1/H2) */
    BSG_K_MSD_PARTITION = 7, /* hybrid route: the two unordered byte partitions (msd.cu MA/MB) */
    BSG_K_MSD_LOCAL = 8,     /* hybrid route: local sort of the top-16-bit buckets (msd.cu MC) */
    BSG_K_CLASSES = 9
};
int bsg_ctx_set_timing(bsg_ctx* ctx, int enable);
/* Synchronises the recorded events and returns the summed duration (ms) and
 * launch count of one class since timing was (re-)enabled. */
int bsg_ctx_get_timing(bsg_ctx* ctx, int kernel_class, double* total_ms, uint64_t* launches);

/* ---- host-side helpers (no GPU needed) -------------------------------- */
/* core.hpp:93-99 generate_uniform_keys: mt19937_64(seed), low 32 bits. */
int bsg_generate_uniform_u32(uint32_t* out, uint64_t n, uint64_t seed);
/* Draws [offset, offset + n) of the same stream (random access by
 * jump-ahead: x^offset mod the generator's characteristic polynomial). */
int bsg_generate_uniform_at_u32(uint32_t* out, uint64_t n, uint64_t seed, uint64_t offset);
/* bench.hpp:77-88 derive_seed (splitmix64). */
uint64_t bsg_derive_seed(uint64_t seed, int32_t rep);
/* core.hpp:60-64 digit_bits + radix.hpp:32-40 checked_digit_bits:
 * lg r for r in {2,4,16,256,65536}, else -1 (and sets the error message). */
int bsg_checked_digit_bits(uint64_t radix);
/* Builder-defined skewed inputs for config 3 (not in the
 * reference): kind 0 = uniform keys & 0xFFFF, 1 = Zipf(s) over ranks
 * 1..2^32 (key = rank-1) by rejection-inversion driven by mt19937_64(seed),
 * 2 = all keys 0xABCD1234 (acceptance.cpp:63). */
int bsg_generate_skewed_u32(uint32_t* out, uint64_t n, uint64_t seed, int kind, double zipf_s);
/* netsort.hpp:70-89 / 95-108: stage-major partner[s*p+i] (-1 = idle) and
 * keep_low[s*p+i]; *stages receives the stage count (only the first
 * cap_stages are written). */
int bsg_network_schedule(int network, int p, int32_t* partner, int32_t* keep_low, int cap_stages,
                         int* stages);
/* radix.hpp:96-118 detail::Partition */
uint64_t bsg_partition_size_of(uint64_t n, int p, int w);
uint64_t bsg_partition_offset_of(uint64_t n, int p, int w);
int bsg_partition_owner_of(uint64_t n, int p, uint64_t pos);

/* ---- sorts ------------------------------------------------------------ */
/* radix.hpp:69-90 serial_radix_sort(KeyArray, radix): 32/lg r stable
 * count-sort rounds (SR4 when r = 256).  Output is ascending.  Only the
 * final array is returned, as in the reference; the passes in between keep
 * the order by key VALUE that the next pass needs (K3f/K3r), not
 * positions among equal keys.  A round whose result is returned
 * (bsg_count_sort_round_u32, a rounds-limited bsg_parallel_radix_sort_u32, or
 * one that returns RunStats, whose count matrices depend on it) is strictly
 * stable. */
int bsg_radix_sort_u32(bsg_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n,
                       int radix_log2, int mem_kind, void* stream);

/* radix.hpp:44-65 count_sort_round(keys, round, radix): one stable pass
 * over digit `round` (low digit first).  radix_log2 in {1,2,4,8,16}. */
int bsg_count_sort_round_u32(bsg_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n,
                             int round, int radix_log2, int mem_kind, void* stream);

/* netsort.hpp:30-51 merge_split(a, b): low = |a| smallest of a U b, high =
 * |b| largest, both ascending; a and b must each be ascending. */
int bsg_merge_split_u32(bsg_ctx* ctx, const uint32_t* a, uint64_t na, const uint32_t* b,
                        uint64_t nb, uint32_t* low, uint32_t* high, int mem_kind, void* stream);

/* netsort.hpp:124-199 prepare_btn/prepare_oet + run_block_network over a
 * BATCH of independent arrays (the reference sorts one array per call;
 * SURVEY §8(b)).  in/out hold num_arrays consecutive arrays of `len` keys.
 * Each array is padded to p*ceil(len/p) with 0xFFFFFFFF, blocks are sorted
 * locally, then the network's merge-split stages run.  stages_limit < 0 runs
 * all stages and writes the stripped len keys per array; stages_limit >= 0
 * stops early and writes the padded p*ceil(len/p) block states per array
 * (out must then hold num_arrays*p*ceil(len/p) keys).  `stats` (optional)
 * receives one array's RunStats. */
int bsg_block_network_batched_u32(bsg_ctx* ctx, int network, const uint32_t* in, uint32_t* out,
                                  uint64_t num_arrays, uint32_t len, int p, int stages_limit,
                                  bsg_run_stats* stats, int mem_kind, void* stream);

/* radix.hpp:233-303 prepare_parallel_radix + run_parallel_radix (PR4 at
 * r=256, PR2 at r=65536) with p logical workers resident on the context's
 * GPU: per round a digit count per worker, the p x r count exchange, the
 * stable local pass, slice routing and the rebuild, all as kernels.
 * rounds_limit >= 0 stops after that many rounds (the reference's
 * plan.rounds override) -- the concatenated per-worker blocks are then the
 * intermediate state.  On a group context (bsg_ctx_create_group) the
 * workers are spread over the group's GPUs (BSG_PR_PEER rounds); in/out are
 * then host pointers (BSG_MEM_HOST) or device pointers on member 0's GPU.
 * Multi-GPU with one process per GPU runs the same steps through
 * paper_1708_09495_b200.distributed over torch.distributed / NCCL. */
int bsg_parallel_radix_sort_u32(bsg_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n,
                                int p, int radix_log2, int rounds_limit, bsg_run_stats* stats,
                                int mem_kind, void* stream);

/* bspsort.hpp:15-25 sort_instance: validate (core.hpp:74-88) + dispatch. */
int bsg_sort_instance_u32(bsg_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n,
                          int processors, int algorithm, uint64_t radix, int mem_kind,
                          void* stream);

/* ---- parallel-radix step kernels (one rank = one GPU) -------------------
 * The building blocks of one PR round on one worker, exported so a host
 * orchestrator (Python over torch.distributed / NCCL) can interleave them
 * with the collectives.  All pointers are device pointers, all calls are
 * asynchronous on `stream`.  Counts are uint64. */

/* radix.hpp:127-132 count_digits: counts[d] = #{keys in block with digit d}. */
int bsg_pr_count_digits(bsg_ctx* ctx, const uint32_t* block, uint64_t len, int round,
                        int radix_log2, uint64_t* counts, void* stream);

/* radix.hpp:137-179 digit_starts + the routing part of sort_and_scatter,
 * from the gathered count matrix counts[v*r + d] (p x r, device):
 *   send_counts[w] = #keys worker `me` sends to worker w,
 *   recv_counts[v] = #keys worker `me` receives from worker v,
 *   rebuild_delta[v*r + d] (int64) = where the keys of digit d received from
 *   v land in me's rebuilt block: out_index = rebuild_delta + index within
 *   the received (source-major) buffer.  Host-visible outputs are device
 *   arrays; copy send/recv counts back to size the exchange. */
int bsg_pr_plan(bsg_ctx* ctx, const uint64_t* counts, uint64_t n, int p, int me, int round,
                int radix_log2, uint64_t* send_counts, uint64_t* recv_counts,
                int64_t* rebuild_delta, void* stream);

/* radix.hpp:151-179 sort_and_scatter's local stable count-sort: sorted =
 * count_sort_round(block, round, radix).  Because global positions increase
 * along the digit-sorted block, the slice for worker w is the contiguous
 * range [sum(send_counts[<w]), +send_counts[w]) of `sorted` -- no per-key
 * owner_of division. */
int bsg_pr_local_sort(bsg_ctx* ctx, const uint32_t* block, uint32_t* sorted, uint64_t len,
                      int round, int radix_log2, void* stream);

/* Host (CPU) restatement of bsg_pr_plan over a host count matrix -- the
 * same routing arithmetic, for hosts that plan on the CPU and for
 * cross-checking the device planner.  No GPU needed. */
int bsg_pr_plan_host(const uint64_t* counts, uint64_t n, int p, int me, int radix_log2,
                     uint64_t* send_counts, uint64_t* recv_counts, int64_t* rebuild_delta);

/* radix.hpp:184-222 gather_slices: rebuilds the block from the source-major
 * receive buffer (recv_len keys) by scattering each key to
 * rebuild_delta[src*r + digit] + index. */
int bsg_pr_rebuild(bsg_ctx* ctx, const uint32_t* recv, uint64_t recv_len,
                   const uint64_t* recv_counts, int p, int round, int radix_log2,
                   const int64_t* rebuild_delta, uint32_t* block, void* stream);

/* Enables direct loads/stores from the context's device to every other
 * device that supports peer access (NVLink / NVSwitch), for the peer-memory
 * PR exchange.  Idempotent; devices without peer access are skipped.
 * *enabled (optional) receives the number of peers now accessible. */
int bsg_ctx_enable_peer_access(bsg_ctx* ctx, int* enabled);

/* Fused exchange + rebuild over peer memory (NVLink): replaces the
 * all-to-all-v of sort_and_scatter (radix.hpp:164-179) and gather_slices
 * (radix.hpp:184-222) for one round of worker `me`.  `sorted` is me's block
 * after its local stable pass (bsg_pr_local_sort), `counts_all` the gathered
 * p x r digit-count matrix (device).  Every key is stored directly at its
 * position in the next-round block of its owner: peer_blocks[w] (host array
 * of p device pointers, CUDA-IPC mapped for w != me) holds worker w's
 * Partition(n, p) block.  The caller orders the round with a barrier across
 * workers after this call (all stores land before any owner reads). */
int bsg_pr_peer_scatter(bsg_ctx* ctx, const uint32_t* sorted, uint64_t len,
                        const uint64_t* counts_all, uint64_t n, int p, int me,
                        int round, int radix_log2, uint32_t* const* peer_blocks,
                        void* stream);

/* One whole PR round of worker `me` as ONE pass (r <= 2^8): the local stable
 * pass of sort_and_scatter (radix.hpp:151-159) writes every key of `block`
 * (me's current block, len = size_of(me)) directly at its final position in
 * its owner's next-round block (peer_blocks as in bsg_pr_peer_scatter), i.e.
 * count_sort_round + all-to-all-v + gather_slices fused.  counts_all is the
 * gathered p x r count matrix of this round (bsg_pr_count_digits on every
 * worker).  For r = 2^16 the call runs bsg_pr_local_sort + the peer scatter.
 * Any block size at r >= 2^8 (blocks above 2^29 keys run 64-bit status words
 * and positions); r < 2^8 needs len <= 2^29 (BSG_EINVAL otherwise).
 * Same ordering contract as bsg_pr_peer_scatter. */
int bsg_pr_fused_round(bsg_ctx* ctx, const uint32_t* block, uint64_t len,
                       const uint64_t* counts_all, uint64_t n, int p, int me,
                       int round, int radix_log2, uint32_t* const* peer_blocks,
                       void* stream);

/* ---- multi-GPU parallel radix sort in ONE process ----
 * The reference runs run_parallel_radix's p workers as threads of one
 * process (radix.hpp:260-303, bsp.hpp:211-315); here a GROUP context spreads
 * the p logical workers over G GPUs of one node: member g (devices[g]) owns
 * the contiguous worker group Partition(p, G) block g, i.e. the key range
 * [bsg_group_range_offset(n,p,G,g), + bsg_group_range_size(n,p,G,g)).
 * Every round is the reference's round: digit counts per worker, the p x r
 * count matrix exchanged between members, then
 *   BSG_PR_PEER: ONE segmented one-sweep pass per member whose write-out
 *     stores every key at its global position in the owning member's
 *     next-round buffer over NVLink (peer access; count_sort_round +
 *     all-to-all-v + gather_slices fused), a cross-GPU event barrier per round;
 *   BSG_PR_NCCL: the stable local pass, an NCCL all-to-all-v of the
 *     contiguous slices (ncclSend/ncclRecv in one group, communicators from
 *     ncclCommInitAll owned by the context) and the rebuild; needs p == G.
 * Per-round states are bit-identical to run_parallel_radix with
 * plan.rounds = rounds_limit.  devices may repeat (several members on one
 * GPU: the same code path with local "peer" stores; NCCL needs distinct
 * devices). */
#define BSG_PR_PEER 0
#define BSG_PR_NCCL 1
int bsg_ctx_create_group(const int* devices, int ndevices, bsg_ctx** out);
/* members of a group context (1 for a single-device context) */
int bsg_ctx_group_size(const bsg_ctx* ctx);
/* the device of member g */
int bsg_ctx_group_device(const bsg_ctx* ctx, int member);
uint64_t bsg_group_range_offset(uint64_t n, int p, int G, int g);
uint64_t bsg_group_range_size(uint64_t n, int p, int G, int g);

/* Per-phase device time of one group sort, max over members (ms). */
typedef struct bsg_pr_timing {
    double total_ms;    /* the whole call (first kernel to last event) */
    double count_ms;    /* digit counts + count-matrix exchange */
    double exchange_ms; /* NCCL: the all-to-all-v; PEER: the fused pass (local pass + NVLink stores) */
    double local_ms;    /* NCCL: local stable pass + rebuild; PEER: 0 (inside the fused pass) */
    uint64_t remote_bytes; /* key bytes moved to another member, all rounds (from the count matrices) */
} bsg_pr_timing;

/* blocks[g]: device pointer on member g holding its key range (in/out, sorted
 * in place).  streams[g] (optional, cudaStream_t): work already queued there
 * (e.g. what produced blocks[g]) is ordered before the sort; NULL = every
 * member device is synchronised first.  Synchronous: returns when every
 * member is done.  stats / timing optional. */
int bsg_pr_group_sort_u32(bsg_ctx* group, uint32_t* const* blocks, uint64_t n, int p, int radix_log2,
                          int rounds_limit, int variant, bsg_run_stats* stats, bsg_pr_timing* timing,
                          void* const* streams);

/* core.hpp:93-99 generate_uniform_keys on the GPU: the same n keys,
 * bit-identical, written to device memory (`out`) on `stream`.  Segments of
 * the stream start from jump-ahead states; the first call per process
 * derives the generator's characteristic polynomial (host, ~0.1 s). */
int bsg_generate_uniform_device_u32(bsg_ctx* ctx, uint32_t* out, uint64_t n,
                                    uint64_t seed, void* stream);
/* Keys [offset, offset + n) of the same stream on the GPU (one jump-ahead of
 * the seeded state on the host, then as above): a rank's block of a
 * block-distributed generate_uniform_keys(N, seed) (config 5). */
int bsg_generate_uniform_device_at_u32(bsg_ctx* ctx, uint32_t* out, uint64_t n,
                                       uint64_t seed, uint64_t offset, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BSG_H_ */
