// api.cu -- C ABI implementation (include/bsg.h): contexts, workspace, the
// host<->device staging of BSG_MEM_HOST calls, argument validation with the
// reference's error behaviour, and dispatch to the kernels.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>
#include "msd.cuh"
#include "context.cuh"
#include "netsort.cuh"
#include "pr.cuh"
#include "radix.cuh"

namespace bsg {

static thread_local std::string g_last_error;
thread_local KTimer* tl_timer = nullptr;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int status, const std::string& msg) {
    g_last_error = msg;
    return status;
}
int cuda_fail(cudaError_t e, const char* what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return e == cudaErrorMemoryAllocation ? BSG_ENOMEM : BSG_ECUDA;
}

} // namespace bsg

using namespace bsg;

int bsg_ctx::radix_ws(uint64_t n, RadixWorkspace* ws) {
    const uint64_t chunks = n ? (n + kChunkKeys - 1) / kChunkKeys : 1;
    cudaError_t e;
    if ((e = tmp.ensure(std::max<uint64_t>(n, 4) * sizeof(uint32_t))) != cudaSuccess) return cuda_fail(e, "workspace tmp");
    if ((e = status.ensure(onesweep_status_words(std::max<uint64_t>(n, 1)) * sizeof(uint32_t))) != cudaSuccess)
        return cuda_fail(e, "workspace status");
    if ((e = hist.ensure(chunks * kMaxPasses * 256 * sizeof(uint32_t))) != cudaSuccess) return cuda_fail(e, "workspace hist");
    if ((e = base.ensure(chunks * kMaxPasses * 256 * sizeof(uint64_t))) != cudaSuccess) return cuda_fail(e, "workspace base");
    if ((e = plan.ensure(sizeof(PassPlan))) != cudaSuccess) return cuda_fail(e, "workspace plan");
    ws->tmp = tmp.as<uint32_t>();
    ws->status = status.as<uint32_t>();
    ws->hist = hist.as<uint32_t>();
    ws->base = base.as<uint64_t>();
    ws->plan = plan.as<PassPlan>();
    return BSG_OK;
}

namespace {

// Serialises the context's calls, selects its device, binds its kernel timer
// and brackets the call in an NVTX range named after the entry point (a no-op
// unless a tool such as nsys or ncu --nvtx is attached).
struct CallGuard {
    std::lock_guard<std::mutex> lock;
    DeviceGuard dev;
    CallGuard(bsg_ctx* c, const char* entry) : lock(c->mu), dev(c->device) {
        tl_timer = &c->timer;
        nvtxRangePushA(entry);
    }
    ~CallGuard() {
        nvtxRangePop();
        tl_timer = nullptr;
    }
};

int check_ctx(bsg_ctx* ctx) {
    if (!ctx) return fail(BSG_EINVAL, "null context");
    return BSG_OK;
}

// Runs `body(d_in, d_out, stream)` with device buffers.  For HOST memory the
// keys are staged through the context's device buffers (H2D, body, D2H) and
// the stream is synchronised before returning.
template <class Body>
int with_device_io(bsg_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n_in, uint64_t n_out, int mem_kind,
                   cudaStream_t stream, Body&& body) {
    if (mem_kind == BSG_MEM_DEVICE) return body(in, out, stream);
    if (mem_kind != BSG_MEM_HOST) return fail(BSG_EINVAL, "mem_kind must be BSG_MEM_HOST or BSG_MEM_DEVICE");
    cudaError_t e;
    if ((e = ctx->stage_in.ensure(std::max<uint64_t>(n_in, 4) * 4)) != cudaSuccess) return cuda_fail(e, "host staging");
    if ((e = ctx->stage_out.ensure(std::max<uint64_t>(n_out, 4) * 4)) != cudaSuccess) return cuda_fail(e, "host staging");
    uint32_t* d_in = ctx->stage_in.as<uint32_t>();
    uint32_t* d_out = ctx->stage_out.as<uint32_t>();
    if (n_in)
        if (int rc = copy_h2d(ctx, d_in, in, n_in * 4, stream)) return rc;
    int rc = body(d_in, d_out, stream);
    if (rc != BSG_OK) return rc;
    if (n_out)
        if (int rc2 = copy_d2h(ctx, out, d_out, n_out * 4, stream)) return rc2;
    if ((e = cudaStreamSynchronize(stream)) != cudaSuccess) return cuda_fail(e, "stream synchronize");
    return BSG_OK;
}

bool ranges_overlap(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb) {
    if (!na || !nb) return false;
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
    return a0 < b0 + nb * 4 && b0 < a0 + na * 4;
}

int radix_bits_or_fail(int radix_log2) {
    if (radix_log2 != 1 && radix_log2 != 2 && radix_log2 != 4 && radix_log2 != 8 && radix_log2 != 16) {
        if (radix_log2 > 16 && radix_log2 <= 32 && 32 % radix_log2 == 0)
            return fail(BSG_EINVAL, "radix 2^" + std::to_string(radix_log2) +
                                         " needs a count array larger than memory; use r <= 65536");
        return fail(BSG_EINVAL, "radix must be a power of two whose bit width divides 32");
    }
    return BSG_OK;
}

// bsg_parallel_radix_sort_u32 on a group context: the member ranges are
// staged from host memory (BSG_MEM_HOST) or from device memory on member 0's
// GPU (BSG_MEM_DEVICE, peer copies), sorted by the group (BSG_PR_PEER rounds,
// or NCCL when the members lack peer access and p equals the group size),
// and copied back.  Synchronous.
int parallel_radix_sort_group(bsg_ctx* grp, const uint32_t* in, uint32_t* out, uint64_t n, int p, int bits,
                              int rounds, bsg_run_stats* stats, int mem_kind, cudaStream_t caller) {
    if (mem_kind != BSG_MEM_HOST && mem_kind != BSG_MEM_DEVICE)
        return fail(BSG_EINVAL, "mem_kind must be BSG_MEM_HOST or BSG_MEM_DEVICE");
    std::lock_guard<std::mutex> lock(grp->mu);
    const int G = static_cast<int>(grp->members.size());
    std::vector<uint32_t*> blocks(G);
    cudaError_t e;
    if (mem_kind == BSG_MEM_DEVICE) { // caller's work on `in` happens before the staging copies
        DeviceGuard dg(grp->device);
        if ((e = cudaStreamSynchronize(caller)) != cudaSuccess) return cuda_fail(e, "group staging");
    }
    for (int g = 0; g < G; ++g) {
        bsg_ctx* m = grp->members[g];
        DeviceGuard dg(m->device);
        const uint64_t off = group_range_offset(n, p, G, g), len = group_range_offset(n, p, G, g + 1) - off;
        if ((e = m->grp_cur.ensure(std::max<uint64_t>(len, 4) * 4)) != cudaSuccess) return cuda_fail(e, "group staging");
        blocks[g] = m->grp_cur.as<uint32_t>();
        if (len && mem_kind == BSG_MEM_HOST) {
            if (int rc = copy_h2d(m, blocks[g], in + off, len * 4, grp->member_streams[g])) return rc;
        } else if (len && (e = cudaMemcpyAsync(blocks[g], in + off, len * 4, cudaMemcpyDefault,
                                               grp->member_streams[g])) != cudaSuccess) {
            return cuda_fail(e, "group staging");
        }
    }
    const int variant = grp->peer_ok || p != G ? BSG_PR_PEER : BSG_PR_NCCL;
    if (int rc = run_parallel_radix_group(grp, blocks.data(), n, p, bits, rounds, variant, stats, nullptr)) return rc;
    for (int g = 0; g < G; ++g) {
        bsg_ctx* m = grp->members[g];
        DeviceGuard dg(m->device);
        const uint64_t off = group_range_offset(n, p, G, g), len = group_range_offset(n, p, G, g + 1) - off;
        if (len && mem_kind == BSG_MEM_HOST) {
            if (int rc = copy_d2h(m, out + off, blocks[g], len * 4, grp->member_streams[g])) return rc;
        } else if (len && (e = cudaMemcpyAsync(out + off, blocks[g], len * 4, cudaMemcpyDefault,
                                               grp->member_streams[g])) != cudaSuccess) {
            return cuda_fail(e, "group copy out");
        }
    }
    for (int g = 0; g < G; ++g) {
        DeviceGuard dg(grp->members[g]->device);
        if ((e = cudaStreamSynchronize(grp->member_streams[g])) != cudaSuccess) return cuda_fail(e, "group copy out");
    }
    return BSG_OK;
}

} // namespace

extern "C" {

int bsg_abi_version(void) { return BSG_ABI_VERSION; }
const char* bsg_last_error(void) { return g_last_error.c_str(); }
uint64_t bsg_ctx_launch_count(const bsg_ctx* ctx) { return ctx ? ctx->launches : 0; }

int bsg_ctx_create(int device, bsg_ctx** out) {
    if (!out) return fail(BSG_EINVAL, "null output pointer");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount (no usable GPU; there is no CPU fallback)");
    if (device < 0 || device >= count) return fail(BSG_EINVAL, "device index out of range");
    DeviceGuard g(device);
    if (g.err != cudaSuccess) return cuda_fail(g.err, "cudaSetDevice");
    cudaDeviceProp prop;
    if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
    if (prop.major != 10) return fail(BSG_ECUDA, std::string("kernels are built for sm_100a; device is ") + prop.name);
    auto* c = new (std::nothrow) bsg_ctx();
    if (!c) return fail(BSG_ENOMEM, "context allocation");
    c->device = device;
    *out = c;
    return BSG_OK;
}

int bsg_ctx_release(bsg_ctx* ctx) {
    if (int rc = check_ctx(ctx)) return rc;
    for (bsg_ctx* m : ctx->members)
        if (int rc = bsg_ctx_release(m)) return rc;
    CallGuard g(ctx, __func__);
    if (ctx->used && ctx->last_use) {
        const cudaError_t e = cudaEventSynchronize(ctx->last_use);
        if (e != cudaSuccess) return cuda_fail(e, "ctx release");
    }
    for (DevBuf* b : {&ctx->tmp, &ctx->status, &ctx->hist, &ctx->base, &ctx->plan, &ctx->stage_in, &ctx->stage_out,
                      &ctx->stage_b, &ctx->pr_counts, &ctx->pr_sorted, &ctx->pr_recv, &ctx->pr_block, &ctx->pr_misc,
                      &ctx->pr_delta, &ctx->net_sched, &ctx->cnt32, &ctx->proto, &ctx->mt_ws, &ctx->msd_ws, &ctx->grp_cur,
                      &ctx->grp_nxt, &ctx->grp_recv})
        b->release();
    return BSG_OK;
}

int bsg_ctx_destroy(bsg_ctx* ctx) {
    if (!ctx) return BSG_OK;
    if (!ctx->members.empty()) {
        destroy_group_nccl(ctx);
        for (size_t g = 0; g < ctx->members.size(); ++g) {
            DeviceGuard dg(ctx->members[g]->device);
            if (ctx->member_streams[g]) cudaStreamDestroy(ctx->member_streams[g]);
            for (DevBuf* b : {&ctx->members[g]->grp_cur, &ctx->members[g]->grp_nxt, &ctx->members[g]->grp_recv})
                b->release();
        }
        for (bsg_ctx* m : ctx->members) bsg_ctx_destroy(m);
        ctx->members.clear();
        ctx->member_streams.clear();
    }
    {
        CallGuard g(ctx, __func__);
        for (DevBuf* b : {&ctx->tmp, &ctx->status, &ctx->hist, &ctx->base, &ctx->plan, &ctx->stage_in, &ctx->stage_out,
                          &ctx->stage_b, &ctx->pr_counts, &ctx->pr_sorted, &ctx->pr_recv, &ctx->pr_block, &ctx->pr_misc,
                          &ctx->pr_delta, &ctx->net_sched, &ctx->cnt32, &ctx->proto, &ctx->mt_ws, &ctx->msd_ws})
            b->release();
        if (ctx->last_use) cudaEventDestroy(ctx->last_use);
        release_stage(ctx);
    }
    delete ctx;
    return BSG_OK;
}

int bsg_ctx_create_group(const int* devices, int ndevices, bsg_ctx** out) {
    if (!out) return fail(BSG_EINVAL, "null output pointer");
    *out = nullptr;
    if (!devices || ndevices < 1 || ndevices > kPeerMax) return fail(BSG_EINVAL, "group: 1..64 member devices");
    bsg_ctx* grp = nullptr;
    if (int rc = bsg_ctx_create(devices[0], &grp)) return rc;
    for (int g = 0; g < ndevices; ++g) {
        bsg_ctx* m = nullptr;
        int rc = bsg_ctx_create(devices[g], &m);
        cudaStream_t s = nullptr;
        if (rc == BSG_OK) {
            DeviceGuard dg(devices[g]);
            cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
            if (e != cudaSuccess) rc = cuda_fail(e, "group stream");
        }
        if (rc != BSG_OK) {
            if (m) bsg_ctx_destroy(m);
            bsg_ctx_destroy(grp);
            return rc;
        }
        grp->members.push_back(m);
        grp->member_streams.push_back(s);
    }
    // NVLink peer access between every pair of distinct member devices
    for (int a = 0; a < ndevices && grp->peer_ok; ++a)
        for (int b = 0; b < ndevices; ++b) {
            if (devices[a] == devices[b]) continue;
            int can = 0;
            if (cudaDeviceCanAccessPeer(&can, devices[a], devices[b]) != cudaSuccess || !can) {
                grp->peer_ok = false;
                break;
            }
            DeviceGuard dg(devices[a]);
            cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) {
                cudaGetLastError();
                e = cudaSuccess;
            }
            if (e != cudaSuccess) {
                cudaGetLastError();
                grp->peer_ok = false;
                break;
            }
        }
    *out = grp;
    return BSG_OK;
}

int bsg_ctx_group_size(const bsg_ctx* ctx) {
    if (!ctx) return 0;
    return ctx->members.empty() ? 1 : static_cast<int>(ctx->members.size());
}

int bsg_ctx_group_device(const bsg_ctx* ctx, int member) {
    if (!ctx || member < 0 || member >= bsg_ctx_group_size(ctx)) return -1;
    return ctx->members.empty() ? ctx->device : ctx->members[member]->device;
}

int bsg_ctx_set_timing(bsg_ctx* ctx, int enable) {
    if (int rc = check_ctx(ctx)) return rc;
    CallGuard g(ctx, __func__);
    ctx->timer.reset();
    ctx->timer.enabled = enable != 0;
    return BSG_OK;
}

int bsg_ctx_get_timing(bsg_ctx* ctx, int kernel_class, double* total_ms, uint64_t* launches) {
    if (int rc = check_ctx(ctx)) return rc;
    if (kernel_class < 0 || kernel_class >= BSG_K_CLASSES) return fail(BSG_EINVAL, "unknown kernel class");
    CallGuard g(ctx, __func__);
    double ms = 0;
    uint64_t cnt = 0;
    for (auto& r : ctx->timer.recs) {
        if (r.cls != kernel_class) continue;
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e != cudaSuccess) return cuda_fail(e, "timing event");
        float f = 0;
        cudaEventElapsedTime(&f, r.a, r.b);
        ms += f;
        ++cnt;
    }
    if (total_ms) *total_ms = ms;
    if (launches) *launches = cnt;
    return BSG_OK;
}

int bsg_ctx_reserve(bsg_ctx* ctx, uint64_t n) {
    if (int rc = check_ctx(ctx)) return rc;
    CallGuard g(ctx, __func__);
    RadixWorkspace ws;
    return ctx->radix_ws(n, &ws);
}

int bsg_radix_sort_u32(bsg_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n, int radix_log2, int mem_kind,
                       void* stream) {
    if (int rc = check_ctx(ctx)) return rc;
    if (int rc = radix_bits_or_fail(radix_log2)) return rc;
    if (n && (!in || !out)) return fail(BSG_EINVAL, "null key pointer");
    CallGuard g(ctx, __func__);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder order(ctx, st);
    return with_device_io(ctx, in, out, n, n, mem_kind, st, [&](const uint32_t* d_in, uint32_t* d_out, cudaStream_t s) -> int {
        RadixWorkspace ws;
        if (int rc = ctx->radix_ws(n, &ws)) return rc;
        // Any digit width yields the same stable LSD result (the output of
        // serial_radix_sort is independent of r); 8-bit passes are used for
        // lg r <= 8.  r = 2^16 runs each 16-bit round as two stable 8-bit
        // sub-passes (low byte then high byte of the digit), which is
        // bit-identical to count_sort_round(., round, 65536).
        // Large inputs first try the hybrid route (msd.cu); the LSD sort
        // below then runs only if that route's device-side plan declined or
        // its local sort gave up (gate word), re-sorting the untouched input.
        const uint32_t* gate = nullptr;
        if (msd_sort_applies(d_in, d_out, n)) {
            cudaError_t e = ctx->msd_ws.ensure(msd_workspace_bytes());
            if (e != cudaSuccess) return cuda_fail(e, "workspace msd");
            const int lm = launch_msd_sort(d_in, d_out, ws.tmp, n, ctx->msd_ws.ptr, s, &gate);
            if (lm < 0) return cuda_fail(cudaGetLastError(), "hybrid sort launch");
            ctx->launches += static_cast<uint64_t>(lm);
        }
        const int l = launch_radix_sort8(d_in, d_out, n, ws, s, true, gate);
        if (l < 0) return cuda_fail(cudaGetLastError(), "radix sort launch");
        ctx->launches += static_cast<uint64_t>(l);
        return BSG_OK;
    });
}

int bsg_count_sort_round_u32(bsg_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n, int round, int radix_log2,
                             int mem_kind, void* stream) {
    if (int rc = check_ctx(ctx)) return rc;
    if (int rc = radix_bits_or_fail(radix_log2)) return rc;
    const int rounds = 32 / radix_log2;
    if (round < 0 || round >= rounds)
        return fail(BSG_EINVAL, "round " + std::to_string(round) + " outside [0, " + std::to_string(rounds) + ")");
    if (n && (!in || !out)) return fail(BSG_EINVAL, "null key pointer");
    CallGuard g(ctx, __func__);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder order(ctx, st);
    return with_device_io(ctx, in, out, n, n, mem_kind, st, [&](const uint32_t* d_in, uint32_t* d_out, cudaStream_t s) -> int {
        RadixWorkspace ws;
        if (int rc = ctx->radix_ws(n, &ws)) return rc;
        int l = 0;
        if (radix_log2 <= 8) {
            l = launch_count_pass(d_in, d_out, n, radix_log2, round * radix_log2, ws, s, true);
        } else {
            // K4: one r = 2^16 round = a stable pass on the digit's low byte,
            // then on its high byte (stable LSD within the digit), both byte
            // histograms from ONE read of the input: 4 + 8 + 8 B/key
            l = launch_byte_passes(d_in, d_out, n, 2 * round, 2, ws, s, true);
        }
        if (l < 0) return cuda_fail(cudaGetLastError(), "count-sort round launch");
        ctx->launches += static_cast<uint64_t>(l);
        return BSG_OK;
    });
}

int bsg_merge_split_u32(bsg_ctx* ctx, const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb, uint32_t* low,
                        uint32_t* high, int mem_kind, void* stream) {
    if (int rc = check_ctx(ctx)) return rc;
    if ((na && (!a || !low)) || (nb && (!b || !high))) return fail(BSG_EINVAL, "null key pointer");
    if (na + nb >= (uint64_t{1} << 31)) return fail(BSG_EINVAL, "merge_split: |a|+|b| must be < 2^31");
    CallGuard g(ctx, __func__);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder order(ctx, st);
    if (mem_kind == BSG_MEM_DEVICE) {
        // merge_split_kernel reads a/b while other CTAs write low/high: when
        // an output overlaps an input, stage the inputs through workspace
        if (ranges_overlap(a, na, low, na) || ranges_overlap(a, na, high, nb) || ranges_overlap(b, nb, low, na) ||
            ranges_overlap(b, nb, high, nb)) {
            cudaError_t e = ctx->stage_b.ensure(std::max<uint64_t>(na + nb, 4) * 4);
            if (e != cudaSuccess) return cuda_fail(e, "merge_split staging");
            uint32_t* sa = ctx->stage_b.as<uint32_t>();
            if (na && (e = cudaMemcpyAsync(sa, a, na * 4, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
                return cuda_fail(e, "merge_split staging");
            if (nb && (e = cudaMemcpyAsync(sa + na, b, nb * 4, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
                return cuda_fail(e, "merge_split staging");
            a = sa;
            b = sa + na;
        }
        const int l = launch_merge_split(a, na, b, nb, low, high, st);
        if (l < 0) return cuda_fail(cudaGetLastError(), "merge_split launch");
        ctx->launches += static_cast<uint64_t>(l);
        return BSG_OK;
    }
    if (mem_kind != BSG_MEM_HOST) return fail(BSG_EINVAL, "mem_kind must be BSG_MEM_HOST or BSG_MEM_DEVICE");
    cudaError_t e;
    const uint64_t tot = std::max<uint64_t>(na + nb, 4);
    if ((e = ctx->stage_in.ensure(tot * 4)) != cudaSuccess) return cuda_fail(e, "host staging");
    if ((e = ctx->stage_out.ensure(tot * 4)) != cudaSuccess) return cuda_fail(e, "host staging");
    uint32_t* da = ctx->stage_in.as<uint32_t>();
    uint32_t* db = da + na;
    uint32_t* dl = ctx->stage_out.as<uint32_t>();
    uint32_t* dh = dl + na;
    if (na && (e = cudaMemcpyAsync(da, a, na * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess) return cuda_fail(e, "H2D");
    if (nb && (e = cudaMemcpyAsync(db, b, nb * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess) return cuda_fail(e, "H2D");
    const int l = launch_merge_split(da, na, db, nb, dl, dh, st);
    if (l < 0) return cuda_fail(cudaGetLastError(), "merge_split launch");
    ctx->launches += static_cast<uint64_t>(l);
    if (na && (e = cudaMemcpyAsync(low, dl, na * 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return cuda_fail(e, "D2H");
    if (nb && (e = cudaMemcpyAsync(high, dh, nb * 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return cuda_fail(e, "D2H");
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "stream synchronize");
    return BSG_OK;
}

int bsg_block_network_batched_u32(bsg_ctx* ctx, int network, const uint32_t* in, uint32_t* out, uint64_t num_arrays,
                                  uint32_t len, int p, int stages_limit, bsg_run_stats* stats, int mem_kind,
                                  void* stream) {
    if (int rc = check_ctx(ctx)) return rc;
    int S = 0;
    if (int rc = bsg_network_schedule(network, p, nullptr, nullptr, 0, &S)) return rc;
    const uint64_t L = (static_cast<uint64_t>(len) + p - 1) / p;
    const uint64_t padded = L * static_cast<uint64_t>(p);
    const bool full = stages_limit < 0 || stages_limit >= S;
    const int run = full ? S : stages_limit;
    const uint64_t out_per = full ? len : padded;
    if (num_arrays && len && (!in || !out)) return fail(BSG_EINVAL, "null key pointer");
    if (stats) {
        std::vector<int32_t> partner(static_cast<size_t>(S) * p), keep(static_cast<size_t>(S) * p);
        bsg_network_schedule(network, p, partner.data(), keep.data(), S, &S);
        bsg_run_stats st{};
        st.supersteps = 1 + run;
        for (int s = 0; s < run; ++s)
            for (int i = 0; i < p; ++i)
                if (partner[static_cast<size_t>(s) * p + i] >= 0) {
                    st.messages_sent += 1;
                    st.words_sent += L;
                }
        st.messages_delivered = st.messages_sent;
        st.words_delivered = st.words_sent;
        *stats = st;
    }
    CallGuard g(ctx, __func__);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder order(ctx, st);
    const uint64_t n_in = num_arrays * len, n_out = num_arrays * out_per;
    return with_device_io(ctx, in, out, n_in, n_out, mem_kind, st, [&](const uint32_t* d_in, uint32_t* d_out, cudaStream_t s) -> int {
        if (num_arrays == 0 || len == 0) return BSG_OK;
        if (padded <= kNetMaxPadded) { // shared-memory resident arrays: one CTA per array
            // one CTA reads array a and writes array a at the same stride: in
            // place is safe; a different output stride (padded intermediate
            // states) or a shifted overlap would overwrite arrays other CTAs
            // have yet to read, so stage the input through workspace
            if (ranges_overlap(d_in, n_in, d_out, n_out) && !(d_in == d_out && out_per == len)) {
                cudaError_t e = ctx->stage_b.ensure(std::max<uint64_t>(n_in, 4) * 4);
                if (e != cudaSuccess) return cuda_fail(e, "network staging");
                if ((e = cudaMemcpyAsync(ctx->stage_b.as<uint32_t>(), d_in, n_in * 4, cudaMemcpyDeviceToDevice, s)) !=
                    cudaSuccess)
                    return cuda_fail(e, "network staging");
                d_in = ctx->stage_b.as<uint32_t>();
            }
            const int l = launch_block_network(network, d_in, d_out, num_arrays, len, p, run, full, s);
            if (l < 0) return cuda_fail(cudaGetLastError(), "block network launch");
            ctx->launches += static_cast<uint64_t>(l);
            return BSG_OK;
        }
        // large arrays: blocks live in global memory; local sort = the radix
        // sort of each block (netsort.hpp:167 uses serial_radix_sort(., 256)),
        // each merge-split stage = one merge-path kernel over all pairs.
        cudaError_t e;
        if ((e = ctx->stage_b.ensure(padded * 4)) != cudaSuccess) return cuda_fail(e, "network workspace");
        if ((e = ctx->net_sched.ensure(padded * 4)) != cudaSuccess) return cuda_fail(e, "network workspace");
        RadixWorkspace ws;
        if (int rc = ctx->radix_ws(L, &ws)) return rc;
        uint32_t* A = ctx->net_sched.as<uint32_t>();
        uint32_t* B = ctx->stage_b.as<uint32_t>();
        for (uint64_t a = 0; a < num_arrays; ++a) {
            if ((e = cudaMemcpyAsync(A, d_in + a * len, static_cast<size_t>(len) * 4, cudaMemcpyDeviceToDevice, s)) !=
                cudaSuccess)
                return cuda_fail(e, "network copy");
            if (padded > len && (e = cudaMemsetAsync(A + len, 0xFF, (padded - len) * 4, s)) != cudaSuccess)
                return cuda_fail(e, "network pad");
            for (int w = 0; w < p; ++w) {
                const int l = launch_radix_sort8(A + static_cast<uint64_t>(w) * L, B + static_cast<uint64_t>(w) * L, L,
                                                 ws, s, true);
                if (l < 0) return cuda_fail(cudaGetLastError(), "network local sort");
                ctx->launches += static_cast<uint64_t>(l);
            }
            uint32_t* cur = B;
            uint32_t* oth = A;
            for (int st = 0; st < run; ++st) {
                if (launch_net_stage(cur, oth, p, static_cast<uint32_t>(L), network, st, s) < 0)
                    return cuda_fail(cudaGetLastError(), "network stage");
                ctx->launches += 1;
                std::swap(cur, oth);
            }
            if ((e = cudaMemcpyAsync(d_out + a * out_per, cur, out_per * 4, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
                return cuda_fail(e, "network copy out");
        }
        return BSG_OK;
    });
}

int bsg_parallel_radix_sort_u32(bsg_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n, int p, int radix_log2,
                                int rounds_limit, bsg_run_stats* stats, int mem_kind, void* stream) {
    if (int rc = check_ctx(ctx)) return rc;
    if (p < 1) return fail(BSG_EINVAL, "parallel radix sort: p must be >= 1");
    if (int rc = radix_bits_or_fail(radix_log2)) return rc;
    if (n && (!in || !out)) return fail(BSG_EINVAL, "null key pointer");
    const int all_rounds = 32 / radix_log2;
    const int rounds = (rounds_limit >= 0 && rounds_limit < all_rounds) ? rounds_limit : all_rounds;
    if (ctx->members.size() > 1) return parallel_radix_sort_group(ctx, in, out, n, p, radix_log2, rounds, stats, mem_kind,
                                                                  static_cast<cudaStream_t>(stream));
    CallGuard g(ctx, __func__);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder order(ctx, st);
    return with_device_io(ctx, in, out, n, n, mem_kind, st, [&](const uint32_t* d_in, uint32_t* d_out, cudaStream_t s) -> int {
        return run_parallel_radix_local(ctx, d_in, d_out, n, p, radix_log2, rounds, stats, s);
    });
}

int bsg_sort_instance_u32(bsg_ctx* ctx, const uint32_t* in, uint32_t* out, uint64_t n, int processors, int algorithm,
                          uint64_t radix, int mem_kind, void* stream) {
    // core.hpp:74-88 SortInstance::validate
    if (processors < 1) return fail(BSG_EINVAL, "SortInstance: processors must be >= 1");
    if (radix == 0 || (radix & (radix - 1)) != 0) return fail(BSG_EINVAL, "SortInstance: radix must be a power of two whose bit width divides 32");
    int bits = 0;
    while ((uint64_t{1} << bits) != radix) ++bits;
    if (bits == 0 || 32 % bits != 0)
        return fail(BSG_EINVAL, "SortInstance: radix must be a power of two whose bit width divides 32");
    if (algorithm == BSG_SR4 && processors != 1) return fail(BSG_EINVAL, "SortInstance: sr4 is serial, requires p = 1");
    if (algorithm == BSG_BTN && (processors & (processors - 1)) != 0)
        return fail(BSG_EINVAL, "SortInstance: btn requires a power-of-two p");
    if (algorithm == BSG_PR4 && radix != 256) return fail(BSG_EINVAL, "SortInstance: pr4 is radix-256 by definition");
    if (algorithm == BSG_PR2 && radix != 65536) return fail(BSG_EINVAL, "SortInstance: pr2 is radix-65536 by definition");
    // bspsort.hpp:15-25 dispatch
    switch (algorithm) {
    case BSG_SR4:
        return bsg_radix_sort_u32(ctx, in, out, n, bits, mem_kind, stream);
    case BSG_PR4:
    case BSG_PR2:
        return bsg_parallel_radix_sort_u32(ctx, in, out, n, processors, bits, -1, nullptr, mem_kind, stream);
    case BSG_BTN:
    case BSG_OET:
        if (n > 0xFFFFFFFFull) return fail(BSG_EINVAL, "block network: n must fit in 32 bits");
        return bsg_block_network_batched_u32(ctx, algorithm == BSG_BTN ? BSG_NET_BTN : BSG_NET_OET, in, out, n ? 1 : 0,
                                             static_cast<uint32_t>(n), processors, -1, nullptr, mem_kind, stream);
    default:
        return fail(BSG_EINVAL, "sort_instance: unknown algorithm");
    }
}

int bsg_pr_count_digits(bsg_ctx* ctx, const uint32_t* block, uint64_t len, int round, int radix_log2, uint64_t* counts,
                        void* stream) {
    if (int rc = check_ctx(ctx)) return rc;
    if (int rc = radix_bits_or_fail(radix_log2)) return rc;
    if (round < 0 || round >= 32 / radix_log2) return fail(BSG_EINVAL, "round out of range");
    CallGuard g(ctx, __func__);
    StreamOrder order(ctx, static_cast<cudaStream_t>(stream));
    const int l = launch_pr_count(ctx, block, len, round, radix_log2, counts, static_cast<cudaStream_t>(stream));
    if (l < 0) return cuda_fail(cudaGetLastError(), "count_digits launch");
    ctx->launches += static_cast<uint64_t>(l);
    return BSG_OK;
}

int bsg_pr_plan(bsg_ctx* ctx, const uint64_t* counts, uint64_t n, int p, int me, int round, int radix_log2,
                uint64_t* send_counts, uint64_t* recv_counts, int64_t* rebuild_delta, void* stream) {
    if (int rc = check_ctx(ctx)) return rc;
    if (int rc = radix_bits_or_fail(radix_log2)) return rc;
    if (p < 1 || me < 0 || me >= p) return fail(BSG_EINVAL, "pr_plan: worker index out of range");
    (void)round;
    CallGuard g(ctx, __func__);
    StreamOrder order(ctx, static_cast<cudaStream_t>(stream));
    // scratch for launch_pr_plan: split[p], coltot[r], dstart[r], colchunk[r/1024], rowchunk[p][r/1024]
    const uint64_t chunks = ((uint64_t{1} << radix_log2) + 1023) / 1024;
    cudaError_t e = ctx->pr_recv.ensure(
        (static_cast<uint64_t>(p) * (1 + chunks) + (uint64_t{2} << radix_log2) + chunks) * sizeof(uint64_t));
    if (e != cudaSuccess) return cuda_fail(e, "pr_plan scratch");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint32_t* flag = nullptr;
    if (int rc = proto_begin(ctx, st, &flag)) return rc;
    if (check_count_rows(counts, p, 1 << radix_log2, n, flag, st) < 0) return cuda_fail(cudaGetLastError(), "pr_plan check");
    const int l = launch_pr_plan(counts, n, p, me, radix_log2, send_counts, recv_counts, rebuild_delta, st,
                                 ctx->pr_recv.as<uint64_t>());
    if (l < 0) return cuda_fail(cudaGetLastError(), "pr_plan launch");
    ctx->launches += static_cast<uint64_t>(l) + 1;
    return proto_end(ctx, st, "bsp_error: a worker's exchanged digit counts do not sum to its block size");
}

int bsg_ctx_enable_peer_access(bsg_ctx* ctx, int* enabled) {
    if (int rc = check_ctx(ctx)) return rc;
    CallGuard g(ctx, __func__);
    int count = 0, ok = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    for (int d = 0; d < count; ++d) {
        if (d == ctx->device) continue;
        int can = 0;
        if (cudaDeviceCanAccessPeer(&can, ctx->device, d) != cudaSuccess || !can) continue;
        e = cudaDeviceEnablePeerAccess(d, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) {
            cudaGetLastError(); // clear the sticky-free status of this benign error
            e = cudaSuccess;
        }
        if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
        ++ok;
    }
    if (enabled) *enabled = ok;
    return BSG_OK;
}

int bsg_pr_local_sort(bsg_ctx* ctx, const uint32_t* block, uint32_t* sorted, uint64_t len, int round, int radix_log2,
                      void* stream) {
    return bsg_count_sort_round_u32(ctx, block, sorted, len, round, radix_log2, BSG_MEM_DEVICE, stream);
}

int bsg_pr_rebuild(bsg_ctx* ctx, const uint32_t* recv, uint64_t recv_len, const uint64_t* recv_counts, int p, int round,
                   int radix_log2, const int64_t* rebuild_delta, uint32_t* block, void* stream) {
    if (int rc = check_ctx(ctx)) return rc;
    if (int rc = radix_bits_or_fail(radix_log2)) return rc;
    if (round < 0 || round >= 32 / radix_log2) return fail(BSG_EINVAL, "round out of range");
    if (p < 1 || !recv_counts || (recv_len && (!recv || !block || !rebuild_delta))) return fail(BSG_EINVAL, "null pointer");
    CallGuard g(ctx, __func__);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder order(ctx, st);
    uint32_t* flag = nullptr;
    if (int rc = proto_begin(ctx, st, &flag)) return rc;
    const int l = launch_pr_rebuild(recv, recv_len, radix_log2, round * radix_log2, rebuild_delta, block, st,
                                    recv_counts, p, flag);
    if (l < 0) return cuda_fail(cudaGetLastError(), "rebuild launch");
    ctx->launches += static_cast<uint64_t>(l);
    return proto_end(ctx, st, "bsp_error: received key slices do not fill the rebuilt block");
}

} // extern "C"
