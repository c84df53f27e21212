// bspsort_b200/bspsort.hpp -- header-only C++20 mirror of the reference API
// (/root/reference/proj/include/bspsort/{core,radix,netsort,bspsort}.hpp):
// same namespaces, names, argument meaning and error behaviour, implemented
// over the C ABI in bsg.h (link with paper_1708_09495_b200/libbsg.so).  A user
// of the reference switches by replacing `#include "bspsort/bspsort.hpp"`
// with this header; KeyArray-by-value calls stage through the GPU.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "../bsg.h"

namespace bspsort {

using Key = std::uint32_t;
using KeyArray = std::vector<Key>;
inline constexpr int key_bits = 32;

enum class Algorithm { SR4, PR4, PR2, BTN, OET }; // core.hpp:24

inline const char* algorithm_name(Algorithm a) {
    switch (a) {
    case Algorithm::SR4: return "sr4";
    case Algorithm::PR4: return "pr4";
    case Algorithm::PR2: return "pr2";
    case Algorithm::BTN: return "btn";
    case Algorithm::OET: return "oet";
    }
    return "?";
}

inline std::optional<Algorithm> algorithm_from_name(std::string_view name) {
    std::string s(name);
    for (auto& c : s) c = static_cast<char>(c >= 'A' && c <= 'Z' ? c - 'A' + 'a' : c);
    if (s == "sr4") return Algorithm::SR4;
    if (s == "pr4") return Algorithm::PR4;
    if (s == "pr2") return Algorithm::PR2;
    if (s == "btn") return Algorithm::BTN;
    if (s == "oet") return Algorithm::OET;
    return std::nullopt;
}

inline constexpr bool is_power_of_two(std::uint64_t x) { return x != 0 && (x & (x - 1)) == 0; }
inline constexpr int log2_exact(std::uint64_t x) {
    int b = -1;
    while (x) { x >>= 1; ++b; }
    return b;
}
inline constexpr int digit_bits(std::uint64_t radix) {
    if (!is_power_of_two(radix)) return -1;
    const int b = log2_exact(radix);
    return (b > 0 && key_bits % b == 0) ? b : -1;
}

namespace bsp {
using Word = std::uint32_t;          // bsp.hpp:26
using Block = std::vector<Word>;     // bsp.hpp:27
// bsp.hpp:38-41; protocol failures reported by the GPU path (BSG_EPROTO).
class bsp_error : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};
// bsp.hpp:86-92
struct RunStats {
    int supersteps = 0;
    std::uint64_t messages_sent = 0, messages_delivered = 0, words_sent = 0, words_delivered = 0;
};
} // namespace bsp

namespace detail {
// Maps C-ABI status codes to the reference's exception types.
inline void check(int status) {
    if (status == BSG_OK) return;
    const std::string msg = bsg_last_error();
    if (status == BSG_EINVAL) throw std::invalid_argument(msg);
    if (status == BSG_EPROTO) throw bsp::bsp_error(msg);
    if (status == BSG_ENOMEM) throw std::bad_alloc();
    throw std::runtime_error(msg);
}
// One context per process on device 0.
inline bsg_ctx* context() {
    static std::once_flag once;
    static bsg_ctx* ctx = nullptr;
    static int rc = BSG_OK;
    std::call_once(once, [] { rc = bsg_ctx_create(0, &ctx); });
    check(rc);
    return ctx;
}
// The process-wide multi-GPU group used by run_parallel_radix once
// bspsort::gpu::use_devices() was called (nullptr: one GPU).
struct GroupHolder {
    std::mutex mu;
    bsg_ctx* grp = nullptr;
    ~GroupHolder() {
        if (grp) bsg_ctx_destroy(grp);
    }
};
inline GroupHolder& group_holder() {
    static GroupHolder h;
    return h;
}
inline bsp::RunStats to_stats(const bsg_run_stats& s) {
    return bsp::RunStats{s.supersteps, s.messages_sent, s.messages_delivered, s.words_sent, s.words_delivered};
}
} // namespace detail

struct SortInstance { // core.hpp:67-89
    KeyArray input;
    int processors = 1;
    Algorithm algorithm = Algorithm::SR4;
    std::uint64_t radix = 256;
    std::uint64_t seed = 0;

    void validate() const {
        if (processors < 1) throw std::invalid_argument("SortInstance: processors must be >= 1");
        if (digit_bits(radix) < 0)
            throw std::invalid_argument("SortInstance: radix must be a power of two whose bit width divides 32");
        if (algorithm == Algorithm::SR4 && processors != 1)
            throw std::invalid_argument("SortInstance: sr4 is serial, requires p = 1");
        if (algorithm == Algorithm::BTN && !is_power_of_two(static_cast<std::uint64_t>(processors)))
            throw std::invalid_argument("SortInstance: btn requires a power-of-two p");
        if (algorithm == Algorithm::PR4 && radix != 256)
            throw std::invalid_argument("SortInstance: pr4 is radix-256 by definition");
        if (algorithm == Algorithm::PR2 && radix != 65536)
            throw std::invalid_argument("SortInstance: pr2 is radix-65536 by definition");
    }
};

inline KeyArray generate_uniform_keys(std::size_t n, std::uint64_t seed) { // core.hpp:93-99
    KeyArray keys(n);
    detail::check(bsg_generate_uniform_u32(keys.data(), n, seed));
    return keys;
}

inline bool verify_sorted_permutation(const KeyArray& input, const KeyArray& output); // defined below

namespace radix {

inline constexpr Key digit_of(Key key, int round, int bits) { // radix.hpp:28-30
    return (key >> (round * bits)) & ((std::uint64_t{1} << bits) - 1);
}

inline int checked_digit_bits(std::uint64_t radix) { // radix.hpp:32-40
    const int b = bsg_checked_digit_bits(radix);
    if (b < 0) throw std::invalid_argument(bsg_last_error());
    return b;
}

inline KeyArray count_sort_round(const KeyArray& keys, int round, std::uint64_t radix) { // radix.hpp:44-65
    const int bits = checked_digit_bits(radix);
    KeyArray out(keys.size());
    detail::check(bsg_count_sort_round_u32(detail::context(), keys.data(), out.data(), keys.size(), round, bits,
                                           BSG_MEM_HOST, nullptr));
    return out;
}

inline KeyArray serial_radix_sort(KeyArray keys, std::uint64_t radix) { // radix.hpp:69-90
    const int bits = checked_digit_bits(radix);
    detail::check(bsg_radix_sort_u32(detail::context(), keys.data(), keys.data(), keys.size(), bits, BSG_MEM_HOST,
                                     nullptr));
    return keys;
}

namespace detail {
struct Partition { // radix.hpp:96-118
    std::uint64_t n = 0;
    int p = 1;
    std::uint64_t small() const { return n / p; }
    std::uint64_t big_count() const { return n % p; }
    std::uint64_t size_of(int w) const { return bsg_partition_size_of(n, p, w); }
    std::uint64_t offset_of(int w) const { return bsg_partition_offset_of(n, p, w); }
    int owner_of(std::uint64_t pos) const { return bsg_partition_owner_of(n, p, pos); }
};
struct RadixPlan { // radix.hpp:120-125
    Partition part;
    std::uint64_t radix = 256;
    int bits = 8;
    int rounds = 4;
};
} // namespace detail

struct PreparedRadix { // radix.hpp:228-231
    detail::RadixPlan plan;
    std::vector<bsp::Block> blocks;
};

inline PreparedRadix prepare_parallel_radix(const KeyArray& keys, int p, std::uint64_t radix) { // radix.hpp:233-249
    if (p < 1) throw std::invalid_argument("parallel radix sort: p must be >= 1");
    const int bits = checked_digit_bits(radix);
    PreparedRadix prep;
    prep.plan.part = detail::Partition{keys.size(), p};
    prep.plan.radix = radix;
    prep.plan.bits = bits;
    prep.plan.rounds = key_bits / bits;
    prep.blocks.resize(p);
    for (int w = 0; w < p; ++w) {
        const auto begin = keys.begin() + static_cast<std::ptrdiff_t>(prep.plan.part.offset_of(w));
        prep.blocks[w].assign(begin, begin + static_cast<std::ptrdiff_t>(prep.plan.part.size_of(w)));
    }
    return prep;
}

struct ParallelSortResult { // radix.hpp:251-254
    KeyArray output;
    bsp::RunStats stats;
};

// radix.hpp:260-303; the executor flag is accepted, results are identical.
// The workers run on the GPU -- or on every GPU given to gpu::use_devices().
// Blocks must be the plan's Partition (bsp_error otherwise, as the
// reference's gather_slices consistency checks would raise).
inline ParallelSortResult run_parallel_radix(PreparedRadix prep, bool use_sequential_executor = false) {
    (void)use_sequential_executor;
    const int p = prep.plan.part.p;
    if (static_cast<int>(prep.blocks.size()) != p) throw bsp::bsp_error("run_parallel_radix: expected p blocks");
    std::uint64_t n = 0;
    for (const auto& b : prep.blocks) n += b.size();
    if (n != prep.plan.part.n) throw bsp::bsp_error("run_parallel_radix: blocks do not hold the plan's n keys");
    KeyArray keys;
    keys.reserve(n);
    for (int w = 0; w < p; ++w) {
        if (prep.blocks[w].size() != prep.plan.part.size_of(w))
            throw bsp::bsp_error("run_parallel_radix: block sizes differ from the balanced partition");
        keys.insert(keys.end(), prep.blocks[w].begin(), prep.blocks[w].end());
    }
    const int all = key_bits / prep.plan.bits;
    const int limit = prep.plan.rounds >= all ? -1 : prep.plan.rounds;
    ParallelSortResult res;
    res.output.resize(n);
    bsg_run_stats st{};
    bsg_ctx* ctx = ::bspsort::detail::context();
    auto& gh = ::bspsort::detail::group_holder();
    {
        std::lock_guard<std::mutex> lk(gh.mu);
        if (gh.grp) ctx = gh.grp;
    }
    ::bspsort::detail::check(bsg_parallel_radix_sort_u32(ctx, keys.data(), res.output.data(), n, p, prep.plan.bits,
                                                         limit, &st, BSG_MEM_HOST, nullptr));
    res.stats = ::bspsort::detail::to_stats(st);
    return res;
}

inline KeyArray parallel_radix_sort(const SortInstance& instance) { // radix.hpp:306-312
    instance.validate();
    if (instance.algorithm != Algorithm::PR4 && instance.algorithm != Algorithm::PR2)
        throw std::invalid_argument("parallel_radix_sort handles pr4 and pr2 only");
    return run_parallel_radix(prepare_parallel_radix(instance.input, instance.processors, instance.radix)).output;
}

} // namespace radix

namespace netsort {

inline constexpr std::uint64_t local_sort_radix = 256;

inline std::pair<KeyArray, KeyArray> merge_split(const KeyArray& a, const KeyArray& b) { // netsort.hpp:30-51
    KeyArray low(a.size()), high(b.size());
    ::bspsort::detail::check(bsg_merge_split_u32(::bspsort::detail::context(), a.data(), a.size(), b.data(), b.size(),
                                                 low.data(), high.data(), BSG_MEM_HOST, nullptr));
    return {std::move(low), std::move(high)};
}

struct StageAssignment { // netsort.hpp:56-59
    int partner = -1;
    bool keep_low = false;
};
struct BitonicSchedule { // netsort.hpp:61-64
    int p = 1;
    std::vector<std::vector<StageAssignment>> stages;
};

namespace detail {
inline std::vector<std::vector<StageAssignment>> schedule(int network, int p) {
    int S = 0;
    ::bspsort::detail::check(bsg_network_schedule(network, p, nullptr, nullptr, 0, &S));
    std::vector<std::int32_t> partner(static_cast<std::size_t>(S) * p), keep(static_cast<std::size_t>(S) * p);
    ::bspsort::detail::check(bsg_network_schedule(network, p, partner.data(), keep.data(), S, &S));
    std::vector<std::vector<StageAssignment>> st(S, std::vector<StageAssignment>(p));
    for (int s = 0; s < S; ++s)
        for (int i = 0; i < p; ++i) st[s][i] = StageAssignment{partner[s * p + i], keep[s * p + i] != 0};
    return st;
}
} // namespace detail

inline BitonicSchedule bitonic_schedule(int p) { return BitonicSchedule{p, detail::schedule(BSG_NET_BTN, p)}; }
inline std::vector<std::vector<StageAssignment>> odd_even_rounds(int p) { return detail::schedule(BSG_NET_OET, p); }

struct PreparedNetwork { // netsort.hpp:112-118 (+ which network the table came from)
    int p = 1;
    std::uint64_t n = 0;   // keys before padding
    std::size_t pad = 0;   // trailing max-value keys to strip from the output
    std::vector<bsp::Block> blocks;
    std::vector<std::vector<StageAssignment>> stages;
    int network = BSG_NET_BTN;
};

namespace detail {
// netsort.hpp:124-141: blocks of ceil(n/p) keys padded with ~Key{0}
inline PreparedNetwork prepare_blocks(const KeyArray& keys, int p, std::vector<std::vector<StageAssignment>> stages,
                                      int network) {
    PreparedNetwork prep;
    prep.p = p;
    prep.n = keys.size();
    prep.stages = std::move(stages);
    prep.network = network;
    const std::size_t block_len = (keys.size() + p - 1) / p;
    prep.pad = block_len * p - keys.size();
    prep.blocks.assign(p, {});
    for (int w = 0; w < p; ++w) {
        const std::size_t begin = std::min(keys.size(), w * block_len);
        const std::size_t end = std::min(keys.size(), begin + block_len);
        prep.blocks[w].assign(keys.begin() + begin, keys.begin() + end);
        prep.blocks[w].resize(block_len, ~Key{0});
    }
    return prep;
}
// The GPU path runs the closed-form BTN / OET schedules: a stage table must
// be a prefix of one of them (a truncated table stops early); other custom
// tables are rejected rather than silently replaced.
inline int prefix_of_network(const PreparedNetwork& prep) {
    const int other = prep.network == BSG_NET_BTN ? static_cast<int>(BSG_NET_OET) : static_cast<int>(BSG_NET_BTN);
    for (int net : {prep.network, other}) {
        if (net == BSG_NET_BTN && !is_power_of_two(static_cast<std::uint64_t>(prep.p))) continue;
        const auto full = schedule(net, prep.p);
        if (prep.stages.size() > full.size()) continue;
        bool same = true;
        for (std::size_t s = 0; s < prep.stages.size() && same; ++s) {
            if (prep.stages[s].size() != static_cast<std::size_t>(prep.p)) same = false;
            for (int i = 0; i < prep.p && same; ++i)
                same = prep.stages[s][i].partner == full[s][i].partner &&
                       (prep.stages[s][i].partner < 0 || prep.stages[s][i].keep_low == full[s][i].keep_low);
        }
        if (same) return net;
    }
    throw std::invalid_argument("run_block_network: the GPU path runs the BTN/OET schedules (or a prefix of them); "
                                "custom stage tables are not supported");
}
} // namespace detail

inline PreparedNetwork prepare_btn(const KeyArray& keys, int p) { // netsort.hpp:145-147
    return detail::prepare_blocks(keys, p, bitonic_schedule(p).stages, BSG_NET_BTN);
}
inline PreparedNetwork prepare_oet(const KeyArray& keys, int p) { // netsort.hpp:149-151
    return detail::prepare_blocks(keys, p, odd_even_rounds(p), BSG_NET_OET);
}

// netsort.hpp:157-199; a truncated stage table stops the network early.  The
// concatenated (padded) blocks are the device input; the output is stripped
// to n keys (netsort.hpp:197).
inline radix::ParallelSortResult run_block_network(PreparedNetwork prep, bool use_sequential_executor = false) {
    (void)use_sequential_executor;
    if (static_cast<int>(prep.blocks.size()) != prep.p) throw bsp::bsp_error("run_block_network: expected p blocks");
    const std::size_t L = prep.blocks.empty() ? 0 : prep.blocks[0].size();
    KeyArray keys;
    keys.reserve(L * prep.p);
    for (const auto& b : prep.blocks) {
        if (b.size() != L) throw bsp::bsp_error("merge_split: blocks differ in size"); // netsort.hpp:172-176
        keys.insert(keys.end(), b.begin(), b.end());
    }
    const int net = detail::prefix_of_network(prep);
    int S = 0;
    ::bspsort::detail::check(bsg_network_schedule(net, prep.p, nullptr, nullptr, 0, &S));
    const int limit = static_cast<int>(prep.stages.size()) >= S ? -1 : static_cast<int>(prep.stages.size());
    if (keys.size() > 0xFFFFFFFFull) throw std::invalid_argument("block network: n must fit in 32 bits");
    KeyArray out(keys.size());
    bsg_run_stats st{};
    ::bspsort::detail::check(bsg_block_network_batched_u32(::bspsort::detail::context(), net, keys.data(), out.data(),
                                                           keys.empty() ? 0 : 1, static_cast<std::uint32_t>(keys.size()),
                                                           prep.p, limit, &st, BSG_MEM_HOST, nullptr));
    out.resize(prep.n); // netsort.hpp:197
    return radix::ParallelSortResult{std::move(out), ::bspsort::detail::to_stats(st)};
}

inline KeyArray btn_sort(const SortInstance& instance) { // netsort.hpp:202-207
    instance.validate();
    if (instance.algorithm != Algorithm::BTN) throw std::invalid_argument("btn_sort expects a BTN instance");
    return run_block_network(prepare_btn(instance.input, instance.processors)).output;
}
inline KeyArray oet_sort(const SortInstance& instance) { // netsort.hpp:210-215
    instance.validate();
    if (instance.algorithm != Algorithm::OET) throw std::invalid_argument("oet_sort expects an OET instance");
    return run_block_network(prepare_oet(instance.input, instance.processors)).output;
}

} // namespace netsort

// B200 extension: run the parallel radix sort's p workers over several GPUs
// of this process (a group context, bsg_ctx_create_group).  Call once before
// run_parallel_radix / parallel_radix_sort / sort_instance; an empty list
// returns to one GPU.  Reference code is otherwise unchanged.
namespace gpu {
inline void use_devices(const std::vector<int>& devices) {
    auto& gh = ::bspsort::detail::group_holder();
    std::lock_guard<std::mutex> lk(gh.mu);
    if (gh.grp) {
        bsg_ctx_destroy(gh.grp);
        gh.grp = nullptr;
    }
    if (devices.empty()) return;
    bsg_ctx* g = nullptr;
    ::bspsort::detail::check(bsg_ctx_create_group(devices.data(), static_cast<int>(devices.size()), &g));
    gh.grp = g;
}
} // namespace gpu

inline KeyArray sort_instance(const SortInstance& instance) { // bspsort.hpp:15-25
    instance.validate();
    switch (instance.algorithm) {
    case Algorithm::SR4: return radix::serial_radix_sort(instance.input, instance.radix);
    case Algorithm::PR4:
    case Algorithm::PR2: return radix::parallel_radix_sort(instance);
    case Algorithm::BTN: return netsort::btn_sort(instance);
    case Algorithm::OET: return netsort::oet_sort(instance);
    }
    throw std::invalid_argument("sort_instance: unknown algorithm");
}

inline bool verify_sorted_permutation(const KeyArray& input, const KeyArray& output) { // core.hpp:103-109
    if (input.size() != output.size()) return false;
    for (std::size_t i = 1; i < output.size(); ++i)
        if (output[i - 1] > output[i]) return false;
    // the permutation check runs on the GPU sort (an independent algorithm
    // from the one under test is the caller's choice)
    return radix::serial_radix_sort(input, 256) == output;
}

} // namespace bspsort
