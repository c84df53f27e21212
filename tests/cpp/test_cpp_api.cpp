// Restates a subset of the reference's own GTest cases (radix_test.cpp,
// netsort_test.cpp, core_test.cpp) against the C++ mirror
// include/bspsort_b200/bspsort.hpp, i.e. through the C ABI on the GPU.
// Prints "OK <n>" and returns 0 when every check holds.
#include <algorithm>
#include <cstdio>
#include <stdexcept>

#include "bspsort_b200/bspsort.hpp"

using namespace bspsort;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                                   \
    do {                                                                              \
        ++g_checks;                                                                   \
        if (!(cond)) {                                                                \
            ++g_fail;                                                                 \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);               \
        }                                                                             \
    } while (0)

template <class F> static bool throws_invalid(F&& f) {
    try {
        f();
    } catch (const std::invalid_argument&) {
        return true;
    }
    return false;
}

static KeyArray oracle_sort(KeyArray k) {
    std::sort(k.begin(), k.end());
    return k;
}

int main() {
    // core_test.cpp:24-31
    CHECK((generate_uniform_keys(6, 42) ==
           KeyArray{0x6ee5e2d6u, 0xb92502a8u, 0x0e5e7b0au, 0x8a1ad34eu, 0x4d361955u, 0x9c7f4f7cu}));
    // radix_test.cpp:137-151
    CHECK(radix::count_sort_round({}, 0, 256).empty());
    CHECK((radix::count_sort_round({0x0103, 0x0201, 0x0102}, 0, 256) == KeyArray{0x0201, 0x0102, 0x0103}));
    CHECK((radix::count_sort_round({0x0101, 0x0001}, 0, 256) == KeyArray{0x0101, 0x0001}));
    // radix_test.cpp:189-195
    CHECK(throws_invalid([] { radix::count_sort_round({1}, 4, 256); }));
    CHECK(throws_invalid([] { radix::count_sort_round({1}, 0, 100); }));
    // radix_test.cpp:197-223
    const auto in = generate_uniform_keys(100000, 3);
    const auto expect = oracle_sort(in);
    CHECK(radix::serial_radix_sort(in, 256) == expect);
    CHECK(radix::serial_radix_sort(in, 65536) == expect);
    CHECK(radix::serial_radix_sort(in, 2) == expect);
    KeyArray composed = generate_uniform_keys(5000, 11);
    const KeyArray base = composed;
    for (int r = 0; r < 4; ++r) composed = radix::count_sort_round(composed, r, 256);
    CHECK(radix::serial_radix_sort(base, 256) == composed);
    // radix_test.cpp:233-267
    const auto in9 = generate_uniform_keys(100000, 9);
    const auto exp9 = oracle_sort(in9);
    for (int p : {2, 3, 4, 5, 8, 16}) {
        SortInstance s;
        s.input = in9;
        s.processors = p;
        s.algorithm = Algorithm::PR4;
        s.radix = 256;
        CHECK(radix::parallel_radix_sort(s) == exp9);
    }
    {
        auto prep = radix::prepare_parallel_radix(generate_uniform_keys(5000, 21), 4, 256);
        CHECK(radix::run_parallel_radix(std::move(prep)).stats.supersteps == 9);
        auto prep2 = radix::prepare_parallel_radix(generate_uniform_keys(5000, 21), 4, 65536);
        CHECK(radix::run_parallel_radix(std::move(prep2)).stats.supersteps == 5);
    }
    {
        SortInstance s;
        s.input = {5, 1, 4};
        s.processors = 8;
        s.algorithm = Algorithm::PR4;
        CHECK((radix::parallel_radix_sort(s) == KeyArray{1, 4, 5}));
    }
    // netsort_test.cpp:52-82
    {
        auto [lo, hi] = netsort::merge_split({1, 9}, {5});
        CHECK((lo == KeyArray{1, 5}) && (hi == KeyArray{9}));
        auto [lo2, hi2] = netsort::merge_split({1, 3, 5}, {2, 4, 6});
        CHECK((lo2 == KeyArray{1, 2, 3}) && (hi2 == KeyArray{4, 5, 6}));
    }
    CHECK(netsort::bitonic_schedule(16).stages.size() == 10u);
    CHECK(throws_invalid([] { netsort::bitonic_schedule(3); }));
    // netsort_test.cpp:174-232
    const auto in31 = generate_uniform_keys(100000, 31);
    const auto exp31 = oracle_sort(in31);
    for (int p : {2, 4, 8, 16}) {
        SortInstance s;
        s.input = in31;
        s.processors = p;
        s.algorithm = Algorithm::BTN;
        CHECK(netsort::btn_sort(s) == exp31);
    }
    const auto in23 = generate_uniform_keys(10000, 23);
    for (int p : {2, 3, 4, 5, 7, 8, 16}) {
        SortInstance s;
        s.input = in23;
        s.processors = p;
        s.algorithm = Algorithm::OET;
        CHECK(netsort::oet_sort(s) == oracle_sort(in23));
    }
    for (int p : {1, 2, 5, 8}) {
        auto res = netsort::run_block_network(netsort::prepare_oet(generate_uniform_keys(6000, 2), p));
        CHECK(res.stats.supersteps == 1 + p);
    }
    // bspsort.hpp:15-25 + core.hpp:74-88
    {
        SortInstance bad;
        bad.input = {3, 2, 1};
        bad.processors = 2;
        bad.algorithm = Algorithm::SR4;
        CHECK(throws_invalid([&] { sort_instance(bad); }));
        SortInstance ok;
        ok.input = {3, 2, 1};
        ok.algorithm = Algorithm::SR4;
        CHECK((sort_instance(ok) == KeyArray{1, 2, 3}));
    }
    // PreparedRadix::blocks / PreparedNetwork::blocks as in the reference
    // (radix.hpp:228-249, netsort.hpp:112-141), and the intermediate states
    // the reference exposes through plan.rounds / a truncated stage table
    {
        const auto k = generate_uniform_keys(10007, 5);
        auto prep = radix::prepare_parallel_radix(k, 3, 256);
        CHECK(prep.blocks.size() == 3u && prep.blocks[0].size() == 3336u && prep.blocks[2].size() == 3335u);
        prep.plan.rounds = 1;
        CHECK(radix::run_parallel_radix(prep).output == radix::count_sort_round(k, 0, 256));
        prep.blocks[1].pop_back();
        bool threw = false;
        try {
            radix::run_parallel_radix(prep);
        } catch (const bsp::bsp_error&) {
            threw = true;
        }
        CHECK(threw);
        auto net = netsort::prepare_btn(k, 4);
        CHECK(net.blocks.size() == 4u && net.blocks[3].size() == 2502u && net.pad == 1u && net.blocks[3].back() == ~Key{0});
        CHECK(netsort::run_block_network(net).output == oracle_sort(k));
        auto bad = net;
        bad.stages[0][0].partner = 2;
        CHECK(throws_invalid([&] { netsort::run_block_network(bad); }));
    }
    // several GPUs through the unchanged reference API (cuda:0 listed twice
    // on a one-GPU box: the group code path with local stores)
    {
        gpu::use_devices({0, 0});
        const auto k = generate_uniform_keys(300001, 6);
        for (int p : {2, 3, 8}) {
            SortInstance s;
            s.input = k;
            s.processors = p;
            s.algorithm = Algorithm::PR2;
            s.radix = 65536;
            CHECK(radix::parallel_radix_sort(s) == oracle_sort(k));
            auto prep = radix::prepare_parallel_radix(k, p, 256);
            prep.plan.rounds = 2;
            KeyArray two = radix::count_sort_round(radix::count_sort_round(k, 0, 256), 1, 256);
            CHECK(radix::run_parallel_radix(prep).output == two);
        }
        gpu::use_devices({});
    }
    CHECK(verify_sorted_permutation({3, 1, 2}, {1, 2, 3}));
    CHECK(!verify_sorted_permutation({3, 1, 2}, {1, 2, 4}));
    std::printf("%s %d checks, %d failed\n", g_fail ? "FAILED" : "OK", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
