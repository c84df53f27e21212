// ref_shim.cpp -- extern "C" wrappers around the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (see oracle/bsg_oracle.c header).  This file holds
// no reference source: it #includes the read-only hot-path headers from
// $(BSPSORT_REF_INCLUDE) (default /root/reference/proj/include) and is built by
// oracle/Makefile into oracle/_ref/libbspref.so.  bench.py's cpu_baseline and
// --impl reference legs time these entry points on the GPU box's host cores
// (the .so travels; /root/reference does not).
//
// Only core/bsp/radix/netsort are included: bench.hpp and bspsort.hpp pull in
// costmodel.hpp, which needs Boost.Multiprecision (absent), so the 5-way
// dispatch of bspsort.hpp:15-25 is restated in ref_sort_instance below.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>

#include "bspsort/core.hpp"
#include "bspsort/bsp.hpp"
#include "bspsort/radix.hpp"
#include "bspsort/netsort.hpp"

using namespace bspsort;

struct ref_run_stats {
    int supersteps;
    std::uint64_t messages_sent, messages_delivered, words_sent, words_delivered;
};

static void fill_stats(ref_run_stats* out, const bsp::RunStats& s) {
    if (!out) return;
    out->supersteps = s.supersteps;
    out->messages_sent = s.messages_sent;
    out->messages_delivered = s.messages_delivered;
    out->words_sent = s.words_sent;
    out->words_delivered = s.words_delivered;
}

// 0 ok, 1 invalid_argument, 2 bsp_error, 3 other
template <class F> static int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const bsp::bsp_error&) {
        return 2;
    } catch (...) {
        return 3;
    }
}

extern "C" {

int ref_generate_uniform_keys(std::uint32_t* out, std::uint64_t n, std::uint64_t seed) {
    return guard([&] {
        auto k = generate_uniform_keys(n, seed);
        std::memcpy(out, k.data(), n * sizeof(std::uint32_t));
    });
}

int ref_count_sort_round(const std::uint32_t* in, std::uint64_t n, int round, std::uint64_t radix,
                         std::uint32_t* out) {
    return guard([&] {
        KeyArray keys(in, in + n);
        auto r = radix::count_sort_round(keys, round, radix);
        std::memcpy(out, r.data(), n * sizeof(std::uint32_t));
    });
}

// Timed entry for the CPU baseline: input copy outside, like bench.hpp run_once.
int ref_serial_radix_sort(const std::uint32_t* in, std::uint64_t n, std::uint64_t radix,
                          std::uint32_t* out) {
    return guard([&] {
        KeyArray keys(in, in + n);
        auto r = radix::serial_radix_sort(std::move(keys), radix);
        std::memcpy(out, r.data(), n * sizeof(std::uint32_t));
    });
}

// prepare_parallel_radix + run_parallel_radix; rounds_limit >= 0 overrides
// plan.rounds (SURVEY §8(c) per-round oracle).
int ref_parallel_radix(const std::uint32_t* in, std::uint64_t n, int p, std::uint64_t radix,
                       int rounds_limit, int use_sequential, std::uint32_t* out,
                       ref_run_stats* stats) {
    return guard([&] {
        KeyArray keys(in, in + n);
        auto prep = radix::prepare_parallel_radix(keys, p, radix);
        if (rounds_limit >= 0 && rounds_limit < prep.plan.rounds) prep.plan.rounds = rounds_limit;
        auto res = radix::run_parallel_radix(std::move(prep), use_sequential != 0);
        std::memcpy(out, res.output.data(), res.output.size() * sizeof(std::uint32_t));
        fill_stats(stats, res.stats);
    });
}

// prepare_btn/oet + run_block_network; stages_limit >= 0 truncates the
// stage table (valid as a per-stage oracle only when p | n).
// Writes out_len keys (n, or the padded length when truncated and padded).
int ref_block_network(int network, const std::uint32_t* in, std::uint64_t n, int p,
                      int stages_limit, int use_sequential, std::uint32_t* out,
                      std::uint64_t* out_len, ref_run_stats* stats) {
    return guard([&] {
        KeyArray keys(in, in + n);
        auto prep = network == 0 ? netsort::prepare_btn(keys, p) : netsort::prepare_oet(keys, p);
        if (stages_limit >= 0 && static_cast<std::size_t>(stages_limit) < prep.stages.size())
            prep.stages.resize(static_cast<std::size_t>(stages_limit));
        auto res = netsort::run_block_network(std::move(prep), use_sequential != 0);
        std::memcpy(out, res.output.data(), res.output.size() * sizeof(std::uint32_t));
        if (out_len) *out_len = res.output.size();
        fill_stats(stats, res.stats);
    });
}

int ref_merge_split(const std::uint32_t* a, std::uint64_t na, const std::uint32_t* b,
                    std::uint64_t nb, std::uint32_t* low, std::uint32_t* high) {
    return guard([&] {
        KeyArray va(a, a + na), vb(b, b + nb);
        auto [lo, hi] = netsort::merge_split(va, vb);
        std::memcpy(low, lo.data(), lo.size() * sizeof(std::uint32_t));
        std::memcpy(high, hi.data(), hi.size() * sizeof(std::uint32_t));
    });
}

// bitonic_schedule / odd_even_rounds, stage-major partner/keep_low arrays.
int ref_schedule(int network, int p, int* partner, int* keep_low, int cap_stages, int* stages) {
    return guard([&] {
        auto st = network == 0 ? netsort::bitonic_schedule(p).stages : netsort::odd_even_rounds(p);
        *stages = static_cast<int>(st.size());
        for (int s = 0; s < static_cast<int>(st.size()) && s < cap_stages; ++s)
            for (int i = 0; i < p; ++i) {
                partner[s * p + i] = st[s][i].partner;
                keep_low[s * p + i] = st[s][i].keep_low ? 1 : 0;
            }
    });
}

// Timed entry points mirroring bench::detail::run_once (bench.hpp:114-141):
// the input copy / prepare stay outside the timer, only the sort is timed
// (steady_clock, bench.hpp:92-97).  Return seconds, or a negative value on
// error.
double ref_time_serial_radix_sort(const std::uint32_t* in, std::uint64_t n, std::uint64_t radix,
                                  std::uint32_t* out) {
    try {
        KeyArray work(in, in + n);
        const auto t0 = std::chrono::steady_clock::now();
        KeyArray r = radix::serial_radix_sort(std::move(work), radix);
        const auto t1 = std::chrono::steady_clock::now();
        std::memcpy(out, r.data(), n * sizeof(std::uint32_t));
        return std::chrono::duration<double>(t1 - t0).count();
    } catch (...) {
        return -1.0;
    }
}

double ref_time_parallel_radix(const std::uint32_t* in, std::uint64_t n, int p, std::uint64_t radix,
                               std::uint32_t* out) {
    try {
        KeyArray keys(in, in + n);
        auto prep = radix::prepare_parallel_radix(keys, p, radix);
        const auto t0 = std::chrono::steady_clock::now();
        auto res = radix::run_parallel_radix(std::move(prep));
        const auto t1 = std::chrono::steady_clock::now();
        std::memcpy(out, res.output.data(), n * sizeof(std::uint32_t));
        return std::chrono::duration<double>(t1 - t0).count();
    } catch (...) {
        return -1.0;
    }
}

double ref_time_block_network(int network, const std::uint32_t* in, std::uint64_t num_arrays, std::uint64_t len,
                              int p, std::uint32_t* out) {
    // The reference has no batched API: one run_block_network per array with
    // the sequential executor, timed over the whole batch.
    try {
        double total = 0;
        for (std::uint64_t a = 0; a < num_arrays; ++a) {
            KeyArray keys(in + a * len, in + (a + 1) * len);
            auto prep = network == 0 ? netsort::prepare_btn(keys, p) : netsort::prepare_oet(keys, p);
            const auto t0 = std::chrono::steady_clock::now();
            auto res = netsort::run_block_network(std::move(prep), true);
            const auto t1 = std::chrono::steady_clock::now();
            total += std::chrono::duration<double>(t1 - t0).count();
            std::memcpy(out + a * len, res.output.data(), len * sizeof(std::uint32_t));
        }
        return total;
    } catch (...) {
        return -1.0;
    }
}

// bench.hpp:131-137 run_once for BTN/OET: run_block_network with its default
// executor, timed around the call (bench CSV rows, scripts/bench_csv.py).
double ref_time_network_once(int network, const std::uint32_t* in, std::uint64_t len, int p, std::uint32_t* out) {
    try {
        KeyArray keys(in, in + len);
        auto prep = network == 0 ? netsort::prepare_btn(keys, p) : netsort::prepare_oet(keys, p);
        const auto t0 = std::chrono::steady_clock::now();
        auto res = netsort::run_block_network(std::move(prep));
        const auto t1 = std::chrono::steady_clock::now();
        std::memcpy(out, res.output.data(), len * sizeof(std::uint32_t));
        return std::chrono::duration<double>(t1 - t0).count();
    } catch (...) {
        return -1.0;
    }
}

// The 5-way dispatch of bspsort.hpp:15-25 (that header needs Boost).
// algorithm: 0 SR4, 1 PR4, 2 PR2, 3 BTN, 4 OET (core.hpp:24 order).
int ref_sort_instance(const std::uint32_t* in, std::uint64_t n, int processors, int algorithm,
                      std::uint64_t radix, std::uint32_t* out) {
    return guard([&] {
        SortInstance inst;
        inst.input.assign(in, in + n);
        inst.processors = processors;
        inst.algorithm = static_cast<Algorithm>(algorithm);
        inst.radix = radix;
        inst.validate();
        KeyArray r;
        switch (inst.algorithm) {
        case Algorithm::SR4: r = radix::serial_radix_sort(inst.input, inst.radix); break;
        case Algorithm::PR4:
        case Algorithm::PR2: r = radix::parallel_radix_sort(inst); break;
        case Algorithm::BTN: r = netsort::btn_sort(inst); break;
        case Algorithm::OET: r = netsort::oet_sort(inst); break;
        }
        std::memcpy(out, r.data(), r.size() * sizeof(std::uint32_t));
    });
}

} // extern "C"
