// host_util.cpp -- host-only parts of the C ABI (no GPU needed): the
// reference's input generator, seed derivation, digit-width validation,
// network schedules, balanced partition and the builder-defined skewed inputs
// of config 3.  These are API surface (core.hpp / netsort.hpp / bench.hpp),
// not a compute fallback.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bsg.h"

namespace bsg {
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
} // namespace bsg

extern "C" {

// core.hpp:93-99
int bsg_generate_uniform_u32(uint32_t* out, uint64_t n, uint64_t seed) {
    if (n && !out) return bsg::fail(BSG_EINVAL, "generate_uniform: null output");
    std::mt19937_64 rng(seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = static_cast<uint32_t>(rng());
    return BSG_OK;
}

static uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// bench.hpp:86-88
uint64_t bsg_derive_seed(uint64_t seed, int32_t rep) {
    return splitmix64(seed ^ splitmix64(static_cast<uint64_t>(static_cast<int64_t>(rep))));
}

// core.hpp:60-64 + radix.hpp:32-40
int bsg_checked_digit_bits(uint64_t radix) {
    if (radix == 0 || (radix & (radix - 1)) != 0) {
        bsg::set_error("radix must be a power of two whose bit width divides 32");
        return -1;
    }
    int b = 0;
    while ((uint64_t{1} << b) != radix) ++b;
    if (b == 0 || 32 % b != 0) {
        bsg::set_error("radix must be a power of two whose bit width divides 32");
        return -1;
    }
    if (b > 16) {
        bsg::set_error("radix " + std::to_string(radix) + " needs a count array larger than memory; use r <= 65536");
        return -1;
    }
    return b;
}

// netsort.hpp:70-89 (BTN) and 95-108 (OET)
int bsg_network_schedule(int network, int p, int32_t* partner, int32_t* keep_low, int cap_stages, int* stages) {
    if (!stages) return bsg::fail(BSG_EINVAL, "network_schedule: null stages");
    if (network == BSG_NET_BTN) {
        if (p < 1 || (p & (p - 1)) != 0)
            return bsg::fail(BSG_EINVAL, "bitonic_schedule: p must be a power of two, got " + std::to_string(p));
        int s = 0;
        for (int k = 2; k <= p; k *= 2)
            for (int j = k / 2; j >= 1; j /= 2) {
                if (s < cap_stages && partner && keep_low)
                    for (int i = 0; i < p; ++i) {
                        const int q = i ^ j;
                        const bool asc = (i & k) == 0;
                        partner[s * p + i] = q;
                        keep_low[s * p + i] = asc ? (i < q) : (i > q);
                    }
                ++s;
            }
        *stages = s;
        return BSG_OK;
    }
    if (network == BSG_NET_OET) {
        if (p < 1) return bsg::fail(BSG_EINVAL, "odd_even_rounds: p must be >= 1");
        for (int r = 0; r < p && r < cap_stages && partner && keep_low; ++r) {
            for (int i = 0; i < p; ++i) {
                partner[r * p + i] = -1;
                keep_low[r * p + i] = 0;
            }
            for (int i = r % 2; i + 1 < p; i += 2) {
                partner[r * p + i] = i + 1;
                keep_low[r * p + i] = 1;
                partner[r * p + i + 1] = i;
                keep_low[r * p + i + 1] = 0;
            }
        }
        *stages = p;
        return BSG_OK;
    }
    return bsg::fail(BSG_EINVAL, "unknown network " + std::to_string(network));
}

// radix.hpp:96-118
uint64_t bsg_partition_size_of(uint64_t n, int p, int w) {
    return n / static_cast<uint64_t>(p) + (static_cast<uint64_t>(w) < n % static_cast<uint64_t>(p) ? 1 : 0);
}
uint64_t bsg_partition_offset_of(uint64_t n, int p, int w) {
    const uint64_t uw = static_cast<uint64_t>(w), big = n % static_cast<uint64_t>(p);
    return uw * (n / static_cast<uint64_t>(p)) + (uw < big ? uw : big);
}
int bsg_partition_owner_of(uint64_t n, int p, uint64_t pos) {
    const uint64_t small = n / static_cast<uint64_t>(p), bigc = n % static_cast<uint64_t>(p);
    const uint64_t big = small + 1, split = bigc * big;
    if (pos < split) return static_cast<int>(pos / big);
    return static_cast<int>(bigc + (pos - split) / small);
}

} // extern "C"

namespace {
// Zipf(s) over ranks 1..N by rejection-inversion (Hoermann & Derflinger 1996),
// driven by mt19937_64 -> 53-bit uniforms.  Builder-defined.
struct ZipfRI {
    double s, N, hx1, hN, sq;
    static double helper1(double x) { return std::fabs(x) > 1e-8 ? std::log1p(x) / x : 1.0 - x * (0.5 - x / 3.0); }
    static double helper2(double x) { return std::fabs(x) > 1e-8 ? std::expm1(x) / x : 1.0 + x * 0.5 * (1.0 + x / 3.0); }
    double h(double x) const { return std::exp(-s * std::log(x)); }
    double H(double x) const {
        const double lx = std::log(x);
        return helper2((1.0 - s) * lx) * lx;
    }
    double Hinv(double x) const {
        double t = x * (1.0 - s);
        if (t < -1.0) t = -1.0;
        return std::exp(helper1(t) * x);
    }
    ZipfRI(double s_, double n_) : s(s_), N(n_) {
        hx1 = H(1.5) - 1.0;
        hN = H(N + 0.5);
        sq = 2.0 - Hinv(H(2.5) - h(2.0));
    }
    uint64_t sample(std::mt19937_64& rng) const {
        while (true) {
            const double u01 = static_cast<double>(rng() >> 11) * (1.0 / 9007199254740992.0);
            const double u = hN + u01 * (hx1 - hN);
            const double x = Hinv(u);
            double k = std::floor(x + 0.5);
            if (k < 1.0) k = 1.0;
            else if (k > N) k = N;
            if (k - x <= sq || u >= H(k + 0.5) - h(k)) return static_cast<uint64_t>(k);
        }
    }
};
} // namespace

extern "C" int bsg_generate_skewed_u32(uint32_t* out, uint64_t n, uint64_t seed, int kind, double zipf_s) {
    if (n && !out) return bsg::fail(BSG_EINVAL, "generate_skewed: null output");
    switch (kind) {
    case 0: {
        std::mt19937_64 rng(seed);
        for (uint64_t i = 0; i < n; ++i) out[i] = static_cast<uint32_t>(rng()) & 0xFFFFu;
        return BSG_OK;
    }
    case 1: {
        if (!(zipf_s > 1.0)) return bsg::fail(BSG_EINVAL, "zipf exponent must be > 1");
        std::mt19937_64 rng(seed);
        ZipfRI z(zipf_s, 4294967296.0);
        for (uint64_t i = 0; i < n; ++i) out[i] = static_cast<uint32_t>(z.sample(rng) - 1);
        return BSG_OK;
    }
    case 2:
        for (uint64_t i = 0; i < n; ++i) out[i] = 0xABCD1234u;
        return BSG_OK;
    default:
        return bsg::fail(BSG_EINVAL, "unknown skewed-input kind " + std::to_string(kind));
    }
}
