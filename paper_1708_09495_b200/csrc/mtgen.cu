// mtgen.cu -- generate_uniform_keys (core.hpp:93-99: std::mt19937_64(seed),
// low 32 bits of each draw) on the GPU, bit-identical to the host stream
// (SURVEY §8(f)4), and random access into that stream on the host.
//
// MT19937-64 as a sequence: x[0..311] = seeded state, and for k >= 0
//   x[k+312] = x[k+156] ^ (y >> 1) ^ (y & 1 ? A : 0),
//   y = (x[k] & UPPER33) | (x[k+1] & LOWER31);
// draw j = temper(x[312 + j]).  From index 312 on, every bit position of the
// word sequence satisfies the characteristic recurrence P(E) x = 0 of the
// 19937-bit state transition (the seed word's low 31 bits are outside the
// state, so jumps start from the window x[312..623]).  With
// q(x) = x^J mod P(x), x[k+J+i] = sum_j q_j x[k+j+i]  (GF(2) sums of words).
//
//   host   : P by Berlekamp-Massey on bit 0 of the sequence (once per
//            process); q = x^J mod P by square-and-multiply (cached per J).
//   device : jump = Horner over q in blocks of 156 coefficients: the 156
//            words x[k+312 .. k+467] depend only on x[k .. k+311], so one
//            block step is a parallel T^156 of the accumulator plus a GF(2)
//            convolution of the 156 coefficient bits with the source window
//            extended by 155 words.  Segment start states come from log2(S)
//            rounds of jumps (tree doubling); each CTA then emits its
//            segment window by window (312 tempered words, two 156-word
//            half twists).
#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "context.cuh"
#include "timer.cuh"

namespace bsg {
namespace mt {

constexpr int NW = 312, MW = 156;
constexpr int DEG = 19937;
constexpr uint64_t MATRIX_A = 0xB5026F5AA96619E9ull;
constexpr uint64_t UPPER = 0xFFFFFFFF80000000ull, LOWER = 0x7FFFFFFFull;
constexpr int PW = (DEG + 64) / 64;      // words of a reduced polynomial (degree < DEG)
constexpr int NBLK = (DEG + MW - 1) / MW; // 156-coefficient Horner blocks

__host__ __device__ __forceinline__ uint64_t rec(uint64_t a, uint64_t b, uint64_t c) {
    const uint64_t y = (a & UPPER) | (b & LOWER);
    return c ^ (y >> 1) ^ ((y & 1ull) ? MATRIX_A : 0ull);
}
__host__ __device__ __forceinline__ uint64_t temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
}

// x[312 .. 623] for a seed (the std::mersenne_twister_engine seeding + first twist).
void base_window(uint64_t seed, uint64_t* win) {
    uint64_t x[NW];
    x[0] = seed;
    for (int i = 1; i < NW; ++i) x[i] = 6364136223846793005ull * (x[i - 1] ^ (x[i - 1] >> 62)) + static_cast<uint64_t>(i);
    for (int i = 0; i < NW; ++i) {
        const uint64_t a = x[i], b = i + 1 < NW ? x[i + 1] : win[0];
        const uint64_t c = i + MW < NW ? x[i + MW] : win[i + MW - NW];
        win[i] = rec(a, b, c);
    }
}

using Poly = std::vector<uint64_t>;

// P(x) (monic, degree DEG) by Berlekamp-Massey on bit 0 of x[312 ..].
const Poly& char_poly() {
    static Poly P;
    static std::once_flag once;
    std::call_once(once, [] {
        const int N = 2 * DEG + 64;
        std::vector<uint64_t> win(NW);
        base_window(5489ull, win.data());
        std::vector<uint64_t> xs(win.begin(), win.end());
        xs.reserve(N + NW);
        for (int k = 0; static_cast<int>(xs.size()) < N; ++k) xs.push_back(rec(xs[k], xs[k + 1], xs[k + MW]));
        // reversed bit sequence rs[j] = s[N-1-j] (s_n = bit 0 of xs[n])
        const int RW = (N + 63) / 64 + 2;
        std::vector<uint64_t> rs(RW, 0);
        for (int n = 0; n < N; ++n)
            if (xs[n] & 1ull) {
                const int j = N - 1 - n;
                rs[j >> 6] |= 1ull << (j & 63);
            }
        const int CW = (DEG + 64) / 64 + 2;
        std::vector<uint64_t> C(CW, 0), B(CW, 0), T;
        C[0] = B[0] = 1;
        int L = 0, m = 1;
        auto rs_word = [&](int off) -> uint64_t { // 64 bits of rs starting at bit off
            const int w = off >> 6, sh = off & 63;
            const uint64_t lo = w < RW ? rs[w] : 0, hi = w + 1 < RW ? rs[w + 1] : 0;
            return sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
        };
        for (int n = 0; n < N; ++n) {
            // d = s_n + sum_{i=1..L} C_i s_{n-i};  s_{n-i} = rs[N-1-n+i]
            uint64_t acc = 0;
            const int base = N - 1 - n; // rs index of s_n; C_i pairs with rs[base + i]
            for (int w = 0; w * 64 <= L; ++w) acc ^= C[w] & rs_word(base + w * 64);
            const int d = __builtin_popcountll(acc) & 1; // C_0 = 1 pairs with s_n itself
            if (!d) {
                ++m;
                continue;
            }
            T = C;
            // C ^= B << m
            const int ws = m >> 6, bs = m & 63;
            for (int w = CW - 1; w >= ws; --w) {
                uint64_t v = B[w - ws] << bs;
                if (bs && w - ws - 1 >= 0) v |= B[w - ws - 1] >> (64 - bs);
                C[w] ^= v;
            }
            if (2 * L <= n) {
                L = n + 1 - L;
                B = T;
                m = 1;
            } else {
                ++m;
            }
        }
        // characteristic polynomial = reciprocal of the connection polynomial
        P.assign(PW + 1, 0);
        for (int k = 0; k <= L; ++k)
            if ((C[(L - k) >> 6] >> ((L - k) & 63)) & 1ull) P[k >> 6] |= 1ull << (k & 63);
        if (L != DEG) P.clear(); // must not happen; callers check
    });
    return P;
}

// a (degree < 2*DEG) reduced mod P in place; result has PW meaningful words.
void reduce(Poly& a, const Poly& P) {
    static std::vector<Poly> shifted; // P << s, s = 0..63
    static std::once_flag once;
    std::call_once(once, [&] {
        shifted.assign(64, Poly(PW + 2, 0));
        for (int s = 0; s < 64; ++s)
            for (int w = 0; w <= PW; ++w) {
                shifted[s][w] ^= P[w] << s;
                if (s) shifted[s][w + 1] ^= P[w] >> (64 - s);
            }
    });
    for (int i = static_cast<int>(a.size()) * 64 - 1; i >= DEG; --i) {
        if (!((a[i >> 6] >> (i & 63)) & 1ull)) continue;
        const int off = i - DEG, wo = off >> 6, so = off & 63;
        const Poly& sp = shifted[so];
        for (int w = 0; w < PW + 2 && w + wo < static_cast<int>(a.size()); ++w) a[w + wo] ^= sp[w];
    }
    a.resize(PW);
}

Poly square(const Poly& a, const Poly& P) {
    Poly r(2 * PW + 2, 0);
    for (int w = 0; w < PW; ++w) {
        uint64_t v = a[w];
        uint64_t lo = 0, hi = 0;
        for (int b = 0; b < 32; ++b) {
            lo |= ((v >> b) & 1ull) << (2 * b);
            hi |= ((v >> (b + 32)) & 1ull) << (2 * b);
        }
        r[2 * w] = lo;
        r[2 * w + 1] = hi;
    }
    reduce(r, P);
    return r;
}

Poly times_x(const Poly& a, const Poly& P) {
    Poly r(PW + 1, 0);
    for (int w = PW; w >= 0; --w) r[w] = (w < PW ? a[w] << 1 : 0) | (w > 0 ? a[w - 1] >> 63 : 0);
    reduce(r, P);
    return r;
}

// x^J mod P
Poly x_pow(uint64_t J, const Poly& P) {
    Poly r(PW, 0);
    r[0] = 1;
    if (J == 0) return r;
    const int top = 63 - __builtin_clzll(J);
    for (int b = top; b >= 0; --b) {
        r = square(r, P);
        if ((J >> b) & 1ull) r = times_x(r, P);
    }
    return r;
}

// Host jump: win <- window x[k+J ..] from window x[k ..] (k >= 312).
void jump_host(uint64_t* win, const Poly& q) {
    std::vector<uint64_t> ext(NW + MW), acc(NW, 0), nxt(NW);
    for (int i = 0; i < NW; ++i) ext[i] = win[i];
    for (int i = 0; i < MW; ++i) ext[NW + i] = rec(ext[i], ext[i + 1], ext[i + MW]);
    for (int blk = NBLK - 1; blk >= 0; --blk) {
        // acc <- T^156(acc): x[k+156+w] is acc[w+156] for w < 156, and for
        // w >= 156 x[k+156+w] = rec(x[k+w-156], x[k+w-155], x[k+w])
        for (int w = 0; w < MW; ++w) nxt[w] = acc[w + MW];
        for (int w = MW; w < NW; ++w) nxt[w] = rec(acc[w - MW], acc[w - MW + 1], acc[w]);
        acc.swap(nxt);
        for (int j = 0; j < MW; ++j) {
            const int e = blk * MW + j;
            if (e >= DEG || !((q[e >> 6] >> (e & 63)) & 1ull)) continue;
            for (int w = 0; w < NW; ++w) acc[w] ^= ext[j + w];
        }
    }
    for (int i = 0; i < NW; ++i) win[i] = acc[i];
}

// ---- device ---------------------------------------------------------------
constexpr int kThreads = NW; // one thread per window word

// dst state = jump(src state, q); one CTA per jump (tree round: dst in
// [first_dst, first_dst + gridDim.x), src = dst - stride).  Three thread
// groups of 312 split each block's 156 coefficients (52 each, set bits only)
// and XOR their partial convolutions.
constexpr int kJumpGroups = 3, kJumpSpan = MW / kJumpGroups; // 52
__global__ void __launch_bounds__(kThreads * kJumpGroups)
    mt_jump_kernel(uint64_t* __restrict__ states, const uint64_t* __restrict__ q, uint32_t first_dst,
                   uint32_t stride) {
    __shared__ uint64_t s_ext[NW + MW];
    __shared__ uint64_t s_acc[NW];
    __shared__ uint64_t s_part[kJumpGroups][NW];
    __shared__ uint64_t s_q[PW + 1];
    const int g = threadIdx.x / kThreads, w = threadIdx.x - g * kThreads;
    const uint32_t dst = first_dst + blockIdx.x, src = dst - stride;
    if (g == 0) {
        s_ext[w] = states[static_cast<uint64_t>(src) * NW + w];
        s_acc[w] = 0;
    }
    for (int i = threadIdx.x; i <= PW; i += kThreads * kJumpGroups) s_q[i] = i < PW ? q[i] : 0;
    __syncthreads();
    if (g == 0 && w < MW) s_ext[NW + w] = rec(s_ext[w], s_ext[w + 1], s_ext[w + MW]);
    __syncthreads();
    for (int blk = NBLK - 1; blk >= 0; --blk) {
        // this group's 52 coefficients: bits [e0, e0 + 52) of q
        const int e0 = blk * MW + g * kJumpSpan;
        const int wo = e0 >> 6, so = e0 & 63;
        uint64_t bits = (s_q[wo] >> so) | (so ? s_q[wo + 1] << (64 - so) : 0ull);
        bits &= (1ull << kJumpSpan) - 1;
        if (e0 + kJumpSpan > DEG) bits &= (DEG > e0) ? ((1ull << (DEG - e0)) - 1) : 0ull;
        uint64_t v = 0;
        const uint64_t* ext = s_ext + g * kJumpSpan + w;
        while (bits) {
            const int j = __ffsll(static_cast<long long>(bits)) - 1;
            bits &= bits - 1;
            v ^= ext[j];
        }
        if (g == 0) { // acc <- T^156(acc)
            v ^= (w < MW) ? s_acc[w + MW] : rec(s_acc[w - MW], s_acc[w - MW + 1], s_acc[w]);
        }
        s_part[g][w] = v;
        __syncthreads();
        if (g == 0) s_acc[w] = s_part[0][w] ^ s_part[1][w] ^ s_part[2][w];
        __syncthreads();
    }
    if (g == 0) states[static_cast<uint64_t>(dst) * NW + w] = s_acc[w];
}

// Segment s emits draws [s*L, min((s+1)*L, n)) from its start window.
__global__ void __launch_bounds__(kThreads)
    mt_gen_kernel(const uint64_t* __restrict__ states, uint32_t* __restrict__ out, uint64_t n, uint64_t L) {
    __shared__ uint64_t s_win[NW];
    const int w = threadIdx.x;
    const uint64_t begin = static_cast<uint64_t>(blockIdx.x) * L;
    if (begin >= n) return;
    const uint64_t end = std::min<uint64_t>(begin + L, n);
    uint64_t x = states[static_cast<uint64_t>(blockIdx.x) * NW + w];
    s_win[w] = x;
    __syncthreads();
    for (uint64_t base = begin;; base += NW) {
        if (base + w < end) out[base + w] = static_cast<uint32_t>(temper(x));
        if (base + NW >= end) break;
        // next window: x'[w] = rec(x[w], x[w+1], x[w+156]) for w < 156, then
        // x'[w] = rec(x[w], x[w+1] (x'[0] for w = 311), x'[w-156]) for w >= 156
        uint64_t nx = 0;
        if (w < MW) nx = rec(x, s_win[w + 1], s_win[w + MW]);
        __syncthreads();
        if (w < MW) s_win[w] = nx;
        __syncthreads();
        if (w >= MW) nx = rec(x, w + 1 < NW ? s_win[w + 1] : s_win[0], s_win[w - MW]);
        // s_win[w+1] for w >= 156 is still the old word x[w+1] (not yet overwritten)
        __syncthreads();
        if (w >= MW) s_win[w] = nx;
        x = nx;
        __syncthreads();
    }
}

struct JumpCache {
    std::mutex mu;
    std::map<uint64_t, std::vector<Poly>> by_len; // L -> [x^(L 2^k) mod P]
};
JumpCache& jump_cache() {
    static JumpCache c;
    return c;
}

} // namespace mt
} // namespace bsg

extern "C" {

int bsg_generate_uniform_at_u32(uint32_t* out, uint64_t n, uint64_t seed, uint64_t offset) {
    using namespace bsg;
    using namespace bsg::mt;
    if (n && !out) return fail(BSG_EINVAL, "generate_uniform_at: null output");
    const Poly& P = char_poly();
    if (P.empty()) return fail(BSG_EPROTO, "mt19937_64 characteristic polynomial: unexpected degree");
    uint64_t win[NW];
    base_window(seed, win);
    if (offset) jump_host(win, x_pow(offset, P));
    uint64_t i = 0;
    while (i < n) {
        for (int w = 0; w < NW && i < n; ++w, ++i) out[i] = static_cast<uint32_t>(temper(win[w]));
        if (i >= n) break;
        uint64_t nx[NW];
        for (int w = 0; w < MW; ++w) nx[w] = rec(win[w], win[w + 1], win[w + MW]);
        for (int w = MW; w < NW; ++w) nx[w] = rec(win[w], w + 1 < NW ? win[w + 1] : nx[0], nx[w - MW]);
        for (int w = 0; w < NW; ++w) win[w] = nx[w];
    }
    return BSG_OK;
}

int bsg_generate_uniform_device_u32(bsg_ctx* ctx, uint32_t* out, uint64_t n, uint64_t seed, void* stream) {
    return bsg_generate_uniform_device_at_u32(ctx, out, n, seed, 0, stream);
}

int bsg_generate_uniform_device_at_u32(bsg_ctx* ctx, uint32_t* out, uint64_t n, uint64_t seed, uint64_t offset,
                                       void* stream) {
    using namespace bsg;
    using namespace bsg::mt;
    if (!ctx) return fail(BSG_EINVAL, "null context");
    if (n && !out) return fail(BSG_EINVAL, "generate_uniform_device: null output");
    if (n == 0) return BSG_OK;
    const Poly& P = char_poly();
    if (P.empty()) return fail(BSG_EPROTO, "mt19937_64 characteristic polynomial: unexpected degree");
    // segments of >= 2^18 draws, at most 4096
    const uint64_t S = std::max<uint64_t>(1, std::min<uint64_t>(4096, (n + (1ull << 18) - 1) >> 18));
    const uint64_t L = (n + S - 1) / S;
    int rounds = 0;
    while ((1ull << rounds) < S) ++rounds;
    std::vector<Poly> qs;
    {
        JumpCache& jc = jump_cache();
        std::lock_guard<std::mutex> lk(jc.mu);
        auto& v = jc.by_len[L];
        if (static_cast<int>(v.size()) < rounds) {
            if (v.empty()) v.push_back(x_pow(L, P));
            while (static_cast<int>(v.size()) < rounds) v.push_back(square(v.back(), P));
        }
        qs.assign(v.begin(), v.begin() + rounds);
    }
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceGuard dev(ctx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder order(ctx, st);
    const uint64_t words = S * NW + static_cast<uint64_t>(std::max(rounds, 1)) * PW;
    cudaError_t e = ctx->mt_ws.ensure(words * sizeof(uint64_t));
    if (e != cudaSuccess) return cuda_fail(e, "generator workspace");
    uint64_t* states = ctx->mt_ws.as<uint64_t>();
    uint64_t* qdev = states + S * NW;
    std::vector<uint64_t> host(NW + static_cast<uint64_t>(rounds) * PW);
    base_window(seed, host.data());
    if (offset) jump_host(host.data(), x_pow(offset, P)); // draws [offset, offset + n) of the stream
    for (int k = 0; k < rounds; ++k) std::copy(qs[k].begin(), qs[k].begin() + PW, host.begin() + NW + k * PW);
    // pageable copies are synchronous w.r.t. the host buffer, which then may go out of scope
    if ((e = cudaMemcpyAsync(states, host.data(), NW * sizeof(uint64_t), cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (rounds && (e = cudaMemcpyAsync(qdev, host.data() + NW, static_cast<uint64_t>(rounds) * PW * sizeof(uint64_t),
                                        cudaMemcpyHostToDevice, st)) != cudaSuccess) ||
        (e = cudaStreamSynchronize(st)) != cudaSuccess)
        return cuda_fail(e, "generator upload");
    for (int k = 0; k < rounds; ++k) {
        const uint64_t first = 1ull << k, last = std::min<uint64_t>(2ull << k, S);
        mt_jump_kernel<<<static_cast<unsigned>(last - first), kThreads * kJumpGroups, 0, st>>>(states, qdev + k * PW,
                                                                                 static_cast<uint32_t>(first),
                                                                                 static_cast<uint32_t>(first));
        ++ctx->launches;
    }
    mt_gen_kernel<<<static_cast<unsigned>(S), kThreads, 0, st>>>(states, out, n, L);
    ++ctx->launches;
    if ((e = cudaPeekAtLastError()) != cudaSuccess) return cuda_fail(cudaGetLastError(), "generator launch");
    return BSG_OK;
}

} // extern "C"
