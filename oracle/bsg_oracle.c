/*
 * bsg_oracle.c -- CPU restatement of the reference's integer-sorting hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker (or the timed CPU baseline) -- never as the product
 * path.  The product (paper_1708_09495_b200/libbsg.so) has no CPU fallback.
 *
 * Every function restates one reference function (file:line relative to
 * /root/reference/proj/include/bspsort/).  Parity of this restatement is
 * pinned against (1) the reference's own known-answer tests (frozen
 * generator draws core_test.cpp:24-31, count_sort_round KATs
 * radix_test.cpp:142-151, merge_split KATs netsort_test.cpp:52-82, the
 * reverse-block OET KAT netsort_test.cpp:211-215) -- see
 * tests/test_oracle_golden.py -- and (2) the reference's own headers compiled
 * into oracle/_ref/libbspref.so by oracle/Makefile (checked against it by tests/test_oracle_golden.py::test_oracle_vs_reference_live).
 *
 * Plain C99, single-threaded, no allocation hidden from the caller except
 * where noted (scratch via malloc, freed before return).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ENOMEM 4
#define ORC_EPROTO 2

/* ---------------------------------------------------------------------- */
/* core.hpp:93-99 generate_uniform_keys: std::mt19937_64(seed), low 32 bits */
/* of each draw.  mt19937_64 parameters are fixed by the C++ standard.      */
/* ---------------------------------------------------------------------- */
typedef struct { uint64_t mt[312]; int idx; } orc_mt64;

static void orc_mt64_seed(orc_mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

static uint64_t orc_mt64_next(orc_mt64* s) {
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t y = s->mt[s->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

void orc_generate_uniform_keys(uint32_t* out, uint64_t n, uint64_t seed) {
    orc_mt64 s;
    orc_mt64_seed(&s, seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = (uint32_t)orc_mt64_next(&s);
}

/* Raw 64-bit draws, used by tests that restate the reference tests' own   */
/* std::mt19937_64 streams (e.g. radix_test.cpp:67-83 index tagging).       */
void orc_mt64_draws(uint64_t* out, uint64_t n, uint64_t seed) {
    orc_mt64 s;
    orc_mt64_seed(&s, seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = orc_mt64_next(&s);
}

/* bench.hpp:77-88 splitmix64 / derive_seed */
uint64_t orc_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t orc_derive_seed(uint64_t seed, int rep) {
    return orc_splitmix64(seed ^ orc_splitmix64((uint64_t)(int64_t)rep));
}

/* core.hpp:60-64 digit_bits + radix.hpp:32-40 checked_digit_bits:        */
/* returns lg r, or -1 if r is not a power of two whose width divides 32,  */
/* or -2 if lg r > 16.                                                      */
int orc_checked_digit_bits(uint64_t radix) {
    if (radix == 0 || (radix & (radix - 1)) != 0) return -1;
    int b = 0;
    while ((1ULL << b) != radix) ++b;
    if (b == 0 || 32 % b != 0) return -1;
    if (b > 16) return -2;
    return b;
}

/* radix.hpp:28-30 digit_of */
static inline uint32_t orc_digit_of(uint32_t key, int round, int bits) {
    return (uint32_t)(((uint64_t)key >> (round * bits)) & ((1ULL << bits) - 1));
}

/* radix.hpp:44-65 count_sort_round: histogram, exclusive scan, forward   */
/* stable scatter.                                                          */
int orc_count_sort_round(const uint32_t* keys, uint64_t n, int round, uint64_t radix, uint32_t* out) {
    const int bits = orc_checked_digit_bits(radix);
    if (bits < 0) return ORC_EINVAL;
    if (round < 0 || round >= 32 / bits) return ORC_EINVAL;
    uint64_t* counts = (uint64_t*)calloc(radix, sizeof(uint64_t));
    if (!counts) return ORC_ENOMEM;
    for (uint64_t i = 0; i < n; ++i) ++counts[orc_digit_of(keys[i], round, bits)];
    uint64_t running = 0;
    for (uint64_t d = 0; d < radix; ++d) {
        uint64_t c = counts[d];
        counts[d] = running;
        running += c;
    }
    for (uint64_t i = 0; i < n; ++i) out[counts[orc_digit_of(keys[i], round, bits)]++] = keys[i];
    free(counts);
    return ORC_OK;
}

/* radix.hpp:69-90 serial_radix_sort: 32/lg r rounds with ping-pong.     */
/* `out` receives the sorted keys; `in` is not modified.                    */
int orc_serial_radix_sort(const uint32_t* in, uint64_t n, uint64_t radix, uint32_t* out) {
    const int bits = orc_checked_digit_bits(radix);
    if (bits < 0) return ORC_EINVAL;
    const int rounds = 32 / bits;
    uint32_t* buf = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    uint64_t* counts = (uint64_t*)malloc(radix * sizeof(uint64_t));
    if (!buf || !counts) { free(buf); free(counts); return ORC_ENOMEM; }
    memcpy(out, in, n * sizeof(uint32_t));
    uint32_t* keys = out;
    uint32_t* other = buf;
    for (int round = 0; round < rounds; ++round) {
        memset(counts, 0, radix * sizeof(uint64_t));
        for (uint64_t i = 0; i < n; ++i) ++counts[orc_digit_of(keys[i], round, bits)];
        uint64_t running = 0;
        for (uint64_t d = 0; d < radix; ++d) {
            uint64_t c = counts[d];
            counts[d] = running;
            running += c;
        }
        for (uint64_t i = 0; i < n; ++i) other[counts[orc_digit_of(keys[i], round, bits)]++] = keys[i];
        uint32_t* t = keys; keys = other; other = t;
    }
    /* rounds is even for every legal radix except r=2^32 (rejected), so the */
    /* result is back in `out`; copy defensively otherwise.                  */
    if (keys != out) memcpy(out, keys, n * sizeof(uint32_t));
    free(buf);
    free(counts);
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* radix.hpp:96-118 detail::Partition (balanced contiguous cut)           */
/* ---------------------------------------------------------------------- */
uint64_t orc_part_size_of(uint64_t n, int p, int w) {
    return n / (uint64_t)p + ((uint64_t)w < n % (uint64_t)p ? 1 : 0);
}
uint64_t orc_part_offset_of(uint64_t n, int p, int w) {
    uint64_t uw = (uint64_t)w, big = n % (uint64_t)p;
    return uw * (n / (uint64_t)p) + (uw < big ? uw : big);
}
int orc_part_owner_of(uint64_t n, int p, uint64_t pos) {
    uint64_t small = n / (uint64_t)p, bigc = n % (uint64_t)p;
    uint64_t big = small + 1, split = bigc * big;
    if (pos < split) return (int)(pos / big);
    return (int)(bigc + (pos - split) / small);
}

typedef struct {
    int supersteps;
    uint64_t messages_sent, messages_delivered, words_sent, words_delivered;
} orc_run_stats;

/* radix.hpp:233-303 prepare_parallel_radix + run_parallel_radix, with      */
/* plan.rounds overridable (rounds_limit < 0 => all 32/lg r rounds), the   */
/* per-round oracle of SURVEY §8(c).  Restates the BSP program directly:   */
/* per round every worker counts its digits (radix.hpp:127-132) and sends  */
/* the count block to all p workers (radix.hpp:275-277); then sorts its   */
/* block with count_sort_round, routes each key to owner_of(next_pos)      */
/* (radix.hpp:151-179); the owner rebuilds its block by walking (digit,    */
/* source) and clipping (radix.hpp:184-222).  Output = concatenation of   */
/* final blocks in worker order (radix.hpp:297-302).  Stats follow          */
/* bsp.hpp:50-58,139-148 (words = payload sizes).                          */
int orc_parallel_radix(const uint32_t* in, uint64_t n, int p, uint64_t radix, int rounds_limit,
                       uint32_t* out, orc_run_stats* stats) {
    if (p < 1) return ORC_EINVAL;
    const int bits = orc_checked_digit_bits(radix);
    if (bits < 0) return ORC_EINVAL;
    int rounds = 32 / bits;
    if (rounds_limit >= 0 && rounds_limit < rounds) rounds = rounds_limit;

    uint32_t** blocks = (uint32_t**)calloc((size_t)p, sizeof(uint32_t*));
    uint64_t* counts = (uint64_t*)calloc((size_t)p * radix, sizeof(uint64_t)); /* counts[v*r+d] */
    uint64_t* starts = (uint64_t*)calloc(radix + 1, sizeof(uint64_t));
    uint64_t* next_pos = (uint64_t*)calloc(radix, sizeof(uint64_t));
    uint32_t* sorted = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    /* routed[v] holds worker v's digit-sorted block; slices are contiguous */
    /* ranges of it, [slice_lo[v*p+w], slice_hi[v*p+w]).                   */
    uint32_t** routed = (uint32_t**)calloc((size_t)p, sizeof(uint32_t*));
    uint64_t* slice_lo = (uint64_t*)calloc((size_t)p * p, sizeof(uint64_t));
    uint64_t* slice_hi = (uint64_t*)calloc((size_t)p * p, sizeof(uint64_t));
    uint64_t* cursor = (uint64_t*)calloc((size_t)p, sizeof(uint64_t));
    int rc = ORC_OK;
    if (!blocks || !counts || !starts || !next_pos || !sorted || !routed || !slice_lo || !slice_hi || !cursor) {
        rc = ORC_ENOMEM;
        goto done;
    }
    for (int w = 0; w < p; ++w) {
        uint64_t sz = orc_part_size_of(n, p, w);
        blocks[w] = (uint32_t*)malloc((sz ? sz : 1) * sizeof(uint32_t));
        routed[w] = (uint32_t*)malloc((sz ? sz : 1) * sizeof(uint32_t));
        if (!blocks[w] || !routed[w]) { rc = ORC_ENOMEM; goto done; }
        memcpy(blocks[w], in + orc_part_offset_of(n, p, w), sz * sizeof(uint32_t));
    }
    orc_run_stats st = {0, 0, 0, 0, 0};

    for (int round = 0; round < rounds; ++round) {
        /* superstep 2*round: count_digits + send to all (radix.hpp:275-277) */
        memset(counts, 0, (size_t)p * radix * sizeof(uint64_t));
        for (int w = 0; w < p; ++w) {
            uint64_t sz = orc_part_size_of(n, p, w);
            for (uint64_t i = 0; i < sz; ++i) ++counts[(uint64_t)w * radix + orc_digit_of(blocks[w][i], round, bits)];
        }
        st.messages_sent += (uint64_t)p * p;
        st.words_sent += (uint64_t)p * p * radix;
        /* digit_starts (radix.hpp:137-145) */
        memset(starts, 0, (radix + 1) * sizeof(uint64_t));
        for (int v = 0; v < p; ++v)
            for (uint64_t d = 0; d < radix; ++d) starts[d + 1] += counts[(uint64_t)v * radix + d];
        for (uint64_t d = 0; d < radix; ++d) starts[d + 1] += starts[d];

        /* superstep 2*round+1: sort_and_scatter (radix.hpp:151-179) */
        for (int w = 0; w < p; ++w) {
            uint64_t sz = orc_part_size_of(n, p, w);
            rc = orc_count_sort_round(blocks[w], sz, round, radix, routed[w]);
            if (rc) goto done;
            for (uint64_t d = 0; d < radix; ++d) {
                uint64_t before_me = 0;
                for (int v = 0; v < w; ++v) before_me += counts[(uint64_t)v * radix + d];
                next_pos[d] = starts[d] + before_me;
            }
            for (int dst = 0; dst < p; ++dst) { slice_lo[w * p + dst] = 0; slice_hi[w * p + dst] = 0; }
            int run_dest = -1;
            uint64_t run_begin = 0;
            for (uint64_t i = 0; i < sz; ++i) {
                uint64_t pos = next_pos[orc_digit_of(routed[w][i], round, bits)]++;
                int dest = orc_part_owner_of(n, p, pos);
                if (dest != run_dest) {
                    if (run_dest >= 0) {
                        slice_lo[w * p + run_dest] = run_begin;
                        slice_hi[w * p + run_dest] = i;
                        st.messages_sent += 1;
                        st.words_sent += i - run_begin;
                    }
                    run_dest = dest;
                    run_begin = i;
                }
            }
            if (run_dest >= 0) {
                slice_lo[w * p + run_dest] = run_begin;
                slice_hi[w * p + run_dest] = sz;
                st.messages_sent += 1;
                st.words_sent += sz - run_begin;
            }
        }
        /* superstep 2*round+2 (first half): gather_slices (radix.hpp:184-222) */
        for (int w = 0; w < p; ++w) {
            const uint64_t lo = orc_part_offset_of(n, p, w);
            const uint64_t hi = lo + orc_part_size_of(n, p, w);
            for (int v = 0; v < p; ++v) cursor[v] = slice_lo[v * p + w];
            uint64_t filled = 0;
            for (uint64_t d = 0; d < radix; ++d) {
                uint64_t seg = starts[d];
                for (int v = 0; v < p; ++v) {
                    uint64_t c = counts[(uint64_t)v * radix + d];
                    uint64_t take_lo = seg > lo ? seg : lo;
                    uint64_t take_hi = (seg + c) < hi ? (seg + c) : hi;
                    seg += c;
                    if (take_hi <= take_lo) continue;
                    uint64_t want = take_hi - take_lo;
                    if (cursor[v] + want > slice_hi[v * p + w]) { rc = ORC_EPROTO; goto done; }
                    memcpy(sorted + lo + filled, routed[v] + cursor[v], want * sizeof(uint32_t));
                    cursor[v] += want;
                    filled += want;
                }
            }
            if (filled != hi - lo) { rc = ORC_EPROTO; goto done; }
        }
        for (int w = 0; w < p; ++w)
            memcpy(blocks[w], sorted + orc_part_offset_of(n, p, w), orc_part_size_of(n, p, w) * sizeof(uint32_t));
    }
    st.supersteps = 2 * rounds + 1;
    st.messages_delivered = st.messages_sent;
    st.words_delivered = st.words_sent;
    for (int w = 0; w < p; ++w)
        memcpy(out + orc_part_offset_of(n, p, w), blocks[w], orc_part_size_of(n, p, w) * sizeof(uint32_t));
    if (stats) *stats = st;
done:
    if (blocks) for (int w = 0; w < p; ++w) free(blocks[w]);
    if (routed) for (int w = 0; w < p; ++w) free(routed[w]);
    free(blocks); free(routed); free(counts); free(starts); free(next_pos); free(sorted);
    free(slice_lo); free(slice_hi); free(cursor);
    return rc;
}

/* ---------------------------------------------------------------------- */
/* netsort.hpp:30-51 merge_split: low = |a| smallest, high = |b| largest,  */
/* ties taken from a first.                                                */
/* ---------------------------------------------------------------------- */
void orc_merge_split(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb,
                     uint32_t* low, uint32_t* high) {
    uint64_t i = 0, j = 0, o = 0;
    while (o < na) {
        if (i < na && (j >= nb || a[i] <= b[j])) low[o++] = a[i++];
        else low[o++] = b[j++];
    }
    o = 0;
    while (i < na || j < nb) {
        if (i < na && (j >= nb || a[i] <= b[j])) high[o++] = a[i++];
        else high[o++] = b[j++];
    }
}

/* netsort.hpp:70-89 bitonic_schedule.  Writes stage-major arrays          */
/* partner[s*p+i], keep_low[s*p+i]; returns the stage count, or -1.        */
int orc_bitonic_schedule(int p, int* partner, int* keep_low, int cap_stages) {
    if (p < 1 || (p & (p - 1)) != 0) return -1;
    int s = 0;
    for (int k = 2; k <= p; k *= 2)
        for (int j = k / 2; j >= 1; j /= 2) {
            if (s < cap_stages)
                for (int i = 0; i < p; ++i) {
                    int q = i ^ j;
                    int asc = (i & k) == 0;
                    partner[s * p + i] = q;
                    keep_low[s * p + i] = asc ? (i < q) : (i > q);
                }
            ++s;
        }
    return s;
}

/* netsort.hpp:95-108 odd_even_rounds: p rounds; round r pairs (i, i+1)    */
/* from i = r%2; lower index keeps low; edge worker idles (partner -1).   */
int orc_odd_even_rounds(int p, int* partner, int* keep_low, int cap_stages) {
    if (p < 1) return -1;
    for (int r = 0; r < p && r < cap_stages; ++r) {
        for (int i = 0; i < p; ++i) { partner[r * p + i] = -1; keep_low[r * p + i] = 0; }
        for (int i = r % 2; i + 1 < p; i += 2) {
            partner[r * p + i] = i + 1; keep_low[r * p + i] = 1;
            partner[r * p + i + 1] = i; keep_low[r * p + i + 1] = 0;
        }
    }
    return p;
}

static int cmp_u32(const void* x, const void* y) {
    uint32_t a = *(const uint32_t*)x, b = *(const uint32_t*)y;
    return a < b ? -1 : a > b;
}

/* netsort.hpp:124-199 prepare_blocks + run_block_network.  network 0=BTN, */
/* 1=OET.  stages_limit < 0 runs every stage; otherwise only the first     */
/* stages_limit merge-split stages run and `out` receives the padded      */
/* concatenation of block states (len out_len = p*ceil(n/p)) -- the         */
/* per-stage oracle of SURVEY §8(c).  With all stages, out has n keys      */
/* (padding stripped, netsort.hpp:197).  Step 0's local sort is           */
/* serial_radix_sort(.,256) (netsort.hpp:167); any correct sort of a block */
/* gives the identical block, so qsort is used here.                       */
int orc_block_network(int network, const uint32_t* in, uint64_t n, int p, int stages_limit,
                      uint32_t* out, orc_run_stats* stats) {
    if (p < 1) return ORC_EINVAL;
    int max_stages = network == 0 ? 64 * 64 : p;
    int* partner = (int*)malloc(sizeof(int) * (size_t)max_stages * p);
    int* keep_low = (int*)malloc(sizeof(int) * (size_t)max_stages * p);
    if (!partner || !keep_low) { free(partner); free(keep_low); return ORC_ENOMEM; }
    int S = network == 0 ? orc_bitonic_schedule(p, partner, keep_low, max_stages)
                         : orc_odd_even_rounds(p, partner, keep_low, max_stages);
    if (S < 0) { free(partner); free(keep_low); return ORC_EINVAL; }
    int run = (stages_limit >= 0 && stages_limit < S) ? stages_limit : S;
    const uint64_t L = (n + (uint64_t)p - 1) / (uint64_t)p;
    const uint64_t total = L * (uint64_t)p;
    uint32_t* state = (uint32_t*)malloc((total ? total : 1) * sizeof(uint32_t));
    uint32_t* next = (uint32_t*)malloc((total ? total : 1) * sizeof(uint32_t));
    uint32_t* scratch = (uint32_t*)malloc((L ? L : 1) * sizeof(uint32_t));
    if (!state || !next || !scratch) {
        free(partner); free(keep_low); free(state); free(next); free(scratch);
        return ORC_ENOMEM;
    }
    /* prepare_blocks (netsort.hpp:124-141): pad with 0xFFFFFFFF */
    for (uint64_t i = 0; i < total; ++i) state[i] = i < n ? in[i] : 0xFFFFFFFFu;
    for (int w = 0; w < p; ++w) qsort(state + (uint64_t)w * L, L, sizeof(uint32_t), cmp_u32);
    orc_run_stats st = {0, 0, 0, 0, 0};
    /* superstep 0 sends each block to its stage-0 partner; superstep s    */
    /* merges and (if s < S) sends to the stage-s partner                  */
    for (int s = 0; s < run; ++s) {
        for (int w = 0; w < p; ++w) {
            int q = partner[s * p + w];
            uint32_t* mine = state + (uint64_t)w * L;
            uint32_t* dst = next + (uint64_t)w * L;
            if (q < 0) { memcpy(dst, mine, L * sizeof(uint32_t)); continue; }
            st.messages_sent += 1;
            st.words_sent += L;
            uint32_t* theirs = state + (uint64_t)q * L;
            if (keep_low[s * p + w]) orc_merge_split(mine, L, theirs, L, dst, scratch);
            else orc_merge_split(mine, L, theirs, L, scratch, dst);
        }
        uint32_t* t = state; state = next; next = t;
    }
    st.supersteps = 1 + run;
    st.messages_delivered = st.messages_sent;
    st.words_delivered = st.words_sent;
    if (run == S) memcpy(out, state, n * sizeof(uint32_t));
    else memcpy(out, state, total * sizeof(uint32_t));
    if (stats) *stats = st;
    free(partner); free(keep_low); free(state); free(next); free(scratch);
    return ORC_OK;
}
