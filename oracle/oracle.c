/*
 * oracle.c -- CPU restatement of the dfakit reference algorithms.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain C, single-threaded, written
 * for clarity.  Each function names the reference file:line it restates;
 * paths are relative to /root/reference/proj.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 (the reference seeds it directly: src/generators.cpp:248,
 * src/minimize.cpp:276).                                                    */
/* ------------------------------------------------------------------------ */

#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ull
#define MT_LOWER 0x000000007FFFFFFFull

void or_mt64_seed(or_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (uint32_t i = 1; i < MT_N; ++i) {
        g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + i;
    }
    g->idx = MT_N;
}

uint64_t or_mt64_next(or_mt64* g) {
    if (g->idx >= MT_N) {
        for (uint32_t i = 0; i < MT_N; ++i) {
            uint64_t x = (g->mt[i] & MT_UPPER) | (g->mt[(i + 1) % MT_N] & MT_LOWER);
            uint64_t xa = x >> 1;
            if (x & 1u) xa ^= 0xB5026F5AA96619E9ull;
            g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

/* uniform_int_distribution<uint32_t>: the engine range (2^64-1) exceeds the
 * requested range, so libstdc++ downscales with Lemire's nearly-divisionless
 * method on a 128-bit product. */
uint32_t or_uniform_u32(or_mt64* g, uint32_t lo, uint32_t hi) {
    uint64_t range = (uint64_t)hi - (uint64_t)lo + 1u;
    unsigned __int128 product = (unsigned __int128)or_mt64_next(g) * range;
    uint64_t low = (uint64_t)product;
    if (low < range) {
        uint64_t threshold = (0 - range) % range;
        while (low < threshold) {
            product = (unsigned __int128)or_mt64_next(g) * range;
            low = (uint64_t)product;
        }
    }
    return (uint32_t)(product >> 64) + lo;
}

/* bernoulli_distribution: generate_canonical<double, 53> < p. */
int or_bernoulli(or_mt64* g, double p) {
    double r = (double)or_mt64_next(g) / 18446744073709551616.0;
    if (r >= 1.0) r = 0.99999999999999988898; /* nextafter(1, 0) */
    return r < p;
}

/* ------------------------------------------------------------------------ */
/* Partitions                                                                */
/* ------------------------------------------------------------------------ */

/* src/dfa.cpp:47-58 -- dense ids in order of first occurrence. */
uint32_t or_normalize(const uint32_t* labels, uint32_t n, uint32_t* out) {
    /* labels may be arbitrary 32-bit values; map via an open-addressing table */
    uint32_t cap = 16;
    while (cap < 2u * n + 2u) cap <<= 1;
    uint32_t* keys = (uint32_t*)malloc(sizeof(uint32_t) * cap);
    uint32_t* vals = (uint32_t*)malloc(sizeof(uint32_t) * cap);
    uint8_t* used = (uint8_t*)calloc(cap, 1);
    uint32_t next = 0;
    for (uint32_t q = 0; q < n; ++q) {
        uint32_t x = labels[q];
        uint32_t h = (uint32_t)((x * 0x9E3779B97F4A7C15ull) >> 32) & (cap - 1);
        while (used[h] && keys[h] != x) h = (h + 1) & (cap - 1);
        if (!used[h]) {
            used[h] = 1;
            keys[h] = x;
            vals[h] = next++;
        }
        out[q] = vals[h];
    }
    free(keys);
    free(vals);
    free(used);
    return next;
}

/* ------------------------------------------------------------------------ */
/* Generators (src/generators.cpp)                                          */
/* ------------------------------------------------------------------------ */

/* src/generators.cpp:241-263: targets letter by letter, then acceptance. */
int or_gen_random(uint32_t n, uint32_t k, double frac, uint64_t seed, uint32_t* delta, uint8_t* acc) {
    if (n < 1 || k < 1 || frac < 0.0 || frac > 1.0) return -1;
    or_mt64 g;
    or_mt64_seed(&g, seed);
    for (uint32_t a = 0; a < k; ++a)
        for (uint32_t q = 0; q < n; ++q) delta[(size_t)a * n + q] = or_uniform_u32(&g, 0, n - 1);
    for (uint32_t q = 0; q < n; ++q) acc[q] = (uint8_t)or_bernoulli(&g, frac);
    return 0;
}

/* src/generators.cpp:22-52: |bits(0)| = |bits(1)| = 1, Fibonacci after. */
uint64_t or_fib_word_len(uint32_t m) {
    uint64_t prev = 1, cur = 1;
    for (uint32_t i = 2; i <= m; ++i) {
        uint64_t nx = prev + cur;
        prev = cur;
        cur = nx;
    }
    return cur;
}

/* bits(0) = 1, bits(1) = 0, bits(i) = bits(i-1) ++ bits(i-2); gen_fib at
 * src/generators.cpp:66-79 (cyclic successor, accepting at the 1-bits). */
int or_gen_fib(uint32_t m, uint32_t* delta, uint8_t* acc) {
    if (m < 2) return -1;
    uint64_t n = or_fib_word_len(m);
    uint8_t* prev = (uint8_t*)malloc(n);
    uint8_t* cur = (uint8_t*)malloc(n);
    uint64_t lp = 1, lc = 1;
    prev[0] = 1;
    cur[0] = 0;
    for (uint32_t i = 2; i <= m; ++i) {
        /* next = cur ++ prev; write it into prev's buffer after shifting */
        uint8_t* nx = (uint8_t*)malloc(n);
        uint64_t ln = lc + lp;
        memcpy(nx, cur, lc);
        memcpy(nx + lc, prev, lp);
        free(prev);
        prev = cur;
        lp = lc;
        cur = nx;
        lc = ln;
    }
    for (uint64_t q = 0; q < n; ++q) {
        delta[q] = (uint32_t)((q + 1) % n);
        acc[q] = cur[q];
    }
    free(prev);
    free(cur);
    return 0;
}

/* src/generators.cpp:81-108: letter a_m (id m-1) flips bit m and clears the
 * lower bits when bit m-1 is set; accepting = upper half. */
int or_gen_bitsplitter(uint32_t nb, uint32_t* delta, uint8_t* acc) {
    if (nb < 1 || nb >= 32) return -1;
    uint32_t N = 1u << nb;
    for (uint32_t m = 1; m < nb; ++m) {
        uint32_t test = 1u << (m - 1), flip = 1u << m, clear = ~(flip - 1);
        uint32_t* row = delta + (size_t)(m - 1) * N;
        for (uint32_t q = 0; q < N; ++q) row[q] = (q & test) ? ((q ^ flip) & clear) : q;
    }
    for (uint32_t q = 0; q < N; ++q) acc[q] = q >= (N >> 1);
    return 0;
}

/* src/generators.cpp:110-166: letters r, b_1..b_n, a_1..a_{n-1}. */
int or_gen_bitsplitter_ext(uint32_t nb, uint32_t* delta, uint8_t* acc) {
    if (nb < 1 || nb >= 31) return -1;
    uint32_t N = 1u << (nb + 1), c = 1u << nb, smask = c - 1;
    size_t row = 0;
    for (uint32_t q = 0; q < N; ++q) delta[q] = q | c;
    row = 1;
    for (uint32_t m = 1; m <= nb; ++m, ++row) {
        uint32_t bit = 1u << (m - 1);
        for (uint32_t q = 0; q < N; ++q) delta[row * N + q] = (q & c) ? q : (q | bit);
    }
    for (uint32_t m = 1; m < nb; ++m, ++row) {
        uint32_t test = 1u << (m - 1), flip = 1u << m, clear = ~(flip - 1);
        for (uint32_t q = 0; q < N; ++q)
            delta[row * N + q] = ((q & c) && (q & test)) ? (c | (((q & smask) ^ flip) & clear & smask)) : q;
    }
    uint32_t top = 1u << (nb - 1);
    for (uint32_t q = 0; q < N; ++q) acc[q] = (q & c) && (q & top);
    return 0;
}

/* src/generators.cpp:54-64: fib(1) = 1, fib(2) = 2. */
uint64_t or_cycle_fib(uint32_t m) {
    if (m == 0) return 0;
    uint64_t a = 1, b = 2;
    if (m == 1) return a;
    for (uint32_t i = 3; i <= m; ++i) {
        uint64_t nx = a + b;
        a = b;
        b = nx;
    }
    return b;
}

uint32_t or_cycle_letters(uint32_t m) {
    uint64_t states = or_cycle_fib(m);
    uint32_t cl = 0;
    for (uint64_t p = 1; p < states; p *= 10) ++cl;
    return (cl > 1 ? cl : 1) + 1;
}

/* src/generators.cpp:168-199: letter j steps by j*100+1 (mod N). */
int or_gen_cycle(uint32_t m, uint32_t* delta, uint8_t* acc) {
    if (m < 2 || m > 85) return -1;
    uint64_t states = or_cycle_fib(m);
    uint32_t N = (uint32_t)states, k = or_cycle_letters(m);
    for (uint32_t j = 0; j < k; ++j) {
        uint32_t step = (uint32_t)(((uint64_t)j * 100 + 1) % states);
        for (uint32_t q = 0; q < N; ++q) {
            uint32_t t = q + step;
            if (t >= N) t -= N;
            delta[(size_t)j * N + q] = t;
        }
    }
    memset(acc, 0, N);
    acc[(uint32_t)or_cycle_fib(m - 1)] = 1;
    return 0;
}

/* src/generators.cpp:201-239: shift register; forgetful resets the states
 * whose two top bits read "10". */
int or_gen_memory(uint32_t depth, int forgetful, uint32_t* delta, uint8_t* acc) {
    if (depth < 1 || depth >= 32 || (forgetful && depth < 2)) return -1;
    uint32_t N = 1u << depth, mask = N - 1;
    for (uint32_t v = 0; v < 2; ++v)
        for (uint32_t q = 0; q < N; ++q) delta[(size_t)v * N + q] = ((q << 1) | v) & mask;
    for (uint32_t q = 0; q < N; ++q) acc[q] = (q >> (depth - 1)) & 1u;
    if (forgetful) {
        uint32_t top = 1u << (depth - 1), second = 1u << (depth - 2);
        for (uint32_t v = 0; v < 2; ++v)
            for (uint32_t q = 0; q < N; ++q)
                if ((q & top) && !(q & second)) delta[(size_t)v * N + q] = v;
    }
    return 0;
}

/* tests/test_minimize.cpp:251-262 generalised to n states. */
int or_gen_chain(uint32_t n, uint32_t* delta, uint8_t* acc) {
    if (n < 1) return -1;
    for (uint32_t q = 0; q + 1 < n; ++q) {
        delta[q] = q + 1;
        acc[q] = 0;
    }
    delta[n - 1] = n - 1;
    acc[n - 1] = 1;
    return 0;
}

static inline uint64_t or_mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

/* Synthetic benchmark family (not in the reference): counter-based so the
 * GPU can generate 1B-transition instances in place.  Same formula as
 * dfakit_gen_synth in the product. */
void or_gen_synth(uint32_t n, uint32_t k, uint64_t seed, uint32_t* delta, uint8_t* acc) {
    for (uint64_t a = 0; a < k; ++a)
        for (uint64_t q = 0; q < n; ++q) {
            uint64_t idx = a * n + q;
            uint64_t h = or_mix64(seed ^ (idx * 0xD1B54A32D192ED03ull));
            delta[idx] = (uint32_t)(((h >> 32) * (uint64_t)n) >> 32);
        }
    for (uint64_t q = 0; q < n; ++q) acc[q] = (uint8_t)(or_mix64(~seed ^ (q * 0xD1B54A32D192ED03ull)) >> 63);
}

/* ------------------------------------------------------------------------ */
/* Moore (src/minimize.cpp:42-86)                                            */
/* ------------------------------------------------------------------------ */

static uint64_t sig_hash(const or_dfa* d, const uint32_t* block, uint32_t q) {
    uint64_t h = 1469598103934665603ull;
    h = (h ^ block[q]) * 1099511628211ull;
    for (uint32_t a = 0; a < d->k; ++a) h = (h ^ block[d->delta[(size_t)a * d->n + q]]) * 1099511628211ull;
    return or_mix64(h);
}

static int sig_equal(const or_dfa* d, const uint32_t* block, uint32_t q, uint32_t r) {
    if (block[q] != block[r]) return 0;
    for (uint32_t a = 0; a < d->k; ++a) {
        const uint32_t* row = d->delta + (size_t)a * d->n;
        if (block[row[q]] != block[row[r]]) return 0;
    }
    return 1;
}

uint32_t or_moore(const or_dfa* d, uint32_t* out_block, uint32_t* iters) {
    const uint32_t n = d->n;
    *iters = 0;
    if (n == 0) return 0;
    uint32_t* block = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* next_block = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t ids[2] = {OR_NONE, OR_NONE}, num_blocks = 0;
    for (uint32_t q = 0; q < n; ++q) {
        int c = d->acc[q] ? 1 : 0;
        if (ids[c] == OR_NONE) ids[c] = num_blocks++;
        block[q] = ids[c];
    }
    uint32_t cap = 16;
    while (cap < 2u * n) cap <<= 1;
    uint32_t* rep = (uint32_t*)malloc(sizeof(uint32_t) * cap);
    uint32_t* rid = (uint32_t*)malloc(sizeof(uint32_t) * cap);
    for (;;) {
        for (uint32_t i = 0; i < cap; ++i) rep[i] = OR_NONE;
        uint32_t next = 0;
        for (uint32_t q = 0; q < n; ++q) {
            uint32_t h = (uint32_t)sig_hash(d, block, q) & (cap - 1);
            while (rep[h] != OR_NONE && !sig_equal(d, block, rep[h], q)) h = (h + 1) & (cap - 1);
            if (rep[h] == OR_NONE) {
                rep[h] = q;
                rid[h] = next++;
            }
            next_block[q] = rid[h];
        }
        if (next == num_blocks) break;
        uint32_t* t = block;
        block = next_block;
        next_block = t;
        num_blocks = next;
        ++*iters;
    }
    uint32_t nb = or_normalize(block, n, out_block);
    free(block);
    free(next_block);
    free(rep);
    free(rid);
    return nb;
}

/* ------------------------------------------------------------------------ */
/* sortPR (src/minimize.cpp:354-419)                                         */
/* ------------------------------------------------------------------------ */

typedef struct {
    const uint32_t* block;
    const uint32_t* sig; /* n*k, state-major */
    uint32_t k;
} sort_ctx;

/* COMPARE of src/minimize.cpp:383-391: block first, then letters upwards. */
static int sort_cmp(const sort_ctx* c, uint32_t q1, uint32_t q2) {
    if (c->block[q1] != c->block[q2]) return c->block[q1] < c->block[q2] ? -1 : 1;
    const uint32_t* s1 = c->sig + (size_t)q1 * c->k;
    const uint32_t* s2 = c->sig + (size_t)q2 * c->k;
    for (uint32_t a = 0; a < c->k; ++a)
        if (s1[a] != s2[a]) return s1[a] < s2[a] ? -1 : 1;
    return 0;
}

/* stable merge sort, like std::stable_sort */
static void merge_sort(const sort_ctx* c, uint32_t* v, uint32_t* tmp, uint32_t len) {
    if (len < 2) return;
    uint32_t mid = len / 2;
    merge_sort(c, v, tmp, mid);
    merge_sort(c, v + mid, tmp, len - mid);
    if (sort_cmp(c, v[mid - 1], v[mid]) <= 0) return;
    uint32_t i = 0, j = mid, o = 0;
    while (i < mid && j < len) tmp[o++] = (sort_cmp(c, v[j], v[i]) < 0) ? v[j++] : v[i++];
    while (i < mid) tmp[o++] = v[i++];
    while (j < len) tmp[o++] = v[j++];
    memcpy(v, tmp, sizeof(uint32_t) * len);
}

uint32_t or_sort_pr(const or_dfa* d, uint32_t* out_block, uint32_t* iters) {
    const uint32_t n = d->n, k = d->k;
    *iters = 0;
    if (n == 0) return 0;
    uint32_t* block = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* state = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* newb = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* sig = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n * k + 1));
    int any_acc = 0, any_rej = 0;
    for (uint32_t q = 0; q < n; ++q) {
        block[q] = d->acc[q] ? 0 : 1;
        if (d->acc[q]) any_acc = 1;
        else any_rej = 1;
        state[q] = q;
    }
    uint32_t num_blocks = (any_acc && any_rej) ? 2 : 1;
    sort_ctx c = {block, sig, k};
    for (;;) {
        for (uint32_t q = 0; q < n; ++q)
            for (uint32_t a = 0; a < k; ++a) sig[(size_t)q * k + a] = block[d->delta[(size_t)a * n + q]];
        merge_sort(&c, state, tmp, n);
        /* ARE_NEQ adjacent difference + inclusive scan (l.394-408) */
        newb[0] = 0;
        for (uint32_t i = 1; i < n; ++i) newb[i] = newb[i - 1] + (sort_cmp(&c, state[i], state[i - 1]) != 0);
        uint32_t new_count = newb[n - 1] + 1;
        if (new_count == num_blocks) break;
        for (uint32_t i = 0; i < n; ++i) block[state[i]] = newb[i];
        num_blocks = new_count;
        ++*iters;
    }
    uint32_t nb = or_normalize(block, n, out_block);
    free(block);
    free(state);
    free(tmp);
    free(newb);
    free(sig);
    return nb;
}

/* ------------------------------------------------------------------------ */
/* naivePR (src/minimize.cpp:214-348)                                        */
/* ------------------------------------------------------------------------ */

/* LeaderRefiner::init_blocks (l.227-238): min-index leaders of F and Q\F. */
static int leaders_init(const or_dfa* d, uint32_t* block) {
    uint32_t qf = OR_NONE, qn = OR_NONE;
    for (uint32_t q = 0; q < d->n && (qf == OR_NONE || qn == OR_NONE); ++q) {
        uint32_t* slot = d->acc[q] ? &qf : &qn;
        if (*slot == OR_NONE) *slot = q;
    }
    if (qf == OR_NONE || qn == OR_NONE) return 0;
    for (uint32_t q = 0; q < d->n; ++q) block[q] = d->acc[q] ? qf : qn;
    return 1;
}

/* collect_split_set (l.242-256): states disagreeing with their leader. */
static uint32_t collect_split(const or_dfa* d, const uint32_t* block, uint32_t* sq, uint32_t* sl) {
    uint32_t cnt = 0;
    const uint32_t n = d->n;
    for (uint32_t q = 0; q < n; ++q) {
        uint32_t leader = block[q];
        if (leader == q) continue;
        for (uint32_t a = 0; a < d->k; ++a) {
            const uint32_t* row = d->delta + (size_t)a * n;
            if (block[row[q]] != block[row[leader]]) {
                sq[cnt] = q;
                sl[cnt] = leader;
                ++cnt;
                break;
            }
        }
    }
    return cnt;
}

uint32_t or_naive_pr(const or_dfa* d, int policy, uint64_t seed, uint32_t* out_block, uint32_t* iters) {
    const uint32_t n = d->n;
    *iters = 0;
    uint32_t* block = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
    if (!leaders_init(d, block)) {
        for (uint32_t q = 0; q < n; ++q) out_block[q] = 0;
        free(block);
        return n > 0 ? 1 : 0;
    }
    uint32_t* new_leader = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* writers = (uint32_t*)calloc(n, sizeof(uint32_t));
    uint32_t* sq = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* sl = (uint32_t*)malloc(sizeof(uint32_t) * n);
    for (uint32_t q = 0; q < n; ++q) new_leader[q] = OR_NONE;
    or_mt64 rng;
    or_mt64_seed(&rng, seed);
    for (;;) {
        uint32_t cnt = collect_split(d, block, sq, sl);
        if (cnt == 0) break;
        ++*iters;
        /* election (l.285-305) */
        for (uint32_t i = 0; i < cnt; ++i) {
            uint32_t q = sq[i], L = sl[i];
            if (new_leader[L] == OR_NONE) {
                new_leader[L] = q;
                writers[L] = 1;
            } else if (policy == 1) {
                ++writers[L];
                if (or_uniform_u32(&rng, 0, writers[L] - 1) == 0) new_leader[L] = q;
            }
        }
        /* split pass (l.308) + slot reset (l.309) */
        for (uint32_t i = 0; i < cnt; ++i) block[sq[i]] = new_leader[sl[i]];
        for (uint32_t i = 0; i < cnt; ++i) new_leader[sl[i]] = OR_NONE;
    }
    uint32_t nb = or_normalize(block, n, out_block);
    free(block);
    free(new_leader);
    free(writers);
    free(sq);
    free(sl);
    return nb;
}

/* l.316-348: the first differing state (scan order) claims the slot. */
uint32_t or_naive_pr_fused(const or_dfa* d, uint32_t* out_block, uint32_t* iters) {
    const uint32_t n = d->n;
    *iters = 0;
    uint32_t* block = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
    if (!leaders_init(d, block)) {
        for (uint32_t q = 0; q < n; ++q) out_block[q] = 0;
        free(block);
        return n > 0 ? 1 : 0;
    }
    uint32_t* new_leader = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* sq = (uint32_t*)malloc(sizeof(uint32_t) * n);
    uint32_t* sl = (uint32_t*)malloc(sizeof(uint32_t) * n);
    for (uint32_t q = 0; q < n; ++q) new_leader[q] = OR_NONE;
    for (;;) {
        uint32_t cnt = collect_split(d, block, sq, sl);
        if (cnt == 0) break;
        ++*iters;
        for (uint32_t i = 0; i < cnt; ++i) {
            uint32_t q = sq[i], L = sl[i];
            if (new_leader[L] == OR_NONE) {
                new_leader[L] = q;
                block[q] = q;
            } else {
                block[q] = new_leader[L];
            }
        }
        for (uint32_t i = 0; i < cnt; ++i) new_leader[sl[i]] = OR_NONE;
    }
    uint32_t nb = or_normalize(block, n, out_block);
    free(block);
    free(new_leader);
    free(sq);
    free(sl);
    return nb;
}

/* ------------------------------------------------------------------------ */
/* transPR (src/minimize.cpp:425-478)                                        */
/* ------------------------------------------------------------------------ */

uint32_t or_floor_log2(uint32_t n) {
    uint32_t r = 0;
    if (n <= 1) return 0;
    while (n >>= 1) ++r;
    return r;
}

/* l.433-470: letter order a^1, a^2, a^4, ... per base letter. */
uint32_t or_build_transitive_alphabet(const or_dfa* d, uint32_t* out) {
    const uint32_t n = d->n, k = d->k, levels = or_floor_log2(n) + 1;
    for (uint32_t a = 0; a < k; ++a) {
        uint32_t* base = out + (size_t)a * levels * n;
        memcpy(base, d->delta + (size_t)a * n, sizeof(uint32_t) * n);
        for (uint32_t i = 1; i < levels; ++i) {
            const uint32_t* prev = base + (size_t)(i - 1) * n;
            uint32_t* cur = base + (size_t)i * n;
            for (uint32_t q = 0; q < n; ++q) cur[q] = prev[prev[q]];
        }
    }
    return k * levels;
}

uint32_t or_trans_pr(const or_dfa* d, int policy, uint64_t seed, uint32_t* out_block, uint32_t* iters,
                     uint32_t* closure_iters) {
    const uint32_t n = d->n, levels = or_floor_log2(n) + 1;
    uint32_t* closed = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)d->k * levels * n + 1));
    or_dfa c = *d;
    c.k = or_build_transitive_alphabet(d, closed);
    c.delta = closed;
    uint32_t nb = or_naive_pr(&c, policy, seed, out_block, iters);
    *closure_iters = or_floor_log2(n);
    free(closed);
    return nb;
}

/* ------------------------------------------------------------------------ */
/* trans: pair-graph closure (src/minimize.cpp:92-206, src/dfa.cpp:424-454)   */
/* ------------------------------------------------------------------------ */

static uint32_t partition_from_apart(const uint8_t* ap, uint32_t n, uint32_t* out) {
    uint32_t* labels = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
    uint32_t* reps = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
    uint32_t nr = 0;
    for (uint32_t q = 0; q < n; ++q) {
        uint32_t found = OR_NONE;
        for (uint32_t i = 0; i < nr; ++i)
            if (!ap[(size_t)reps[i] * n + q]) {
                found = reps[i];
                break;
            }
        if (found == OR_NONE) {
            reps[nr++] = q;
            found = q;
        }
        labels[q] = found;
    }
    uint32_t nb = or_normalize(labels, n, out);
    free(labels);
    free(reps);
    return nb;
}

uint32_t or_trans_minimize(const or_dfa* d, uint64_t max_pair_nodes, uint32_t* out_block, uint32_t* refine_iters,
                           uint32_t* closure_iters, uint8_t* apart_out) {
    const uint32_t n = d->n, k = d->k;
    const uint64_t V = (uint64_t)n * n;
    *refine_iters = 0;
    *closure_iters = 0;
    if (V > max_pair_nodes) return OR_NONE;
    const uint64_t W = (V + 63) / 64;
    uint64_t* reach = (uint64_t*)calloc(V * W + 1, 8);
    uint64_t* next = (uint64_t*)calloc(V * W + 1, 8);
    uint64_t* apart = (uint64_t*)calloc(W + 1, 8);
    uint64_t* changed = (uint64_t*)malloc(8 * (W + 1));
    uint64_t* changed_next = (uint64_t*)calloc(W + 1, 8);
    uint64_t* new_apart = (uint64_t*)calloc(W + 1, 8);
    for (uint32_t q = 0; q < n; ++q)
        for (uint32_t r = 0; r < n; ++r) {
            uint64_t s = (uint64_t)q * n + r;
            if (d->acc[q] != d->acc[r]) apart[s >> 6] |= 1ull << (s & 63);
            for (uint32_t a = 0; a < k; ++a) {
                uint64_t t = (uint64_t)d->delta[(size_t)a * n + q] * n + d->delta[(size_t)a * n + r];
                reach[s * W + (t >> 6)] |= 1ull << (t & 63);
            }
        }
    for (uint64_t w = 0; w < W; ++w) changed[w] = ~0ull;
    if (n > 0) {
        for (;;) {
            ++*closure_iters;
            /* Reach := Reach | Reach.Reach from the pass-start matrix (l.141-175) */
            memset(changed_next, 0, 8 * W);
            for (uint64_t s = 0; s < V; ++s) {
                const uint64_t* rs = reach + s * W;
                uint64_t* ns = next + s * W;
                memcpy(ns, rs, 8 * W);
                int touch = 0;
                for (uint64_t w = 0; w < W && !touch; ++w) touch = (rs[w] & changed[w]) != 0;
                if (!touch) continue;
                for (uint64_t w = 0; w < W; ++w) {
                    uint64_t bits = rs[w];
                    while (bits) {
                        uint64_t t = (w << 6) + (uint64_t)__builtin_ctzll(bits);
                        bits &= bits - 1;
                        const uint64_t* rt = reach + t * W;
                        for (uint64_t v = 0; v < W; ++v) ns[v] |= rt[v];
                    }
                }
                for (uint64_t w = 0; w < W; ++w)
                    if (ns[w] != rs[w]) {
                        changed_next[s >> 6] |= 1ull << (s & 63);
                        break;
                    }
            }
            uint64_t* t = reach;
            reach = next;
            next = t;
            t = changed;
            changed = changed_next;
            changed_next = t;
            /* one apartness propagation step (l.177-194) */
            memset(new_apart, 0, 8 * W);
            int any = 0;
            for (uint64_t s = 0; s < V; ++s) {
                if ((apart[s >> 6] >> (s & 63)) & 1) continue;
                const uint64_t* rs = reach + s * W;
                for (uint64_t w = 0; w < W; ++w)
                    if (rs[w] & apart[w]) {
                        new_apart[s >> 6] |= 1ull << (s & 63);
                        any = 1;
                        break;
                    }
            }
            if (!any) break;
            ++*refine_iters;
            for (uint64_t w = 0; w < W; ++w) apart[w] |= new_apart[w];
        }
    }
    /* symmetric matrix over q < r (l.198-203) */
    uint8_t* ap = (uint8_t*)calloc(V + 1, 1);
    for (uint32_t q = 0; q < n; ++q)
        for (uint32_t r = q + 1; r < n; ++r) {
            uint64_t s = (uint64_t)q * n + r;
            if ((apart[s >> 6] >> (s & 63)) & 1) {
                ap[s] = 1;
                ap[(uint64_t)r * n + q] = 1;
            }
        }
    uint32_t nb = partition_from_apart(ap, n, out_block);
    if (apart_out) memcpy(apart_out, ap, V);
    free(ap);
    free(reach);
    free(next);
    free(apart);
    free(changed);
    free(changed_next);
    free(new_apart);
    return nb;
}

/* ------------------------------------------------------------------------ */
/* Product exploration (src/equivalence.cpp:25-207)                         */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint64_t key;
    uint32_t parent;
    uint32_t letter;
} pair_rec;

typedef struct {
    uint32_t* table;
    uint64_t mask;
    pair_rec* recs;
    uint64_t size, cap_recs, max_visited;
} pair_set;

static void ps_grow(pair_set* s) {
    uint64_t nsz = (s->mask + 1) * 2;
    uint32_t* t = (uint32_t*)malloc(sizeof(uint32_t) * nsz);
    memset(t, 0xff, sizeof(uint32_t) * nsz);
    for (uint64_t i = 0; i < s->size; ++i) {
        uint64_t slot = or_mix64(s->recs[i].key) & (nsz - 1);
        while (t[slot] != OR_NONE) slot = (slot + 1) & (nsz - 1);
        t[slot] = (uint32_t)i;
    }
    free(s->table);
    s->table = t;
    s->mask = nsz - 1;
}

/* PairSet::insert (l.40-55); returns -1 on budget, else fresh flag; *idx set */
static int ps_insert(pair_set* s, uint64_t key, uint32_t parent, uint32_t letter, uint32_t* idx) {
    uint64_t slot = or_mix64(key) & s->mask;
    while (s->table[slot] != OR_NONE) {
        if (s->recs[s->table[slot]].key == key) {
            *idx = s->table[slot];
            return 0;
        }
        slot = (slot + 1) & s->mask;
    }
    if (s->size >= s->max_visited) return -1;
    if (s->size == s->cap_recs) {
        s->cap_recs *= 2;
        s->recs = (pair_rec*)realloc(s->recs, sizeof(pair_rec) * s->cap_recs);
    }
    *idx = (uint32_t)s->size;
    s->recs[s->size].key = key;
    s->recs[s->size].parent = parent;
    s->recs[s->size].letter = letter;
    s->size++;
    s->table[slot] = *idx;
    if (s->size * 2 > s->mask + 1) ps_grow(s);
    return 1;
}

static uint32_t ps_word(const pair_set* s, uint32_t idx, uint32_t* cex, uint32_t cap) {
    uint32_t len = 0;
    for (uint32_t i = idx; i != 0; i = s->recs[i].parent) ++len;
    uint32_t pos = len;
    for (uint32_t i = idx; i != 0; i = s->recs[i].parent) {
        --pos;
        if (pos < cap) cex[pos] = s->recs[i].letter;
    }
    return len;
}

int or_explore_product(const or_dfa* a, const or_dfa* b, int mode, const uint32_t* to_b, uint64_t max_visited,
                       uint32_t* cex, uint32_t cex_cap, or_product* out) {
    if (a->initial < 0 || b->initial < 0) return -1;
    if (!to_b && a->k != b->k) return -2;
    const uint32_t k = a->k;
    memset(out, 0, sizeof(*out));
    pair_set s;
    s.mask = 1023;
    s.table = (uint32_t*)malloc(sizeof(uint32_t) * 1024);
    memset(s.table, 0xff, sizeof(uint32_t) * 1024);
    s.cap_recs = 1024;
    s.recs = (pair_rec*)malloc(sizeof(pair_rec) * s.cap_recs);
    s.size = 0;
    s.max_visited = max_visited < 0xfffffffeull ? max_visited : 0xfffffffeull;
    int rc = 0;
#define FAILS(qa, qb) \
    ((mode == OR_MODE_INCL) ? (a->acc[qa] && !b->acc[qb]) : (a->acc[qa] != b->acc[qb]))
    uint32_t idx, first_fail = OR_NONE;
    uint32_t ia = (uint32_t)a->initial, ib = (uint32_t)b->initial;
    if (ps_insert(&s, ((uint64_t)ia << 32) | ib, 0, 0, &idx) < 0) {
        rc = -3;
        goto done;
    }
    if (FAILS(ia, ib)) {
        if (mode != OR_MODE_FULL) {
            out->verdict = OR_VERDICT_COUNTEREXAMPLE;
            out->explored = 1;
            out->cex_len = 0;
            goto done;
        }
        first_fail = 0;
    }
    {
        uint64_t wb = 0, we = 1;
        while (wb < we) {
            for (uint64_t i = wb; i < we; ++i) {
                uint64_t key = s.recs[i].key;
                uint32_t qa = (uint32_t)(key >> 32), qb = (uint32_t)key;
                for (uint32_t la = 0; la < k; ++la) {
                    uint32_t pa = a->delta[(size_t)la * a->n + qa];
                    uint32_t lb = to_b ? to_b[la] : la;
                    uint32_t pb = b->delta[(size_t)lb * b->n + qb];
                    int fr = ps_insert(&s, ((uint64_t)pa << 32) | pb, (uint32_t)i, la, &idx);
                    if (fr < 0) {
                        rc = -3;
                        goto done;
                    }
                    if (!fr) continue;
                    if (FAILS(pa, pb)) {
                        if (mode != OR_MODE_FULL) {
                            out->verdict = OR_VERDICT_COUNTEREXAMPLE;
                            out->cex_len = ps_word(&s, idx, cex, cex_cap);
                            out->explored = s.size;
                            goto done;
                        }
                        if (first_fail == OR_NONE) first_fail = idx;
                    }
                }
            }
            ++out->levels;
            wb = we;
            we = s.size;
        }
    }
    if (mode == OR_MODE_FULL && first_fail != OR_NONE) {
        out->verdict = OR_VERDICT_COUNTEREXAMPLE;
        out->cex_len = ps_word(&s, first_fail, cex, cex_cap);
    } else {
        out->verdict = mode == OR_MODE_INCL ? OR_VERDICT_INCLUDED : OR_VERDICT_EQUIVALENT;
    }
    out->explored = s.size;
#undef FAILS
done:
    free(s.table);
    free(s.recs);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* helpers                                                                   */
/* ------------------------------------------------------------------------ */

int or_accepts(const or_dfa* d, const uint32_t* word, uint32_t len) {
    uint32_t q = (uint32_t)d->initial;
    for (uint32_t i = 0; i < len; ++i) q = d->delta[(size_t)word[i] * d->n + q];
    return d->acc[q];
}

/* src/dfa.cpp:133-151: BFS numbering, letters upwards. */
uint32_t or_bfs_order(const or_dfa* d, uint32_t* order) {
    for (uint32_t q = 0; q < d->n; ++q) order[q] = OR_NONE;
    if (d->initial < 0) return 0;
    uint32_t* queue = (uint32_t*)malloc(sizeof(uint32_t) * (d->n + 1));
    uint32_t head = 0, tail = 0, next = 0;
    queue[tail++] = (uint32_t)d->initial;
    order[d->initial] = next++;
    while (head < tail) {
        uint32_t q = queue[head++];
        for (uint32_t a = 0; a < d->k; ++a) {
            uint32_t t = d->delta[(size_t)a * d->n + q];
            if (order[t] == OR_NONE) {
                order[t] = next++;
                queue[tail++] = t;
            }
        }
    }
    free(queue);
    return next;
}
