/*
 * oracle.h -- CPU restatement of the dfakit reference algorithms.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2508_20735_b200/)
 * links, loads or calls this code.  Only tests/, __graft_entry__.smoke() and
 * the cpu_baseline leg of bench.py may use it, and only as the checker.
 *
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/...).  The restatement is pinned against outputs of
 * the reference itself (oracle/_ref, built from the reference sources by
 * oracle/Makefile) through the golden fixtures in tests/golden/.
 *
 * Conventions: a DFA is letter-major, delta[a*n + q] = delta(q, a) (the
 * reference's delta[a][q], include/dfakit/dfa.hpp:22), acc[q] in {0,1},
 * initial = -1 when absent.
 */
#ifndef DFAKIT_ORACLE_H
#define DFAKIT_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_NONE 0xffffffffu

typedef struct {
    uint32_t n;
    uint32_t k;
    const uint32_t* delta; /* k*n, letter-major */
    const uint8_t* acc;    /* n */
    int64_t initial;       /* -1: absent */
} or_dfa;

/* ---- libstdc++-identical randomness (reference uses std::mt19937_64) ---- */
typedef struct {
    uint64_t mt[312];
    uint32_t idx;
} or_mt64;

void or_mt64_seed(or_mt64* g, uint64_t seed);
uint64_t or_mt64_next(or_mt64* g);
/* std::uniform_int_distribution<uint32_t>(lo, hi) with a 64-bit engine
 * (libstdc++ 13 bits/uniform_int_dist.h: Lemire downscaling via __int128). */
uint32_t or_uniform_u32(or_mt64* g, uint32_t lo, uint32_t hi);
/* std::bernoulli_distribution(p) via generate_canonical<double,53>. */
int or_bernoulli(or_mt64* g, double p);

/* ---- partitions ---- */
/* Partition::from_labels (src/dfa.cpp:47-58): dense ids by first occurrence. */
uint32_t or_normalize(const uint32_t* labels, uint32_t n, uint32_t* out);

/* ---- generators (src/generators.cpp) ---- */
/* return 0 on success, -1 on invalid parameter / budget */
int or_gen_random(uint32_t n, uint32_t k, double frac, uint64_t seed, uint32_t* delta, uint8_t* acc);
uint64_t or_fib_word_len(uint32_t m);
int or_gen_fib(uint32_t m, uint32_t* delta, uint8_t* acc);             /* n = or_fib_word_len(m), k = 1 */
int or_gen_bitsplitter(uint32_t nbits, uint32_t* delta, uint8_t* acc); /* n = 2^nbits, k = nbits-1 */
int or_gen_bitsplitter_ext(uint32_t nbits, uint32_t* delta, uint8_t* acc); /* n = 2^(nbits+1), k = 2nbits */
uint64_t or_cycle_fib(uint32_t m);
uint32_t or_cycle_letters(uint32_t m);
int or_gen_cycle(uint32_t m, uint32_t* delta, uint8_t* acc);
int or_gen_memory(uint32_t depth, int forgetful, uint32_t* delta, uint8_t* acc); /* n = 2^depth, k = 2 */
/* Unary chain q -> q+1, last state self-loop and accepting (tests/test_minimize.cpp:251-262). */
int or_gen_chain(uint32_t n, uint32_t* delta, uint8_t* acc);
/* Synthetic bench DFA: counter-hash successors, see DESIGN.md "synthetic inputs". */
void or_gen_synth(uint32_t n, uint32_t k, uint64_t seed, uint32_t* delta, uint8_t* acc);

/* ---- minimisers (src/minimize.cpp) ---- */
/* All return the number of blocks; out_block receives the normalized partition. */
uint32_t or_moore(const or_dfa* d, uint32_t* out_block, uint32_t* iters);
uint32_t or_sort_pr(const or_dfa* d, uint32_t* out_block, uint32_t* iters);
/* policy 0 = min_index, 1 = arbitrary(seed) */
uint32_t or_naive_pr(const or_dfa* d, int policy, uint64_t seed, uint32_t* out_block, uint32_t* iters);
uint32_t or_naive_pr_fused(const or_dfa* d, uint32_t* out_block, uint32_t* iters);
uint32_t or_floor_log2(uint32_t n);
/* out_delta: k*(floor_log2(n)+1)*n entries; returns the new alphabet size. */
uint32_t or_build_transitive_alphabet(const or_dfa* d, uint32_t* out_delta);
uint32_t or_trans_pr(const or_dfa* d, int policy, uint64_t seed, uint32_t* out_block, uint32_t* iters,
                     uint32_t* closure_iters);
/* Pair-graph closure (trans).  apart_out may be NULL, else n*n bytes.
 * Returns blocks, or OR_NONE when n*n > max_pair_nodes. */
uint32_t or_trans_minimize(const or_dfa* d, uint64_t max_pair_nodes, uint32_t* out_block, uint32_t* refine_iters,
                           uint32_t* closure_iters, uint8_t* apart_out);

/* ---- product exploration (src/equivalence.cpp) ---- */
enum { OR_MODE_EQUIV = 0, OR_MODE_INCL = 1, OR_MODE_FULL = 2 };
enum { OR_VERDICT_EQUIVALENT = 0, OR_VERDICT_INCLUDED = 1, OR_VERDICT_COUNTEREXAMPLE = 2 };
typedef struct {
    int32_t verdict;
    uint32_t levels;
    uint64_t explored;
    uint32_t cex_len; /* full length, even when > cex_cap */
} or_product;
/* to_b: letter map A->B (NULL = identity).  Returns 0 ok, -1 missing initial,
 * -2 alphabet mismatch, -3 visited budget exceeded. */
int or_explore_product(const or_dfa* a, const or_dfa* b, int mode, const uint32_t* to_b, uint64_t max_visited,
                       uint32_t* cex, uint32_t cex_cap, or_product* out);

/* ---- helpers ---- */
/* run word from initial; returns acceptance */
int or_accepts(const or_dfa* d, const uint32_t* word, uint32_t len);
/* BFS prune (src/dfa.cpp:135-181 restated); returns reachable count, order[q] or OR_NONE */
uint32_t or_bfs_order(const or_dfa* d, uint32_t* order);

#ifdef __cplusplus
}
#endif
#endif
