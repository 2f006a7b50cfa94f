// ref_shim.cpp -- extern "C" wrapper over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libdfakit_ref.so).
//
// TEST INFRASTRUCTURE ONLY: used to pin the C restatement (oracle.c) and to
// generate tests/golden fixtures, and as the CPU baseline arm of bench.py.
// Arrays are letter-major like the reference's delta[a][q].
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "dfakit/dfa.hpp"
#include "dfakit/equivalence.hpp"
#include "dfakit/errors.hpp"
#include "dfakit/generators.hpp"
#include "dfakit/minimize.hpp"

using namespace dfakit;

namespace {

Dfa make_dfa(uint32_t n, uint32_t k, const uint32_t* delta, const uint8_t* acc, int64_t initial) {
    Dfa d;
    d.num_states = n;
    d.alphabet_size = k;
    d.delta.resize(k);
    for (uint32_t a = 0; a < k; ++a) d.delta[a].assign(delta + (size_t)a * n, delta + (size_t)(a + 1) * n);
    d.accepting.resize(n);
    for (uint32_t q = 0; q < n; ++q) d.accepting[q] = acc[q] != 0;
    if (initial >= 0) d.initial = static_cast<StateId>(initial);
    return d;
}

void export_dfa(const Dfa& d, uint32_t* delta, uint8_t* acc) {
    if (delta)
        for (uint32_t a = 0; a < d.alphabet_size; ++a)
            std::memcpy(delta + (size_t)a * d.num_states, d.delta[a].data(), sizeof(uint32_t) * d.num_states);
    if (acc)
        for (uint32_t q = 0; q < d.num_states; ++q) acc[q] = d.accepting[q] ? 1 : 0;
}

}  // namespace

extern "C" {

// family: 0 random(n=param, k=param2, frac, seed), 1 fib(m), 2 bitsplit, 3 bitsplit-ext,
// 4 cycle, 5 memory-perfect, 6 memory-forgetful.  Call with delta == NULL to
// query sizes.  Returns 0, or -1 on any exception.
int ref_generate(int family, uint32_t param, uint32_t param2, double frac, uint64_t seed, uint32_t* delta,
                 uint8_t* acc, uint32_t* n, uint32_t* k, int64_t* initial) {
    try {
        Dfa d;
        switch (family) {
            case 0: d = gen_random_dfa(param, param2, frac, seed); break;
            case 1: d = gen_fib(param); break;
            case 2: d = gen_bitsplitter(param); break;
            case 3: d = gen_bitsplitter_ext(param); break;
            case 4: d = gen_cycle(param); break;
            case 5: d = gen_memory_perfect(param); break;
            case 6: d = gen_memory_forgetful(param); break;
            default: return -1;
        }
        *n = d.num_states;
        *k = d.alphabet_size;
        *initial = d.initial ? static_cast<int64_t>(*d.initial) : -1;
        export_dfa(d, delta, acc);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// algo: 0 moore, 1 trans, 2 naive, 3 naive-fused, 4 sort, 5 transpr.
// Returns the number of blocks, -1 on ResourceError, -2 on other errors.
int64_t ref_minimize(int algo, int policy, uint64_t seed, uint32_t n, uint32_t k, const uint32_t* delta,
                     const uint8_t* acc, uint32_t* out_block, uint32_t* refine_iters, uint32_t* closure_iters) {
    try {
        Dfa d = make_dfa(n, k, delta, acc, -1);
        ElectionPolicy pol = policy ? ElectionPolicy::arbitrary(seed) : ElectionPolicy::min_index();
        RefinementReport r;
        switch (algo) {
            case 0: r = moore_minimize(d); break;
            case 1: r = trans_minimize(d).report; break;
            case 2: r = naive_pr(d, pol); break;
            case 3: r = naive_pr_fused(d); break;
            case 4: r = sort_pr(d); break;
            case 5: r = trans_pr(d, pol); break;
            default: return -2;
        }
        if (out_block) std::memcpy(out_block, r.partition.block_of.data(), sizeof(uint32_t) * n);
        *refine_iters = r.refining_iterations;
        *closure_iters = r.closure_iterations;
        return r.partition.num_blocks;
    } catch (const ResourceError&) {
        return -1;
    } catch (const std::exception&) {
        return -2;
    }
}

int ref_transitive_alphabet(uint32_t n, uint32_t k, const uint32_t* delta, const uint8_t* acc, uint32_t* out,
                            uint32_t* out_k) {
    try {
        Dfa c = build_transitive_alphabet(make_dfa(n, k, delta, acc, -1));
        *out_k = c.alphabet_size;
        if (out) export_dfa(c, out, nullptr);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

// mode: 0 equivalence, 1 inclusion, 2 full.  verdict: 0 equivalent, 1 included, 2 counterexample.
// Returns 0, -1 invalid argument, -3 resource error.
int ref_explore(int mode, uint32_t na, uint32_t ka, const uint32_t* da, const uint8_t* aa, int64_t ia, uint32_t nb,
                uint32_t kb, const uint32_t* db, const uint8_t* ab, int64_t ib, uint64_t max_visited, int32_t* verdict,
                uint64_t* explored, uint32_t* levels, uint32_t* cex, uint32_t cex_cap, uint32_t* cex_len) {
    try {
        Dfa a = make_dfa(na, ka, da, aa, ia);
        Dfa b = make_dfa(nb, kb, db, ab, ib);
        ExploreOptions opts;
        opts.max_visited = max_visited;
        ExploreMode m = mode == 0 ? ExploreMode::equivalence : mode == 1 ? ExploreMode::inclusion : ExploreMode::full;
        ProductResult r = explore_product(a, b, m, opts);
        *verdict = static_cast<int32_t>(r.verdict);
        *explored = r.explored_states;
        *levels = r.levels;
        *cex_len = static_cast<uint32_t>(r.counterexample.size());
        for (uint32_t i = 0; i < *cex_len && i < cex_cap; ++i) cex[i] = r.counterexample[i];
        return 0;
    } catch (const ResourceError&) {
        return -3;
    } catch (const std::exception&) {
        return -1;
    }
}

}  // extern "C"
