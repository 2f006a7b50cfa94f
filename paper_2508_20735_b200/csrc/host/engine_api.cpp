// engine_api.cpp -- the GPU-backed part of the drop-in API: minimisers and
// product exploration forward to the C ABI (dfakit_b200.h).  Every calling
// thread has its own context (stream + memory pool) on device DFAKIT_DEVICE
// or, without it, on the visible devices round-robin: concurrent callers run
// in parallel instead of queueing on one process-wide context.  Errors map
// back to the reference's exception types.
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <unordered_map>

#include "dfakit_b200.h"
#include "dfakit_b200.hpp"

namespace dfakit {

namespace {

void raise(dfakit_status s) {
    if (s == DFAKIT_OK) return;
    const std::string msg = dfakit_last_error();
    if (s == DFAKIT_E_RESOURCE) throw ResourceError(msg);
    if (s == DFAKIT_E_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error("libdfakit_b200: " + msg);
}

int pick_device() {
    if (const char* env = std::getenv("DFAKIT_DEVICE")) return std::atoi(env);
    static std::atomic<unsigned> next{0};
    const int nd = dfakit_device_count();
    return nd > 0 ? (int)(next.fetch_add(1) % (unsigned)nd) : 0;
}

struct ThreadCtx {
    dfakit_ctx* c = nullptr;
    int device = -1;
    ~ThreadCtx() {
        if (c) dfakit_ctx_destroy(c);
    }
};

ThreadCtx& thread_ctx() {
    thread_local ThreadCtx t;
    if (!t.c) {
        const int dev = pick_device();
        raise(dfakit_ctx_create(dev, &t.c));
        t.device = dev;
    }
    return t;
}

dfakit_ctx* context() { return thread_ctx().c; }

// contiguous letter-major copy of a Dfa
struct Flat {
    std::vector<uint32_t> delta;
    std::vector<uint8_t> acc;
    dfakit_dfa view{};
    explicit Flat(const Dfa& d) {
        if (d.delta.size() != d.alphabet_size || d.accepting.size() != d.num_states)
            throw std::invalid_argument("malformed Dfa: " + (validate(d).empty() ? std::string("size mismatch")
                                                                                  : validate(d).front()));
        delta.resize((size_t)d.num_states * d.alphabet_size);
        for (LetterId a = 0; a < d.alphabet_size; ++a) {
            if (d.delta[a].size() != d.num_states) throw std::invalid_argument("malformed Dfa: delta row size");
            std::memcpy(delta.data() + (size_t)a * d.num_states, d.delta[a].data(), sizeof(uint32_t) * d.num_states);
        }
        acc.resize(d.num_states);
        for (StateId q = 0; q < d.num_states; ++q) acc[q] = d.accepting[q] ? 1 : 0;
        view.num_states = d.num_states;
        view.alphabet_size = d.alphabet_size;
        view.delta = delta.data();
        view.accepting = acc.data();
        view.initial = d.initial ? (int64_t)*d.initial : -1;
    }
};

RefinementReport run(const Dfa& d, Algorithm algo, const dfakit_options* o) {
    Flat f(d);
    RefinementReport r;
    r.algorithm = algo;
    r.partition.block_of.resize(d.num_states);
    dfakit_report rep{};
    raise(dfakit_minimize(context(), &f.view, (dfakit_algorithm)algo, o, r.partition.block_of.data(), &rep));
    r.partition.num_blocks = rep.num_blocks;
    r.refining_iterations = rep.refining_iterations;
    r.closure_iterations = rep.closure_iterations;
    return r;
}

dfakit_options policy_opts(const ElectionPolicy& p) {
    dfakit_options o{};
    o.policy = p.kind == ElectionPolicy::Kind::arbitrary ? DFAKIT_POLICY_ARBITRARY : DFAKIT_POLICY_MIN_INDEX;
    o.seed = p.seed;
    return o;
}

}  // namespace

const char* to_string(Algorithm a) {
    switch (a) {
        case Algorithm::moore: return "moore";
        case Algorithm::trans: return "trans";
        case Algorithm::naive_pr: return "naive";
        case Algorithm::naive_pr_fused: return "naive-fused";
        case Algorithm::sort_pr: return "sort";
        case Algorithm::trans_pr: return "transpr";
    }
    return "?";
}

RefinementReport moore_minimize(const Dfa& dfa) { return run(dfa, Algorithm::moore, nullptr); }

RefinementReport sort_pr(const Dfa& dfa) { return run(dfa, Algorithm::sort_pr, nullptr); }

RefinementReport naive_pr(const Dfa& dfa, const ElectionPolicy& policy) {
    dfakit_options o = policy_opts(policy);
    return run(dfa, Algorithm::naive_pr, &o);
}

RefinementReport naive_pr_fused(const Dfa& dfa) { return run(dfa, Algorithm::naive_pr_fused, nullptr); }

RefinementReport trans_pr(const Dfa& dfa, const ElectionPolicy& policy, std::uint64_t max_transitions) {
    dfakit_options o = policy_opts(policy);
    o.max_transitions = max_transitions;
    return run(dfa, Algorithm::trans_pr, &o);
}

TransResult trans_minimize(const Dfa& dfa, std::uint64_t max_pair_nodes) {
    Flat f(dfa);
    const StateId n = dfa.num_states;
    if ((std::uint64_t)n * n > max_pair_nodes) {
        // let the library produce the reference's message
        dfakit_report rep{};
        raise(dfakit_trans_minimize(context(), &f.view, max_pair_nodes, nullptr, nullptr, &rep));
    }
    std::vector<uint8_t> bytes((size_t)n * n);
    RefinementReport r;
    r.algorithm = Algorithm::trans;
    r.partition.block_of.resize(n);
    dfakit_report rep{};
    raise(dfakit_trans_minimize(context(), &f.view, max_pair_nodes, r.partition.block_of.data(), bytes.data(), &rep));
    r.partition.num_blocks = rep.num_blocks;
    r.refining_iterations = rep.refining_iterations;
    r.closure_iterations = rep.closure_iterations;
    ApartMatrix m(n);
    for (StateId q = 0; q < n; ++q)
        for (StateId s = q + 1; s < n; ++s)
            if (bytes[(size_t)q * n + s]) m.set_apart(q, s);
    return TransResult{std::move(r), std::move(m)};
}

Dfa build_transitive_alphabet(const Dfa& dfa, std::uint64_t max_transitions) {
    Flat f(dfa);
    uint32_t k2 = 0;
    raise(dfakit_build_transitive_alphabet(context(), &f.view, max_transitions, nullptr, &k2));
    std::vector<uint32_t> out((size_t)k2 * dfa.num_states);
    raise(dfakit_build_transitive_alphabet(context(), &f.view, max_transitions, out.data(), &k2));
    Dfa c;
    c.num_states = dfa.num_states;
    c.alphabet_size = k2;
    c.accepting = dfa.accepting;
    c.initial = dfa.initial;
    c.delta.resize(k2);
    for (LetterId a = 0; a < k2; ++a)
        c.delta[a].assign(out.begin() + (size_t)a * dfa.num_states, out.begin() + (size_t)(a + 1) * dfa.num_states);
    const LetterId k = dfa.alphabet_size, levels = k ? k2 / k : 1;
    c.letter_names.emplace();
    for (LetterId a = 0; a < k; ++a) {
        const std::string base = dfa.letter_names ? (*dfa.letter_names)[a] : (k == 1 ? "a" : "a" + std::to_string(a));
        for (LetterId i = 0; i < levels; ++i) c.letter_names->push_back(base + "^" + std::to_string(1ull << i));
    }
    return c;
}

namespace {

std::vector<uint32_t> letter_map(const Dfa& a, const Dfa& b, const ExploreOptions& opts) {
    if (!opts.match_letters_by_name) {
        if (a.alphabet_size != b.alphabet_size)
            throw std::invalid_argument("alphabet size mismatch: " + std::to_string(a.alphabet_size) + " vs " +
                                        std::to_string(b.alphabet_size));
        return {};
    }
    if (!a.letter_names || !b.letter_names)
        throw std::invalid_argument("matching letters by name requires letter names on both inputs");
    if (a.alphabet_size != b.alphabet_size) throw std::invalid_argument("letter name sets differ in size");
    std::unordered_map<std::string, uint32_t> in_b;
    for (uint32_t i = 0; i < b.alphabet_size; ++i)
        if (!in_b.emplace((*b.letter_names)[i], i).second)
            throw std::invalid_argument("duplicate letter name '" + (*b.letter_names)[i] + "'");
    std::vector<uint32_t> m(a.alphabet_size);
    std::vector<bool> taken(b.alphabet_size, false);
    for (uint32_t i = 0; i < a.alphabet_size; ++i) {
        auto it = in_b.find((*a.letter_names)[i]);
        if (it == in_b.end()) throw std::invalid_argument("letter '" + (*a.letter_names)[i] + "' has no counterpart");
        if (taken[it->second]) throw std::invalid_argument("duplicate letter name '" + (*a.letter_names)[i] + "'");
        taken[it->second] = true;
        m[i] = it->second;
    }
    return m;
}

ProductResult finish(const dfakit_product& p, std::vector<uint32_t>& word) {
    ProductResult r;
    r.verdict = static_cast<Verdict>(p.verdict);
    r.explored_states = p.explored_states;
    r.levels = p.levels;
    word.resize(p.counterexample_len);
    r.counterexample.assign(word.begin(), word.end());
    return r;
}

}  // namespace

ProductResult explore_product(const Dfa& a, const Dfa& b, ExploreMode mode, const ExploreOptions& opts) {
    if (!a.initial || !b.initial)
        throw std::invalid_argument("product exploration requires initial states on both inputs");
    std::vector<uint32_t> map = letter_map(a, b, opts);
    Flat fa(a), fb(b);
    dfakit_product p{};
    std::vector<uint32_t> word(1u << 16);
    raise(dfakit_explore_product(context(), &fa.view, &fb.view, (dfakit_mode)mode, map.empty() ? nullptr : map.data(),
                                 opts.max_visited, word.data(), (uint32_t)word.size(), &p));
    if (p.counterexample_len > word.size()) {  // rare: longer than the first buffer
        word.assign(p.counterexample_len, 0);
        raise(dfakit_explore_product(context(), &fa.view, &fb.view, (dfakit_mode)mode,
                                     map.empty() ? nullptr : map.data(), opts.max_visited, word.data(),
                                     (uint32_t)word.size(), &p));
    }
    return finish(p, word);
}

ProductResult check_equiv(const Dfa& a, const Dfa& b, const ExploreOptions& opts) {
    return explore_product(a, b, ExploreMode::equivalence, opts);
}

ProductResult check_inclusion(const Dfa& a, const Dfa& b, const ExploreOptions& opts) {
    return explore_product(a, b, ExploreMode::inclusion, opts);
}

ProductResult check_equiv_union_find(const Dfa& a, const Dfa& b) {
    if (!a.initial || !b.initial)
        throw std::invalid_argument("equivalence checking requires initial states on both inputs");
    Flat fa(a), fb(b);
    dfakit_product p{};
    std::vector<uint32_t> word(1u << 16);
    raise(dfakit_check_equiv_uf(context(), &fa.view, &fb.view, word.data(), (uint32_t)word.size(), &p));
    if (p.counterexample_len > word.size()) {
        word.assign(p.counterexample_len, 0);
        raise(dfakit_check_equiv_uf(context(), &fa.view, &fb.view, word.data(), (uint32_t)word.size(), &p));
    }
    return finish(p, word);
}

namespace b200 {

int current_device() { return thread_ctx().device; }

CommId sharded_unique_id() {
    CommId id{};
    raise(dfakit_comm_unique_id(id.data()));
    return id;
}

ShardedComm::ShardedComm(const CommId& id, int world, int rank, int device) : world_(world), rank_(rank) {
    dfakit_ctx* c = nullptr;
    raise(dfakit_ctx_create(device, &c));
    dfakit_comm* m = nullptr;
    const dfakit_status st = dfakit_comm_init(c, id.data(), world, rank, &m);
    if (st != DFAKIT_OK) {
        dfakit_ctx_destroy(c);
        raise(st);
    }
    ctx_ = c;
    comm_ = m;
}

ShardedComm::~ShardedComm() {
    if (comm_) dfakit_comm_destroy(static_cast<dfakit_comm*>(comm_));
    if (ctx_) dfakit_ctx_destroy(static_cast<dfakit_ctx*>(ctx_));
}

RefinementReport sort_pr_sharded(const Dfa& dfa, ShardedComm& comm) {
    Flat f(dfa);
    RefinementReport r;
    r.algorithm = Algorithm::sort_pr;
    r.partition.block_of.resize(dfa.num_states);
    dfakit_report rep{};
    raise(dfakit_sort_pr_sharded_host(static_cast<dfakit_ctx*>(comm.ctx()), static_cast<dfakit_comm*>(comm.comm()),
                                      &f.view, r.partition.block_of.data(), &rep));
    r.partition.num_blocks = rep.num_blocks;
    r.refining_iterations = rep.refining_iterations;
    r.closure_iterations = rep.closure_iterations;
    return r;
}

}  // namespace b200

}  // namespace dfakit
