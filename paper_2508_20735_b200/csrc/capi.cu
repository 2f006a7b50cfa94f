// capi.cu -- the extern "C" boundary (include/dfakit_b200.h).  Translates
// host buffers to device buffers, runs the device engines, maps exceptions
// to dfakit_status.  No CPU algorithm lives here: without a device every
// call fails with DFAKIT_E_NODEVICE.
#include <cstring>
#include <string>
#include <vector>

#include "dfakit_b200.h"
#include "prims.cuh"
#include "refine.cuh"

namespace dk {
Ctx* ctx_create(int device);
void ctx_destroy(Ctx* c);
std::string prof_collect(Ctx* ctx);
}  // namespace dk

struct dfakit_ctx {
    dk::Ctx* c;
};

struct dfakit_comm {
    dk::NcclComm* c;
};

struct dfakit_local_hub {
    dk::LocalHub* h;
};

namespace {

thread_local std::string g_last_error;

constexpr uint64_t kDefaultMaxTransitions = 1ull << 28;  // minimize.hpp:41
constexpr uint64_t kDefaultMaxPairNodes = 1ull << 16;    // minimize.hpp:38

template <typename F>
dfakit_status guard(F&& f) {
    try {
        f();
        return DFAKIT_OK;
    } catch (const dk::Error& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return DFAKIT_E_RESOURCE;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return DFAKIT_E_INVALID;
    }
}

void check_view(const dfakit_dfa* d, const char* who) {
    if (!d) throw dk::Error(DFAKIT_E_INVALID, std::string(who) + ": null DFA");
    if (d->num_states && !d->accepting) throw dk::Error(DFAKIT_E_INVALID, std::string(who) + ": null accepting");
    if ((uint64_t)d->num_states * d->alphabet_size && !d->delta)
        throw dk::Error(DFAKIT_E_INVALID, std::string(who) + ": null delta");
    if (d->initial >= (int64_t)d->num_states) throw dk::Error(DFAKIT_E_INVALID, std::string(who) + ": initial out of range");
}

// Host DFA copied into HBM (validated: every target < n, dfa.cpp:6-40).
struct Staged {
    dk::DBuf<uint32_t> delta;
    dk::DBuf<uint8_t> acc;
    dk::DevDfa view;
};

__global__ void range_check_kernel(const uint32_t* __restrict__ delta, uint64_t total, uint32_t n,
                                   uint32_t* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x)
        if (delta[i] >= n) atomicOr(bad, 1u);
}

void validate_device(dk::Ctx* c, const dk::DevDfa& v, cudaStream_t s) {
    const uint64_t total = (uint64_t)v.n * v.k;
    if (!total) return;
    uint32_t* bad = reinterpret_cast<uint32_t*>(c->dmailbox) + 8;
    DK_CUDA(cudaMemsetAsync(bad, 0, 4, s));
    DK_LAUNCH(c, range_check_kernel, dk::grid_for(total), dk::kThreads, 0, s, v.delta, total, v.n, bad);
    uint32_t b = 0;
    dk::read_words(c, bad, 4, &b, s);
    if (b) throw dk::Error(DFAKIT_E_INVALID, "delta: transition target out of range");
}

void stage(dk::Ctx* c, const dfakit_dfa* d, Staged& st, cudaStream_t s) {
    const uint64_t total = (uint64_t)d->num_states * d->alphabet_size;
    st.delta.alloc(total ? total : 1, s);
    st.acc.alloc(d->num_states ? d->num_states : 1, s);
    if (total) DK_CUDA(cudaMemcpyAsync(st.delta.get(), d->delta, total * 4, cudaMemcpyHostToDevice, s));
    if (d->num_states) DK_CUDA(cudaMemcpyAsync(st.acc.get(), d->accepting, d->num_states, cudaMemcpyHostToDevice, s));
    st.view = dk::DevDfa{d->num_states, d->alphabet_size, st.delta.get(), st.acc.get(), d->initial};
    validate_device(c, st.view, s);
}

dk::DevDfa device_view(const dfakit_dfa* d) {
    return dk::DevDfa{d->num_states, d->alphabet_size, d->delta, d->accepting, d->initial};
}

void fill_report(dfakit_report* r, const dk::RefineResult& rr, uint32_t algo, uint32_t n, uint32_t k, float ms) {
    if (!r) return;
    std::memset(r, 0, sizeof(*r));
    r->num_blocks = rr.num_blocks;
    r->refining_iterations = rr.iters;
    r->closure_iterations = rr.closure;
    r->algorithm = algo;
    r->passes = rr.passes;
    r->transitions_refined = (uint64_t)n * k * rr.passes;
    r->states_sorted = rr.sorted;
    r->hash_collisions = rr.collisions;
    r->device_ms = ms;
}

constexpr uint32_t kStreamMinStates = 1u << 20;  // below this the copy is too short to split
constexpr uint32_t kStreamChunks = 8;

dk::RefineResult run_sort_streamed(dk::Ctx* c, const dk::DevDfa& v, const dfakit_options* o, uint32_t* block_out,
                                   cudaStream_t s, const dk::DeltaStream* ds) {
    dfakit_options def{};
    if (!o) o = &def;
    dk::SortOptions so;
    so.force_exact = o->force_exact != 0;
    so.fingerprint_bits = o->fingerprint_bits ? o->fingerprint_bits : 64;
    so.grouping = o->grouping;
    return dk::sort_pr_device(c, v, so, block_out, s, ds);
}

dk::RefineResult run_algo(dk::Ctx* c, const dk::DevDfa& v, dfakit_algorithm algo, const dfakit_options* o,
                          uint32_t* block_out, uint8_t* apart_dev, cudaStream_t s) {
    dfakit_options def{};
    if (!o) o = &def;
    switch (algo) {
        case DFAKIT_ALGO_MOORE:
        case DFAKIT_ALGO_SORT_PR: {
            dk::SortOptions so;
            so.force_exact = o->force_exact != 0;
            so.fingerprint_bits = o->fingerprint_bits ? o->fingerprint_bits : 64;
            so.grouping = o->grouping;
            return dk::sort_pr_device(c, v, so, block_out, s);
        }
        case DFAKIT_ALGO_NAIVE_PR:
            return dk::naive_pr_device(c, v, (int)o->policy, o->seed, block_out, s);
        case DFAKIT_ALGO_NAIVE_PR_FUSED:
            return dk::naive_pr_fused_device(c, v, block_out, s);
        case DFAKIT_ALGO_TRANS_PR:
            return dk::trans_pr_device(c, v, (int)o->policy, o->seed,
                                       o->max_transitions ? o->max_transitions : kDefaultMaxTransitions, block_out, s);
        case DFAKIT_ALGO_TRANS:
            return dk::trans_minimize_device(c, v, o->max_pair_nodes ? o->max_pair_nodes : kDefaultMaxPairNodes,
                                             block_out, apart_dev, s);
    }
    throw dk::Error(DFAKIT_E_INVALID, "unknown algorithm");
}

void minimize_host(dfakit_ctx* ctx, const dfakit_dfa* dfa, dfakit_algorithm algo, const dfakit_options* opts,
                   uint32_t* block_of, uint8_t* apart, dfakit_report* report) {
    if (!ctx) throw dk::Error(DFAKIT_E_INVALID, "null context");
    check_view(dfa, "minimize");
    dk::Ctx* c = ctx->c;
    DK_CUDA(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    const uint32_t n = dfa->num_states, k = dfa->alphabet_size;
    const bool sortish = algo == DFAKIT_ALGO_SORT_PR || algo == DFAKIT_ALGO_MOORE;
    const bool stream_in = sortish && (!opts || opts->grouping != 1) && n >= kStreamMinStates && k > 0;
    Staged st;
    dk::DeltaStream ds;
    std::vector<uint32_t> bounds;
    std::vector<cudaEvent_t> ready;
    if (stream_in) {
        // delta in state-range chunks on the copy stream; pass 1 consumes
        // them as they land (validation included), hiding under the copy
        const uint64_t total = (uint64_t)n * k;
        st.delta.alloc(total, s);
        st.acc.alloc(n, s);
        DK_CUDA(cudaMemcpyAsync(st.acc.get(), dfa->accepting, n, cudaMemcpyHostToDevice, s));
        if (!c->copy_stream) DK_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        cudaEvent_t allocated;
        DK_CUDA(cudaEventCreateWithFlags(&allocated, cudaEventDisableTiming));
        DK_CUDA(cudaEventRecord(allocated, s));
        DK_CUDA(cudaStreamWaitEvent(c->copy_stream, allocated, 0));
        cudaEventDestroy(allocated);
        const uint32_t chunks = kStreamChunks;
        for (uint32_t i = 0; i <= chunks; ++i) bounds.push_back((uint32_t)((uint64_t)n * i / chunks));
        ready.resize(chunks);
        for (uint32_t i = 0; i < chunks; ++i) {
            const uint32_t q0 = bounds[i], q1 = bounds[i + 1];
            DK_CUDA(cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming));
            if (q1 > q0)
                DK_CUDA(cudaMemcpy2DAsync(st.delta.get() + q0, (size_t)n * 4, dfa->delta + q0, (size_t)n * 4,
                                          (size_t)(q1 - q0) * 4, k, cudaMemcpyHostToDevice, c->copy_stream));
            DK_CUDA(cudaEventRecord(ready[i], c->copy_stream));
        }
        st.view = dk::DevDfa{n, k, st.delta.get(), st.acc.get(), dfa->initial};
        ds.chunks = chunks;
        ds.bounds = bounds.data();
        ds.ready = ready.data();
    } else {
        stage(c, dfa, st, s);
    }
    struct EventsGuard {  // every exit (errors included) drains the copy stream first
        std::vector<cudaEvent_t>& e;
        cudaStream_t cs;
        ~EventsGuard() {
            if (cs && !e.empty()) cudaStreamSynchronize(cs);
            for (auto x : e) cudaEventDestroy(x);
        }
    } guard_events{ready, c->copy_stream};
    dk::DBuf<uint32_t> blocks(n ? n : 1, s);
    dk::DBuf<uint8_t> ap;
    if (apart && algo == DFAKIT_ALGO_TRANS) ap.alloc((uint64_t)n * n ? (uint64_t)n * n : 1, s);
    DK_CUDA(cudaEventRecord(c->ev0, s));
    dk::RefineResult rr = stream_in ? run_sort_streamed(c, st.view, opts, blocks.get(), s, &ds)
                                    : run_algo(c, st.view, algo, opts, blocks.get(), ap.get(), s);
    DK_CUDA(cudaEventRecord(c->ev1, s));
    if (n && block_of) DK_CUDA(cudaMemcpyAsync(block_of, blocks.get(), (size_t)n * 4, cudaMemcpyDeviceToHost, s));
    if (ap.get() && n) DK_CUDA(cudaMemcpyAsync(apart, ap.get(), (size_t)n * n, cudaMemcpyDeviceToHost, s));
    DK_CUDA(cudaStreamSynchronize(s));
    float ms = 0;
    DK_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    fill_report(report, rr, algo, n, dfa->alphabet_size, ms);
}

void product_host(dfakit_ctx* ctx, const dfakit_dfa* a, const dfakit_dfa* b, dfakit_mode mode,
                  const uint32_t* letter_map, uint64_t max_visited, uint32_t* cex, uint32_t cap, dfakit_product* out,
                  bool uf, bool staged_input, cudaStream_t user_stream) {
    if (!ctx) throw dk::Error(DFAKIT_E_INVALID, "null context");
    check_view(a, "explore_product");
    check_view(b, "explore_product");
    if (a->initial < 0 || b->initial < 0)
        throw dk::Error(DFAKIT_E_INVALID, "product exploration requires initial states on both inputs");
    if (!letter_map && a->alphabet_size != b->alphabet_size)
        throw dk::Error(DFAKIT_E_INVALID, "alphabet size mismatch: " + std::to_string(a->alphabet_size) + " vs " +
                                              std::to_string(b->alphabet_size));
    if (letter_map)
        for (uint32_t i = 0; i < a->alphabet_size; ++i)
            if (letter_map[i] >= b->alphabet_size) throw dk::Error(DFAKIT_E_INVALID, "letter map out of range");
    dk::Ctx* c = ctx->c;
    DK_CUDA(cudaSetDevice(c->device));
    cudaStream_t s = user_stream ? user_stream : c->stream;
    Staged sa, sb;
    dk::DevDfa va, vb;
    if (staged_input) {
        stage(c, a, sa, s);
        stage(c, b, sb, s);
        va = sa.view;
        vb = sb.view;
    } else {
        va = device_view(a);
        vb = device_view(b);
    }
    DK_CUDA(cudaEventRecord(c->ev0, s));
    dk::ProductOut po = uf ? dk::check_equiv_uf_device(c, va, vb, s)
                           : dk::explore_product_device(c, va, vb, (int)mode, letter_map, max_visited, s);
    DK_CUDA(cudaEventRecord(c->ev1, s));
    DK_CUDA(cudaStreamSynchronize(s));
    float ms = 0;
    DK_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    if (out) {
        std::memset(out, 0, sizeof(*out));
        out->verdict = po.verdict;
        out->levels = po.levels;
        out->explored_states = po.explored;
        out->counterexample_len = (uint32_t)po.word.size();
        out->device_ms = ms;
    }
    if (cex)
        for (uint32_t i = 0; i < cap && i < po.word.size(); ++i) cex[i] = po.word[i];
}

}  // namespace

namespace {
dk::PassPlan plan_in(const dfakit_pass_plan* p) {
    if (!p) throw dk::Error(DFAKIT_E_INVALID, "null plan");
    dk::PassPlan q;
    q.strategy = p->strategy;
    q.field_bits = p->field_bits;
    q.key_bits = p->key_bits;
    q.keylab_bytes = p->keylab_bytes;
    return q;
}
template <typename F>
dfakit_status on_device(dfakit_ctx* ctx, void* stream, F&& f) {
    return guard([&] {
        if (!ctx) throw dk::Error(DFAKIT_E_INVALID, "null context");
        DK_CUDA(cudaSetDevice(ctx->c->device));
        f(ctx->c, stream ? (cudaStream_t)stream : ctx->c->stream);
    });
}
}  // namespace

extern "C" {

int dfakit_abi_version(void) { return DFAKIT_B200_ABI_VERSION; }

const char* dfakit_last_error(void) { return g_last_error.c_str(); }

int dfakit_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

dfakit_status dfakit_ctx_create(int device, dfakit_ctx** out) {
    return guard([&] {
        if (!out) throw dk::Error(DFAKIT_E_INVALID, "null out");
        *out = nullptr;
        dk::Ctx* c = dk::ctx_create(device);
        *out = new dfakit_ctx{c};
    });
}

void dfakit_ctx_destroy(dfakit_ctx* ctx) {
    if (!ctx) return;
    dk::ctx_destroy(ctx->c);
    delete ctx;
}

void* dfakit_ctx_stream(dfakit_ctx* ctx) { return ctx ? (void*)ctx->c->stream : nullptr; }

uint64_t dfakit_ctx_kernel_launches(dfakit_ctx* ctx) { return ctx ? ctx->c->launches : 0; }

dfakit_status dfakit_profile_begin(dfakit_ctx* ctx) {
    return guard([&] {
        if (!ctx) throw dk::Error(DFAKIT_E_INVALID, "null context");
        dk::prof_collect(ctx->c);
        ctx->c->profiling = true;
    });
}

dfakit_status dfakit_profile_end(dfakit_ctx* ctx, char* json, size_t cap) {
    return guard([&] {
        if (!ctx) throw dk::Error(DFAKIT_E_INVALID, "null context");
        ctx->c->profiling = false;
        std::string s = dk::prof_collect(ctx->c);
        if (json && cap) {
            std::strncpy(json, s.c_str(), cap - 1);
            json[cap - 1] = 0;
        }
        if (s.size() + 1 > cap) throw dk::Error(DFAKIT_E_RESOURCE, "profile buffer too small");
    });
}

dfakit_status dfakit_minimize(dfakit_ctx* ctx, const dfakit_dfa* dfa, dfakit_algorithm algo,
                              const dfakit_options* opts, uint32_t* block_of, dfakit_report* report) {
    return guard([&] { minimize_host(ctx, dfa, algo, opts, block_of, nullptr, report); });
}

dfakit_status dfakit_moore_minimize(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint32_t* block_of,
                                    dfakit_report* report) {
    return guard([&] { minimize_host(ctx, dfa, DFAKIT_ALGO_MOORE, nullptr, block_of, nullptr, report); });
}

dfakit_status dfakit_sort_pr(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint32_t* block_of, dfakit_report* report) {
    return guard([&] { minimize_host(ctx, dfa, DFAKIT_ALGO_SORT_PR, nullptr, block_of, nullptr, report); });
}

dfakit_status dfakit_naive_pr(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint32_t policy, uint64_t seed,
                              uint32_t* block_of, dfakit_report* report) {
    return guard([&] {
        dfakit_options o{};
        o.policy = policy;
        o.seed = seed;
        minimize_host(ctx, dfa, DFAKIT_ALGO_NAIVE_PR, &o, block_of, nullptr, report);
    });
}

dfakit_status dfakit_naive_pr_fused(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint32_t* block_of,
                                    dfakit_report* report) {
    return guard([&] { minimize_host(ctx, dfa, DFAKIT_ALGO_NAIVE_PR_FUSED, nullptr, block_of, nullptr, report); });
}

dfakit_status dfakit_trans_pr(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint32_t policy, uint64_t seed,
                              uint64_t max_transitions, uint32_t* block_of, dfakit_report* report) {
    return guard([&] {
        dfakit_options o{};
        o.policy = policy;
        o.seed = seed;
        o.max_transitions = max_transitions;
        minimize_host(ctx, dfa, DFAKIT_ALGO_TRANS_PR, &o, block_of, nullptr, report);
    });
}

dfakit_status dfakit_trans_minimize(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint64_t max_pair_nodes,
                                    uint32_t* block_of, uint8_t* apart, dfakit_report* report) {
    return guard([&] {
        dfakit_options o{};
        o.max_pair_nodes = max_pair_nodes;
        minimize_host(ctx, dfa, DFAKIT_ALGO_TRANS, &o, block_of, apart, report);
    });
}

dfakit_status dfakit_build_transitive_alphabet(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint64_t max_transitions,
                                               uint32_t* out_delta, uint32_t* out_alphabet) {
    return guard([&] {
        if (!ctx) throw dk::Error(DFAKIT_E_INVALID, "null context");
        check_view(dfa, "build_transitive_alphabet");
        const uint32_t levels = dk::floor_log2_u32(dfa->num_states) + 1;
        const uint64_t total = (uint64_t)dfa->alphabet_size * levels * dfa->num_states;
        if (!max_transitions) max_transitions = kDefaultMaxTransitions;
        if (total > max_transitions)
            throw dk::Error(DFAKIT_E_RESOURCE, "build_transitive_alphabet: doubled alphabet needs " +
                                                   std::to_string(total) + " transition entries; budget is " +
                                                   std::to_string(max_transitions));
        if (out_alphabet) *out_alphabet = dfa->alphabet_size * levels;
        if (!out_delta) return;
        dk::Ctx* c = ctx->c;
        DK_CUDA(cudaSetDevice(c->device));
        cudaStream_t s = c->stream;
        Staged st;
        stage(c, dfa, st, s);
        dk::DBuf<uint32_t> out(total ? total : 1, s);
        dk::transitive_alphabet_device(c, st.view, out.get(), s);
        if (total) DK_CUDA(cudaMemcpyAsync(out_delta, out.get(), total * 4, cudaMemcpyDeviceToHost, s));
        DK_CUDA(cudaStreamSynchronize(s));
    });
}

dfakit_status dfakit_minimize_device(dfakit_ctx* ctx, const dfakit_dfa* dfa, dfakit_algorithm algo,
                                     const dfakit_options* opts, uint32_t* block_of, dfakit_report* report,
                                     void* stream) {
    return guard([&] {
        if (!ctx) throw dk::Error(DFAKIT_E_INVALID, "null context");
        check_view(dfa, "minimize_device");
        dk::Ctx* c = ctx->c;
        DK_CUDA(cudaSetDevice(c->device));
        cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
        DK_CUDA(cudaEventRecord(c->ev0, s));
        dk::RefineResult rr = run_algo(c, device_view(dfa), algo, opts, block_of, nullptr, s);
        DK_CUDA(cudaEventRecord(c->ev1, s));
        DK_CUDA(cudaEventSynchronize(c->ev1));
        float ms = 0;
        DK_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        fill_report(report, rr, algo, dfa->num_states, dfa->alphabet_size, ms);
    });
}

dfakit_status dfakit_explore_product(dfakit_ctx* ctx, const dfakit_dfa* a, const dfakit_dfa* b, dfakit_mode mode,
                                     const uint32_t* letter_map, uint64_t max_visited, uint32_t* counterexample,
                                     uint32_t counterexample_cap, dfakit_product* out) {
    return guard([&] {
        product_host(ctx, a, b, mode, letter_map, max_visited, counterexample, counterexample_cap, out, false, true,
                     nullptr);
    });
}

dfakit_status dfakit_check_equiv(dfakit_ctx* ctx, const dfakit_dfa* a, const dfakit_dfa* b, uint64_t max_visited,
                                 uint32_t* counterexample, uint32_t counterexample_cap, dfakit_product* out) {
    return dfakit_explore_product(ctx, a, b, DFAKIT_MODE_EQUIVALENCE, nullptr, max_visited, counterexample,
                                  counterexample_cap, out);
}

dfakit_status dfakit_check_inclusion(dfakit_ctx* ctx, const dfakit_dfa* a, const dfakit_dfa* b,
                                     uint64_t max_visited, uint32_t* counterexample, uint32_t counterexample_cap,
                                     dfakit_product* out) {
    return dfakit_explore_product(ctx, a, b, DFAKIT_MODE_INCLUSION, nullptr, max_visited, counterexample,
                                  counterexample_cap, out);
}

dfakit_status dfakit_explore_product_device(dfakit_ctx* ctx, const dfakit_dfa* a, const dfakit_dfa* b,
                                            dfakit_mode mode, const uint32_t* letter_map_host, uint64_t max_visited,
                                            uint32_t* counterexample, uint32_t counterexample_cap,
                                            dfakit_product* out, void* stream) {
    return guard([&] {
        product_host(ctx, a, b, mode, letter_map_host, max_visited, counterexample, counterexample_cap, out, false,
                     false, (cudaStream_t)stream);
    });
}

dfakit_status dfakit_check_equiv_uf(dfakit_ctx* ctx, const dfakit_dfa* a, const dfakit_dfa* b,
                                    uint32_t* counterexample, uint32_t counterexample_cap, dfakit_product* out) {
    return guard([&] {
        product_host(ctx, a, b, DFAKIT_MODE_EQUIVALENCE, nullptr, ~0ull, counterexample, counterexample_cap, out, true,
                     true, nullptr);
    });
}

dfakit_status dfakit_check_equiv_uf_device(dfakit_ctx* ctx, const dfakit_dfa* a, const dfakit_dfa* b,
                                           uint32_t* counterexample, uint32_t counterexample_cap,
                                           dfakit_product* out, void* stream) {
    return guard([&] {
        product_host(ctx, a, b, DFAKIT_MODE_EQUIVALENCE, nullptr, ~0ull, counterexample, counterexample_cap, out, true,
                     false, (cudaStream_t)stream);
    });
}

dfakit_status dfakit_gen_synth_device(dfakit_ctx* ctx, uint32_t n, uint32_t k, uint64_t seed, uint32_t* delta,
                                      uint8_t* accepting, void* stream) {
    return guard([&] {
        if (!ctx) throw dk::Error(DFAKIT_E_INVALID, "null context");
        DK_CUDA(cudaSetDevice(ctx->c->device));
        dk::gen_synth_device(ctx->c, n, k, seed, delta, accepting, stream ? (cudaStream_t)stream : ctx->c->stream);
    });
}

dfakit_status dfakit_gen_chain_device(dfakit_ctx* ctx, uint32_t n, uint32_t* delta, uint8_t* accepting,
                                      void* stream) {
    return guard([&] {
        if (!ctx) throw dk::Error(DFAKIT_E_INVALID, "null context");
        DK_CUDA(cudaSetDevice(ctx->c->device));
        dk::gen_chain_device(ctx->c, n, delta, accepting, stream ? (cudaStream_t)stream : ctx->c->stream);
    });
}

dfakit_status dfakit_permute_states_device(dfakit_ctx* ctx, uint32_t n, uint32_t k, uint64_t seed,
                                           const uint32_t* delta, const uint8_t* accepting, uint32_t* out_delta,
                                           uint8_t* out_accepting, uint32_t* initial_out, void* stream) {
    return guard([&] {
        if (!ctx) throw dk::Error(DFAKIT_E_INVALID, "null context");
        DK_CUDA(cudaSetDevice(ctx->c->device));
        uint32_t init = dk::permute_states_device(ctx->c, n, k, seed, delta, accepting, out_delta, out_accepting,
                                                  stream ? (cudaStream_t)stream : ctx->c->stream);
        if (initial_out) *initial_out = init;
    });
}

dfakit_status dfakit_comm_unique_id(uint8_t* id128) {
    return guard([&] {
        if (!id128) throw dk::Error(DFAKIT_E_INVALID, "null id");
        dk::nccl_unique_id(id128);
    });
}

dfakit_status dfakit_comm_init(dfakit_ctx* ctx, const uint8_t* id128, int world, int rank, dfakit_comm** out) {
    return on_device(ctx, nullptr, [&](dk::Ctx* c, cudaStream_t) {
        if (!id128 || !out) throw dk::Error(DFAKIT_E_INVALID, "null argument");
        *out = nullptr;
        dk::NcclComm* nc = dk::nccl_comm_init(c, id128, world, rank);
        *out = new dfakit_comm{nc};
    });
}

void dfakit_comm_destroy(dfakit_comm* comm) {
    if (!comm) return;
    dk::nccl_comm_destroy(comm->c);
    delete comm;
}

dfakit_status dfakit_local_hub_create(int world, dfakit_local_hub** out) {
    return guard([&] {
        if (!out) throw dk::Error(DFAKIT_E_INVALID, "null out");
        *out = new dfakit_local_hub{dk::local_hub_create(world)};
    });
}

void dfakit_local_hub_destroy(dfakit_local_hub* hub) {
    if (!hub) return;
    dk::local_hub_destroy(hub->h);
    delete hub;
}

dfakit_status dfakit_comm_init_local(dfakit_local_hub* hub, int rank, dfakit_comm** out) {
    return guard([&] {
        if (!hub || !out) throw dk::Error(DFAKIT_E_INVALID, "null argument");
        *out = new dfakit_comm{dk::local_comm_init(hub->h, rank)};
    });
}

dfakit_status dfakit_sort_pr_sharded(dfakit_ctx* ctx, dfakit_comm* comm, const dfakit_dfa* dfa, uint32_t* block_of,
                                     dfakit_report* report, uint64_t* exchanged, void* stream) {
    return on_device(ctx, stream, [&](dk::Ctx* c, cudaStream_t s) {
        if (!comm) throw dk::Error(DFAKIT_E_INVALID, "null communicator");
        check_view(dfa, "sort_pr_sharded");
        DK_CUDA(cudaEventRecord(c->ev0, s));
        const dk::RefineResult rr = dk::sort_pr_sharded_device(c, comm->c, device_view(dfa), block_of, s, exchanged);
        DK_CUDA(cudaEventRecord(c->ev1, s));
        DK_CUDA(cudaEventSynchronize(c->ev1));
        float ms = 0;
        DK_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        fill_report(report, rr, DFAKIT_ALGO_SORT_PR, dfa->num_states, dfa->alphabet_size, ms);
    });
}

dfakit_status dfakit_sort_pr_sharded_host(dfakit_ctx* ctx, dfakit_comm* comm, const dfakit_dfa* dfa,
                                          uint32_t* block_of, dfakit_report* report) {
    return guard([&] {
        if (!ctx) throw dk::Error(DFAKIT_E_INVALID, "null context");
        if (!comm) throw dk::Error(DFAKIT_E_INVALID, "null communicator");
        check_view(dfa, "sort_pr_sharded");
        dk::Ctx* c = ctx->c;
        DK_CUDA(cudaSetDevice(c->device));
        cudaStream_t s = c->stream;
        Staged st;
        stage(c, dfa, st, s);
        const uint32_t n = dfa->num_states;
        dk::DBuf<uint32_t> blocks(n ? n : 1, s);
        DK_CUDA(cudaEventRecord(c->ev0, s));
        const dk::RefineResult rr = dk::sort_pr_sharded_device(c, comm->c, st.view, blocks.get(), s, nullptr);
        DK_CUDA(cudaEventRecord(c->ev1, s));
        if (n && block_of) DK_CUDA(cudaMemcpyAsync(block_of, blocks.get(), (size_t)n * 4, cudaMemcpyDeviceToHost, s));
        DK_CUDA(cudaStreamSynchronize(s));
        float ms = 0;
        DK_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        fill_report(report, rr, DFAKIT_ALGO_SORT_PR, n, dfa->alphabet_size, ms);
    });
}

dfakit_status dfakit_radix_sort_pairs_device(dfakit_ctx* ctx, uint64_t* keys, uint32_t* vals, uint64_t* keys_alt,
                                             uint32_t* vals_alt, uint64_t count, uint32_t key_bits,
                                             int32_t* result_in_alt, void* stream) {
    return on_device(ctx, stream, [&](dk::Ctx* c, cudaStream_t s) {
        if (key_bits > 64) throw dk::Error(DFAKIT_E_INVALID, "radix_sort_pairs: key_bits > 64");
        if (count && (!keys || !vals || !keys_alt || !vals_alt))
            throw dk::Error(DFAKIT_E_INVALID, "radix_sort_pairs: null buffer");
        const bool flipped = dk::radix_sort_pairs(c, dk::RadixBuffers{keys, vals, keys_alt, vals_alt}, count, key_bits, s);
        if (result_in_alt) *result_in_alt = flipped ? 1 : 0;
    });
}

dfakit_status dfakit_calibrate_gather(dfakit_ctx* ctx, uint64_t table_words, uint32_t elem_bytes, uint64_t gathers,
                                      double* gathers_per_s) {
    return on_device(ctx, nullptr, [&](dk::Ctx* c, cudaStream_t s) {
        if (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4)
            throw dk::Error(DFAKIT_E_INVALID, "calibrate_gather: elem_bytes must be 1, 2 or 4");
        const double r = dk::calibrate_gather(c, table_words ? table_words : 1, elem_bytes, gathers, s, nullptr);
        if (gathers_per_s) *gathers_per_s = r;
    });
}

// ---- sharded sort_pr primitives ------------------------------------------------

dfakit_status dfakit_plan_pass(uint32_t num_states, uint32_t alphabet_size, uint32_t num_blocks,
                               uint64_t active_states, uint32_t collisions, uint32_t force_exact,
                               dfakit_pass_plan* out) {
    return guard([&] {
        if (!out) throw dk::Error(DFAKIT_E_INVALID, "null plan");
        const dk::PassPlan p = dk::plan_pass(num_states, alphabet_size, num_blocks, active_states, collisions,
                                             force_exact != 0);
        *out = dfakit_pass_plan{p.strategy, p.field_bits, p.key_bits, p.keylab_bytes};
    });
}


dfakit_status dfakit_shard_init(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint32_t lo, uint32_t hi, uint32_t* lab,
                                uint8_t* act, uint32_t* num_blocks, uint32_t* active_blocks,
                                uint64_t* active_states, void* stream) {
    return on_device(ctx, stream, [&](dk::Ctx* c, cudaStream_t s) {
        check_view(dfa, "shard_init");
        if (lo > hi || hi > dfa->num_states) throw dk::Error(DFAKIT_E_INVALID, "shard_init: bad state range");
        const dk::ShardInit r = dk::shard_init(c, device_view(dfa), lo, hi, lab, act, s);
        if (num_blocks) *num_blocks = r.num_blocks;
        if (active_blocks) *active_blocks = r.active_blocks;
        if (active_states) *active_states = r.active_states;
    });
}

dfakit_status dfakit_shard_keylab(dfakit_ctx* ctx, const uint32_t* lab, uint32_t n, uint32_t num_blocks,
                                  const dfakit_pass_plan* plan, void* keylab, void* stream) {
    return on_device(ctx, stream, [&](dk::Ctx* c, cudaStream_t s) {
        const dk::PassPlan p = plan_in(plan);
        if (!p.keylab_bytes || !n) return;
        dk::DBuf<uint32_t> scratch(num_blocks <= 2 ? 1 : (uint64_t)n + 1, s);
        dk::shard_keylab(c, lab, n, num_blocks, p, keylab, scratch.get(), s);
    });
}

dfakit_status dfakit_shard_table_signature(dfakit_ctx* ctx, const dfakit_dfa* dfa, const void* keylab,
                                           const dfakit_pass_plan* plan, const uint32_t* list, uint32_t list_base,
                                           uint64_t m, uint32_t* keys32, uint32_t* tmin, uint32_t* tcnt,
                                           void* stream) {
    return on_device(ctx, stream, [&](dk::Ctx* c, cudaStream_t s) {
        check_view(dfa, "shard_table_signature");
        const dk::PassPlan p = plan_in(plan);
        if (p.strategy != dk::kPlanTable || p.key_bits > 20)
            throw dk::Error(DFAKIT_E_INVALID, "shard_table_signature: not a table plan");
        dk::shard_table_signature(c, device_view(dfa), keylab, p, list, list_base, m, keys32, tmin, tcnt, s);
    });
}

dfakit_status dfakit_shard_table_apply(dfakit_ctx* ctx, const dfakit_pass_plan* plan, const uint32_t* list,
                                       uint32_t list_base, const uint32_t* keys32, uint64_t m, const uint32_t* tmin,
                                       const uint32_t* tcnt, uint32_t* lab, uint8_t* act, void* next_keylab,
                                       uint32_t* counters, void* stream) {
    return on_device(ctx, stream, [&](dk::Ctx* c, cudaStream_t s) {
        dk::shard_table_apply(c, plan_in(plan), list, list_base, keys32, m, tmin, tcnt, lab, act, next_keylab,
                              counters, s);
    });
}

dfakit_status dfakit_shard_partition(dfakit_ctx* ctx, const dfakit_dfa* dfa, const void* keylab,
                                     const dfakit_pass_plan* plan, uint64_t salt, const uint32_t* list,
                                     uint32_t list_base, uint64_t m, uint32_t world, void* send_entries,
                                     uint32_t* send_counts, void* stream) {
    return on_device(ctx, stream, [&](dk::Ctx* c, cudaStream_t s) {
        check_view(dfa, "shard_partition");
        const dk::PassPlan p = plan_in(plan);
        if (p.strategy != dk::kPlanPacked && p.strategy != dk::kPlanFingerprint)
            throw dk::Error(DFAKIT_E_INVALID, "shard_partition: plan is not packed / fingerprint");
        dk::shard_sig_partition(c, device_view(dfa), keylab, p, salt, list, list_base, m, world,
                                static_cast<uint4*>(send_entries), send_counts, s);
    });
}

dfakit_status dfakit_shard_group(dfakit_ctx* ctx, const dfakit_dfa* dfa, const uint32_t* lab,
                                 const dfakit_pass_plan* plan, const void* recv_entries, uint64_t count,
                                 uint32_t* results, uint32_t* counters, void* stream) {
    return on_device(ctx, stream, [&](dk::Ctx* c, cudaStream_t s) {
        check_view(dfa, "shard_group");
        if (dfa->num_states > 0x7fffffffu) throw dk::Error(DFAKIT_E_INVALID, "shard_group: more than 2^31 states");
        dk::shard_group(c, device_view(dfa), lab, 4, plan_in(plan), static_cast<const uint4*>(recv_entries), count,
                        results, counters, s);
    });
}

dfakit_status dfakit_shard_apply(dfakit_ctx* ctx, const void* send_entries, const uint32_t* results, uint64_t count,
                                 uint32_t* lab, uint8_t* act, void* stream) {
    return on_device(ctx, stream, [&](dk::Ctx* c, cudaStream_t s) {
        dk::shard_apply(c, static_cast<const uint4*>(send_entries), results, count, lab, act, s);
    });
}

dfakit_status dfakit_shard_compact(dfakit_ctx* ctx, const uint8_t* act, uint32_t lo, uint32_t hi, uint32_t* list,
                                   uint32_t* count, void* stream) {
    return on_device(ctx, stream, [&](dk::Ctx* c, cudaStream_t s) { dk::shard_compact(c, act, lo, hi, list, count, s); });
}

dfakit_status dfakit_shard_canonical(dfakit_ctx* ctx, const uint32_t* lab, uint32_t n, uint32_t* block_of,
                                     uint32_t* num_blocks, void* stream) {
    return on_device(ctx, stream, [&](dk::Ctx* c, cudaStream_t s) {
        dk::DBuf<uint32_t> scratch((uint64_t)n + 1, s);
        const uint32_t b = dk::canonical_from_min_labels(c, lab, n, block_of, scratch.get(), s);
        if (num_blocks) *num_blocks = b;
    });
}

}  // extern "C"
