/*
 * dfakit_b200.h -- C ABI of the B200-native DFA minimisation / equivalence
 * library (libdfakit_b200.so).
 *
 * Plain pointers and sizes only.  Each entry point names the reference
 * interface it replaces (/root/reference/proj/include/dfakit/...).  The C++
 * drop-in API (include/dfakit_b200.hpp, reached through the reference header
 * names under include/dfakit/, namespace dfakit) is a thin host layer over
 * these calls; see INTEGRATION.md for the bindings.
 *
 * Memory conventions
 *   - delta is letter-major: delta[a * n + q] = delta(q, a), exactly the
 *     reference's `delta[a][q]` (dfa.hpp:22-24) laid out contiguously.
 *   - accepting is one byte per state (0 / 1).
 *   - `dfakit_*` calls take HOST buffers and copy them in and out;
 *     `dfakit_*_device` calls take DEVICE pointers already resident in HBM and
 *     run on the given CUDA stream (NULL = the context's stream; pass
 *     cudaStreamLegacy, (void*)1, for the legacy default stream).
 *   - Block numbering of every returned partition is canonical: blocks are
 *     numbered by first occurrence scanning states upwards (equivalently, by
 *     the minimum state id of each block), the reference's
 *     Partition::from_labels normal form (dfa.hpp:46-60).
 *
 * Errors: every call returns a dfakit_status; dfakit_last_error() returns a
 * thread-local message for the last failure.  There is no CPU fallback: when
 * no CUDA device is present calls return DFAKIT_E_NODEVICE.
 */
#ifndef DFAKIT_B200_H
#define DFAKIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFAKIT_B200_ABI_VERSION 2
#define DFAKIT_NO_STATE 0xffffffffu

typedef enum {
    DFAKIT_OK = 0,
    DFAKIT_E_INVALID = -1,  /* std::invalid_argument in the reference          */
    DFAKIT_E_RESOURCE = -2, /* dfakit::ResourceError (errors.hpp:21-24)         */
    DFAKIT_E_CUDA = -3,     /* CUDA runtime failure                             */
    DFAKIT_E_NODEVICE = -4  /* no CUDA device: the library refuses to run       */
} dfakit_status;

/* Same order as dfakit::Algorithm (minimize.hpp:9). */
typedef enum {
    DFAKIT_ALGO_MOORE = 0,
    DFAKIT_ALGO_TRANS = 1,
    DFAKIT_ALGO_NAIVE_PR = 2,
    DFAKIT_ALGO_NAIVE_PR_FUSED = 3,
    DFAKIT_ALGO_SORT_PR = 4,
    DFAKIT_ALGO_TRANS_PR = 5
} dfakit_algorithm;

/* dfakit::ElectionPolicy (minimize.hpp:16-24). */
typedef enum { DFAKIT_POLICY_MIN_INDEX = 0, DFAKIT_POLICY_ARBITRARY = 1 } dfakit_policy;

/* dfakit::ExploreMode (equivalence.hpp:24). */
typedef enum { DFAKIT_MODE_EQUIVALENCE = 0, DFAKIT_MODE_INCLUSION = 1, DFAKIT_MODE_FULL = 2 } dfakit_mode;

/* dfakit::Verdict (equivalence.hpp:10). */
typedef enum { DFAKIT_EQUIVALENT = 0, DFAKIT_INCLUDED = 1, DFAKIT_COUNTEREXAMPLE = 2 } dfakit_verdict;

/* A DFA view (dfakit::Dfa, dfa.hpp:21-41) over caller-owned memory. */
typedef struct {
    uint32_t num_states;
    uint32_t alphabet_size;
    const uint32_t* delta;     /* alphabet_size * num_states, letter-major */
    const uint8_t* accepting;  /* num_states                               */
    int64_t initial;           /* -1 when absent                           */
} dfakit_dfa;

/* dfakit::RefinementReport (minimize.hpp:26-35) plus device statistics. */
typedef struct {
    uint32_t num_blocks;
    uint32_t refining_iterations; /* passes that changed the partition       */
    uint32_t closure_iterations;  /* trans / trans_pr only                   */
    uint32_t algorithm;           /* dfakit_algorithm                        */
    uint64_t passes;              /* passes executed incl. the confirming one */
    uint64_t transitions_refined; /* n * k * passes (algorithmic work)       */
    uint64_t states_sorted;       /* sum over passes of keys radix-sorted    */
    uint32_t hash_collisions;     /* fingerprint collisions caught + re-run  */
    uint32_t reserved;
    double device_ms;             /* device time of the call (CUDA events)   */
} dfakit_report;

/* dfakit::ProductResult (equivalence.hpp:12-22). */
typedef struct {
    int32_t verdict;              /* dfakit_verdict */
    uint32_t levels;
    uint64_t explored_states;
    uint32_t counterexample_len;  /* full length even when > capacity */
    uint32_t reserved;
    double device_ms;
} dfakit_product;

/* Options for the refinement calls. */
typedef struct {
    uint32_t policy;            /* dfakit_policy                                       */
    uint32_t force_exact;       /* sort_pr: never use fingerprint keys (testing)       */
    uint64_t seed;              /* ElectionPolicy::arbitrary seed                      */
    uint64_t max_transitions;   /* trans_pr budget, minimize.hpp:41 (0 = default 2^28) */
    uint64_t max_pair_nodes;    /* trans budget, minimize.hpp:38 (0 = default 2^16)    */
    uint32_t fingerprint_bits;  /* sort_pr: 0 = 64; smaller values force collisions    */
    uint32_t grouping;          /* sort_pr: 0 = auto (counting table / radix-bucketed
                                   shared-memory hashing; the persistent device loop
                                   once <= 2^17 states are active), 1 = full LSD radix
                                   sort of the keys + adjacent difference + scan
                                   (literal paper Alg. 4), 2 = auto without the
                                   persistent loop (every pass host-staged)          */
} dfakit_options;

typedef struct dfakit_ctx dfakit_ctx;

/* ---- context -------------------------------------------------------------- */
int dfakit_abi_version(void);
const char* dfakit_last_error(void);
/* Number of CUDA devices visible (0 when none). */
int dfakit_device_count(void);
/* Creates a context bound to `device` with its own stream and memory pool. */
dfakit_status dfakit_ctx_create(int device, dfakit_ctx** out);
void dfakit_ctx_destroy(dfakit_ctx* ctx);
/* The context's CUDA stream (cudaStream_t) as an opaque pointer. */
void* dfakit_ctx_stream(dfakit_ctx* ctx);
/* Number of kernels this context has launched so far. */
uint64_t dfakit_ctx_kernel_launches(dfakit_ctx* ctx);
/* Live kernel profiling: between begin and end every launch is bracketed by
 * CUDA events on its stream.  end() writes per-kernel totals as JSON
 * [{"name","launches","ms","bytes"}] where bytes are the algorithmic bytes
 * annotated at the launch site ("roofline"). */
dfakit_status dfakit_profile_begin(dfakit_ctx* ctx);
dfakit_status dfakit_profile_end(dfakit_ctx* ctx, char* json, size_t cap);

/* ---- minimisation: host buffers (minimize.hpp:46-85) ------------------------
 * block_of: num_states entries, canonical numbering.  opts may be NULL.    */
dfakit_status dfakit_minimize(dfakit_ctx* ctx, const dfakit_dfa* dfa, dfakit_algorithm algo,
                              const dfakit_options* opts, uint32_t* block_of, dfakit_report* report);
/* moore_minimize, minimize.hpp:46 (GPU signature refinement; same partition
 * and pass count as Moore's sequential refinement). */
dfakit_status dfakit_moore_minimize(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint32_t* block_of,
                                    dfakit_report* report);
/* sort_pr, minimize.hpp:72 */
dfakit_status dfakit_sort_pr(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint32_t* block_of, dfakit_report* report);
/* naive_pr, minimize.hpp:62 */
dfakit_status dfakit_naive_pr(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint32_t policy, uint64_t seed,
                              uint32_t* block_of, dfakit_report* report);
/* naive_pr_fused, minimize.hpp:66 */
dfakit_status dfakit_naive_pr_fused(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint32_t* block_of,
                                    dfakit_report* report);
/* trans_pr, minimize.hpp:82 */
dfakit_status dfakit_trans_pr(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint32_t policy, uint64_t seed,
                              uint64_t max_transitions, uint32_t* block_of, dfakit_report* report);
/* trans_minimize, minimize.hpp:55 (Cai-Haase pair-graph closure; small n).
 * apart: optional num_states^2 bytes (row-major), may be NULL. */
dfakit_status dfakit_trans_minimize(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint64_t max_pair_nodes,
                                    uint32_t* block_of, uint8_t* apart, dfakit_report* report);
/* build_transitive_alphabet, minimize.hpp:77.  out_delta holds
 * alphabet_size * (floor(log2 n) + 1) * n entries; *out_alphabet receives
 * the new alphabet size.  Call with out_delta == NULL to query the size. */
dfakit_status dfakit_build_transitive_alphabet(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint64_t max_transitions,
                                               uint32_t* out_delta, uint32_t* out_alphabet);

/* ---- minimisation: device-resident ------------------------------------------
 * dfa->delta / dfa->accepting and block_of are device pointers. */
dfakit_status dfakit_minimize_device(dfakit_ctx* ctx, const dfakit_dfa* dfa, dfakit_algorithm algo,
                                     const dfakit_options* opts, uint32_t* block_of, dfakit_report* report,
                                     void* stream);

/* ---- equivalence / inclusion (equivalence.hpp:37-50) -------------------------
 * Naive Hopcroft-Karp: level-synchronous product BFS over a lock-free GPU
 * hash set.  Records are ordered exactly like the reference's sequential
 * insertion order, so verdict, explored_states, levels and the counterexample
 * word are identical to the reference's.  letter_map maps letters of A to
 * letters of B (NULL = positional).  counterexample receives up to
 * counterexample_cap letter ids of A. */
dfakit_status dfakit_explore_product(dfakit_ctx* ctx, const dfakit_dfa* a, const dfakit_dfa* b, dfakit_mode mode,
                                     const uint32_t* letter_map, uint64_t max_visited, uint32_t* counterexample,
                                     uint32_t counterexample_cap, dfakit_product* out);
dfakit_status dfakit_check_equiv(dfakit_ctx* ctx, const dfakit_dfa* a, const dfakit_dfa* b, uint64_t max_visited,
                                 uint32_t* counterexample, uint32_t counterexample_cap, dfakit_product* out);
dfakit_status dfakit_check_inclusion(dfakit_ctx* ctx, const dfakit_dfa* a, const dfakit_dfa* b,
                                     uint64_t max_visited, uint32_t* counterexample, uint32_t counterexample_cap,
                                     dfakit_product* out);
/* Device-resident product (a/b delta & accepting on the device). */
dfakit_status dfakit_explore_product_device(dfakit_ctx* ctx, const dfakit_dfa* a, const dfakit_dfa* b,
                                            dfakit_mode mode, const uint32_t* letter_map_host, uint64_t max_visited,
                                            uint32_t* counterexample, uint32_t counterexample_cap,
                                            dfakit_product* out, void* stream);
/* Hopcroft-Karp with a GPU union-find (path-halving CAS) -- the paper's §6
 * future work; equivalence only.  Verdict identical to check_equiv; the
 * witness (when any) is a valid distinguishing word, explored_states counts
 * the unions performed. */
dfakit_status dfakit_check_equiv_uf(dfakit_ctx* ctx, const dfakit_dfa* a, const dfakit_dfa* b,
                                    uint32_t* counterexample, uint32_t counterexample_cap, dfakit_product* out);
dfakit_status dfakit_check_equiv_uf_device(dfakit_ctx* ctx, const dfakit_dfa* a, const dfakit_dfa* b,
                                           uint32_t* counterexample, uint32_t counterexample_cap,
                                           dfakit_product* out, void* stream);

/* ---- sharded sort_pr (multi-GPU) ---------------------------------------------
 * Pass-level primitives of the sharded engine; the pass loop and the
 * collectives (NCCL all-to-all / allgather / allreduce through
 * torch.distributed) live in paper_2508_20735_b200/sharded.py.  States are
 * sharded in contiguous ranges [lo, hi); delta, accepting and the block-label
 * array `lab` (min-state labels, padded to world * shard entries) are
 * replicated on every rank.  Pointers are device pointers; `counters` is a
 * device uint32[4] = {runs, active blocks, active states, collision}.  Send /
 * receive entries are 16 bytes {hkey lo, hkey hi, state, 0}.  The plan is
 * the same on every rank (it depends on global counts only). */
typedef enum {
    DFAKIT_PLAN_TABLE = 0,       /* packed keys <= 20 bits: allreduced counting table      */
    DFAKIT_PLAN_PACKED = 1,      /* packed exact 64-bit keys: all-to-all + owner grouping   */
    DFAKIT_PLAN_FINGERPRINT = 2, /* 64-bit fingerprints, groups verified tuple by tuple     */
    DFAKIT_PLAN_CHUNKED = 3      /* exact letter chunks (single-GPU engine only)            */
} dfakit_plan_strategy;

typedef struct {
    uint32_t strategy;      /* dfakit_plan_strategy                                   */
    uint32_t field_bits;    /* packed keys: bits per field                            */
    uint32_t key_bits;      /* packed key width; 64 for fingerprints                  */
    uint32_t keylab_bytes;  /* 0: gather min-state labels; 1/2/4: dense block ids;
                               255: one bit per state (callers may set it when the
                               partition has <= 2 blocks; dfakit_shard_keylab then
                               writes a bitmap of (n + 31) / 32 words)            */
} dfakit_pass_plan;

/* Key plan of one sort_pr pass (host only; no device needed). */
dfakit_status dfakit_plan_pass(uint32_t num_states, uint32_t alphabet_size, uint32_t num_blocks,
                               uint64_t active_states, uint32_t collisions, uint32_t force_exact,
                               dfakit_pass_plan* out);
/* Initial partition {F, Q\F}: full `lab`, survivor flags act[lo, hi), global counts. */
dfakit_status dfakit_shard_init(dfakit_ctx* ctx, const dfakit_dfa* dfa, uint32_t lo, uint32_t hi, uint32_t* lab,
                                uint8_t* act, uint32_t* num_blocks, uint32_t* active_blocks,
                                uint64_t* active_states, void* stream);
/* Dense block ids of `lab` (num_blocks blocks) in plan->keylab_bytes-wide
 * entries (no-op when 0). */
dfakit_status dfakit_shard_keylab(dfakit_ctx* ctx, const uint32_t* lab, uint32_t n, uint32_t num_blocks,
                                  const dfakit_pass_plan* plan, void* keylab, void* stream);
/* `list` == NULL everywhere below: the m active states are list_base,
 * list_base + 1, ... (a shard whose states are all active).
 * Table passes: keys of the m local active states in `list`, local (min, count)
 * table of 2^key_bits entries (caller allreduces MIN / SUM), then apply.
 * next_keylab (optional; uint16 when key_bits <= 16, else uint32, indexed by
 * state): compact block ids of the new partition for the local states -- valid
 * as the next pass's key labels when this pass covered every state. */
dfakit_status dfakit_shard_table_signature(dfakit_ctx* ctx, const dfakit_dfa* dfa, const void* keylab,
                                           const dfakit_pass_plan* plan, const uint32_t* list, uint32_t list_base,
                                           uint64_t m, uint32_t* keys32, uint32_t* tmin, uint32_t* tcnt,
                                           void* stream);
dfakit_status dfakit_shard_table_apply(dfakit_ctx* ctx, const dfakit_pass_plan* plan, const uint32_t* list,
                                       uint32_t list_base, const uint32_t* keys32, uint64_t m, const uint32_t* tmin,
                                       const uint32_t* tcnt, uint32_t* lab, uint8_t* act, void* next_keylab,
                                       uint32_t* counters, void* stream);
/* Wide passes: keys of the local active states partitioned by owner rank into
 * send_entries (m entries, destination-contiguous); send_counts[world]. */
dfakit_status dfakit_shard_partition(dfakit_ctx* ctx, const dfakit_dfa* dfa, const void* keylab,
                                     const dfakit_pass_plan* plan, uint64_t salt, const uint32_t* list,
                                     uint32_t list_base, uint64_t m, uint32_t world, void* send_entries,
                                     uint32_t* send_counts, void* stream);
/* Owner side: groups the received entries; results[i] = new label | survivor << 31. */
dfakit_status dfakit_shard_group(dfakit_ctx* ctx, const dfakit_dfa* dfa, const uint32_t* lab,
                                 const dfakit_pass_plan* plan, const void* recv_entries, uint64_t count,
                                 uint32_t* results, uint32_t* counters, void* stream);
/* Home side: returned results applied to lab / act of the sent states. */
dfakit_status dfakit_shard_apply(dfakit_ctx* ctx, const void* send_entries, const uint32_t* results, uint64_t count,
                                 uint32_t* lab, uint8_t* act, void* stream);
/* Next local active list: states q in [lo, hi) with act[q] != 0, increasing. */
dfakit_status dfakit_shard_compact(dfakit_ctx* ctx, const uint8_t* act, uint32_t lo, uint32_t hi, uint32_t* list,
                                   uint32_t* count, void* stream);
/* Canonical first-occurrence numbering of min-state labels. */
dfakit_status dfakit_shard_canonical(dfakit_ctx* ctx, const uint32_t* lab, uint32_t n, uint32_t* block_of,
                                     uint32_t* num_blocks, void* stream);

/* Native sharded driver: the same pass loop in C++ with NCCL collectives on
 * the caller's stream (NCCL resolved with dlopen; DFAKIT_E_RESOURCE when no
 * libnccl.so.2 is found).  Rank 0 calls dfakit_comm_unique_id and shares the
 * 128 bytes with every rank out of band (e.g. a torch.distributed
 * broadcast); every rank then calls dfakit_comm_init and
 * dfakit_sort_pr_sharded with the full automaton resident on its device.
 * block_of (device, n entries) receives the canonical partition on every
 * rank; exchanged (optional) the entries this rank sent. */
typedef struct dfakit_comm dfakit_comm;
dfakit_status dfakit_comm_unique_id(uint8_t* id128);
dfakit_status dfakit_comm_init(dfakit_ctx* ctx, const uint8_t* id128, int world, int rank, dfakit_comm** out);
void dfakit_comm_destroy(dfakit_comm* comm);
dfakit_status dfakit_sort_pr_sharded(dfakit_ctx* ctx, dfakit_comm* comm, const dfakit_dfa* dfa, uint32_t* block_of,
                                     dfakit_report* report, uint64_t* exchanged, void* stream);
/* Same with the automaton in host memory (copied to this rank's device and
 * validated) and block_of in host memory: the C++ extension
 * dfakit::b200::sort_pr_sharded uses it. */
dfakit_status dfakit_sort_pr_sharded_host(dfakit_ctx* ctx, dfakit_comm* comm, const dfakit_dfa* dfa,
                                          uint32_t* block_of, dfakit_report* report);
/* In-process communicator: `world` ranks as threads of one process, each
 * with its own context (on any devices, e.g. all on one GPU), collectives
 * staged through host memory.  Runs the native driver's multi-rank path
 * where NCCL cannot (it refuses two ranks on one device); for testing. */
typedef struct dfakit_local_hub dfakit_local_hub;
dfakit_status dfakit_local_hub_create(int world, dfakit_local_hub** out);
void dfakit_local_hub_destroy(dfakit_local_hub* hub);
dfakit_status dfakit_comm_init_local(dfakit_local_hub* hub, int rank, dfakit_comm** out);

/* ---- primitives -----------------------------------------------------------------
 * The LSD radix sort of sortPR's literal Alg. 4 grouping (one sweep per 8-bit
 * digit, decoupled look-back): stable sort of (key, value) pairs on key bits
 * [0, key_bits), device buffers, ping-ponging between (keys, vals) and the
 * alternates; *result_in_alt = 1 when the sorted pairs ended in the
 * alternates.  Replaces the reference's std::stable_sort of (block,
 * signature) tuples (src/minimize.cpp:392). */
dfakit_status dfakit_radix_sort_pairs_device(dfakit_ctx* ctx, uint64_t* keys, uint32_t* vals, uint64_t* keys_alt,
                                             uint32_t* vals_alt, uint64_t count, uint32_t key_bits,
                                             int32_t* result_in_alt, void* stream);

/* ---- calibration ---------------------------------------------------------------
 * Measured ceiling of the signature kernels' random block-label gathers:
 * independent random gathers of elem_bytes (1, 2, 4) from a table of
 * table_words entries (L2-resident as far as it fits), every SM busy.
 * *gathers_per_s receives the rate (used by bench.py as the gather roofline). */
dfakit_status dfakit_calibrate_gather(dfakit_ctx* ctx, uint64_t table_words, uint32_t elem_bytes, uint64_t gathers,
                                      double* gathers_per_s);

/* ---- device generators (bench inputs built in HBM) --------------------------- */
/* Synthetic random DFA, same formula as oracle/oracle.c or_gen_synth. */
dfakit_status dfakit_gen_synth_device(dfakit_ctx* ctx, uint32_t n, uint32_t k, uint64_t seed, uint32_t* delta,
                                      uint8_t* accepting, void* stream);
/* Unary chain q -> q+1 (last state loops and accepts). */
dfakit_status dfakit_gen_chain_device(dfakit_ctx* ctx, uint32_t n, uint32_t* delta, uint8_t* accepting,
                                      void* stream);
/* Relabel states by a seeded bijection: out(perm(q)) = perm(in(q)).  Used to
 * build a language-equal partner DFA for equivalence benchmarks. */
dfakit_status dfakit_permute_states_device(dfakit_ctx* ctx, uint32_t n, uint32_t k, uint64_t seed,
                                           const uint32_t* delta, const uint8_t* accepting, uint32_t* out_delta,
                                           uint8_t* out_accepting, uint32_t* initial_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DFAKIT_B200_H */
