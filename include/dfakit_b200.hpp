// dfakit_b200.hpp -- C++ drop-in API.
//
// Declares, in namespace dfakit, the same types and functions as the
// reference library's public headers (/root/reference/proj/include/dfakit/
// dfa.hpp, io.hpp, minimize.hpp, equivalence.hpp, generators.hpp, lts.hpp,
// errors.hpp) so existing call sites compile unchanged against
// include/dfakit/*.hpp (one-line forwarders to this file) and link against
// libdfakit_b200.so.  Minimisation and product exploration run on the GPU
// through the C ABI (dfakit_b200.h); parsing, generators, quotient /
// pruning / canonicalisation and the .aut pipeline are host-side plumbing.
#pragma once

#include <cstddef>
#include <array>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace dfakit {

// ---- identifiers & errors (dfa.hpp:11-16, errors.hpp) ------------------------

using StateId = std::uint32_t;
using LetterId = std::uint32_t;
inline constexpr StateId kNoState = static_cast<StateId>(-1);

/// Malformed input text; `line()` is 1-based.
class ParseError : public std::runtime_error {
public:
    ParseError(std::size_t line, const std::string& reason);
    std::size_t line() const { return line_; }

private:
    std::size_t line_;
};

/// A memory / state / time budget would be exceeded.
class ResourceError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

// ---- automata (dfa.hpp) ---------------------------------------------------------

/// Complete DFA, letter-major transitions: delta[a][q].  The initial state
/// is optional (minimisation only needs the transition structure).
struct Dfa {
    StateId num_states = 0;
    LetterId alphabet_size = 0;
    std::vector<std::vector<StateId>> delta;
    std::vector<bool> accepting;
    std::optional<StateId> initial;
    std::optional<std::vector<std::string>> letter_names;

    StateId step(StateId q, LetterId a) const { return delta[a][q]; }
    StateId run(StateId q, std::span<const LetterId> word) const {
        for (LetterId a : word) q = delta[a][q];
        return q;
    }
    bool is_accepting(StateId q) const { return accepting[q]; }
    bool operator==(const Dfa&) const = default;
};

std::vector<std::string> validate(const Dfa& dfa);

/// Block id per state, always in first-occurrence normal form.
struct Partition {
    std::vector<StateId> block_of;
    StateId num_blocks = 0;

    static Partition from_labels(std::span<const StateId> labels);
    static Partition identity(StateId n);
    static Partition single_block(StateId n);
    bool operator==(const Partition&) const = default;
};

/// Symmetric, irreflexive inequivalence relation, bit-packed n x n.
class ApartMatrix {
public:
    explicit ApartMatrix(StateId n);
    StateId num_states() const { return n_; }
    bool apart(StateId q, StateId r) const {
        const std::size_t i = static_cast<std::size_t>(q) * n_ + r;
        return (words_[i >> 6] >> (i & 63)) & 1u;
    }
    void set_apart(StateId q, StateId r);

private:
    StateId n_;
    std::vector<std::uint64_t> words_;
};

Dfa quotient(const Dfa& dfa, const Partition& p);
std::pair<Dfa, std::vector<StateId>> prune_unreachable(const Dfa& dfa);
Dfa canonical_form(const Dfa& dfa);
Partition partition_from_apart(const ApartMatrix& m);

// ---- text format (io.hpp) ----------------------------------------------------------

Dfa read_dfa(std::string_view text);
std::string write_dfa(const Dfa& dfa);
Dfa read_dfa_file(const std::string& path);
void write_dfa_file(const Dfa& dfa, const std::string& path);

// ---- minimisation (minimize.hpp) -------------------------------------------------------

enum class Algorithm { moore, trans, naive_pr, naive_pr_fused, sort_pr, trans_pr };
const char* to_string(Algorithm a);

struct ElectionPolicy {
    enum class Kind { min_index, arbitrary };
    Kind kind = Kind::min_index;
    std::uint64_t seed = 0;
    static ElectionPolicy min_index() { return {Kind::min_index, 0}; }
    static ElectionPolicy arbitrary(std::uint64_t seed) { return {Kind::arbitrary, seed}; }
};

struct RefinementReport {
    Partition partition;
    std::uint32_t refining_iterations = 0;
    Algorithm algorithm = Algorithm::moore;
    std::uint32_t closure_iterations = 0;
};

inline constexpr std::uint64_t kDefaultMaxPairNodes = 1ull << 16;
inline constexpr std::uint64_t kDefaultMaxTransitions = 1ull << 28;

RefinementReport moore_minimize(const Dfa& dfa);

struct TransResult {
    RefinementReport report;
    ApartMatrix apart;
};
TransResult trans_minimize(const Dfa& dfa, std::uint64_t max_pair_nodes = kDefaultMaxPairNodes);
RefinementReport naive_pr(const Dfa& dfa, const ElectionPolicy& policy = ElectionPolicy::min_index());
RefinementReport naive_pr_fused(const Dfa& dfa);
RefinementReport sort_pr(const Dfa& dfa);
Dfa build_transitive_alphabet(const Dfa& dfa, std::uint64_t max_transitions = kDefaultMaxTransitions);
RefinementReport trans_pr(const Dfa& dfa, const ElectionPolicy& policy = ElectionPolicy::min_index(),
                          std::uint64_t max_transitions = kDefaultMaxTransitions);

// ---- equivalence / inclusion (equivalence.hpp) -------------------------------------------

enum class Verdict { equivalent, included, counterexample };

struct ProductResult {
    Verdict verdict = Verdict::equivalent;
    std::vector<LetterId> counterexample;
    std::uint64_t explored_states = 0;
    std::uint32_t levels = 0;
};

enum class ExploreMode { equivalence, inclusion, full };
inline constexpr std::uint64_t kDefaultMaxVisited = 1ull << 26;

struct ExploreOptions {
    bool match_letters_by_name = false;
    std::uint64_t max_visited = kDefaultMaxVisited;
};

ProductResult explore_product(const Dfa& a, const Dfa& b, ExploreMode mode, const ExploreOptions& opts = {});
ProductResult check_equiv(const Dfa& a, const Dfa& b, const ExploreOptions& opts = {});
ProductResult check_inclusion(const Dfa& a, const Dfa& b, const ExploreOptions& opts = {});
/// Hopcroft-Karp with a GPU union-find (B200 extension; paper §6).
ProductResult check_equiv_union_find(const Dfa& a, const Dfa& b);

// ---- benchmark families (generators.hpp) ------------------------------------------------

inline constexpr std::uint64_t kDefaultStateBudget = 1ull << 26;

struct FibWord {
    std::uint32_t index = 0;
    std::vector<bool> bits;
};
FibWord fib_word(std::uint32_t m, std::uint64_t max_length = kDefaultStateBudget);
std::uint64_t cycle_fib(std::uint32_t n);
Dfa gen_fib(std::uint32_t m, std::uint64_t max_states = kDefaultStateBudget);
Dfa gen_bitsplitter(std::uint32_t n, std::uint64_t max_states = kDefaultStateBudget);
Dfa gen_bitsplitter_ext(std::uint32_t n, std::uint64_t max_states = kDefaultStateBudget);
Dfa gen_cycle(std::uint32_t n, std::uint64_t max_states = kDefaultStateBudget);
Dfa gen_memory_perfect(std::uint32_t n, std::uint64_t max_states = kDefaultStateBudget);
Dfa gen_memory_forgetful(std::uint32_t n, std::uint64_t max_states = kDefaultStateBudget);
Dfa gen_random_dfa(StateId n, LetterId k, double accept_fraction, std::uint64_t seed);

// ---- labelled transition systems (lts.hpp) --------------------------------------------------

struct Lts {
    StateId num_states = 0;
    StateId initial = 0;
    struct Transition {
        StateId from;
        std::string label;
        StateId to;
    };
    std::vector<Transition> transitions;
};

Lts load_aut(std::string_view text);

struct DeterminizeOptions {
    std::uint64_t max_states = 1ull << 22;
    double timeout_s = 600.0;
};
Lts determinize(const Lts& lts, const DeterminizeOptions& opts = {});
Dfa complete_to_dfa(const Lts& deterministic);

// ---- B200 extensions (no reference counterpart) ------------------------------------------
//
// Every calling thread runs on its own device context (its own stream and
// memory pool): concurrent callers proceed in parallel.  A thread's context
// is created on its first call -- on device DFAKIT_DEVICE when set, else
// round-robin over the visible devices -- and destroyed when the thread ends.
namespace b200 {

// Device the calling thread's context runs on (creates the context).
int current_device();

// Multi-GPU sortPR (one process per GPU, NCCL): rank 0 creates the id,
// shares its 128 bytes with every rank out of band, every rank constructs a
// ShardedComm on its own device and calls sort_pr_sharded with the same
// automaton; every rank receives the whole canonical partition.
using CommId = std::array<std::uint8_t, 128>;
CommId sharded_unique_id();

class ShardedComm {
public:
    ShardedComm(const CommId& id, int world, int rank, int device);
    ~ShardedComm();
    ShardedComm(const ShardedComm&) = delete;
    ShardedComm& operator=(const ShardedComm&) = delete;
    int world() const { return world_; }
    int rank() const { return rank_; }
    void* ctx() const { return ctx_; }
    void* comm() const { return comm_; }

private:
    int world_, rank_;
    void* ctx_ = nullptr;
    void* comm_ = nullptr;
};

RefinementReport sort_pr_sharded(const Dfa& dfa, ShardedComm& comm);

}  // namespace b200

}  // namespace dfakit
