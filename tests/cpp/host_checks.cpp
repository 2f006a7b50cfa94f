// host_checks.cpp -- CPU-only checks of the C++ drop-in layer (no GPU call):
// text format, validation, partitions, quotient / prune / canonical form,
// apartness, .aut loading and determinisation.  Mirrors the shape of the
// reference's tests/test_core.cpp and test_generators.cpp expectations.
// Prints "OK <n>" and exits 0, or prints the failing check and exits 1.
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>

#include "dfakit/dfa.hpp"
#include "dfakit/errors.hpp"
#include "dfakit/generators.hpp"
#include "dfakit/io.hpp"
#include "dfakit/lts.hpp"

using namespace dfakit;

static int checks = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        ++checks;                                                             \
        if (!(c)) {                                                           \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);          \
            std::exit(1);                                                     \
        }                                                                     \
    } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static Dfa shuffled(const Dfa& d, std::uint64_t seed) {
    std::vector<StateId> perm(d.num_states);
    for (StateId q = 0; q < d.num_states; ++q) perm[q] = q;
    std::mt19937_64 g(seed);
    for (StateId i = d.num_states; i > 1; --i) std::swap(perm[i - 1], perm[g() % i]);
    Dfa o = d;
    for (LetterId a = 0; a < d.alphabet_size; ++a)
        for (StateId q = 0; q < d.num_states; ++q) o.delta[a][perm[q]] = perm[d.delta[a][q]];
    for (StateId q = 0; q < d.num_states; ++q) o.accepting[perm[q]] = d.accepting[q];
    if (d.initial) o.initial = perm[*d.initial];
    return o;
}

int main() {
    // validation
    Dfa one;
    one.num_states = 1;
    one.alphabet_size = 1;
    one.delta = {{0}};
    one.accepting = {true};
    one.initial = 0;
    CHECK(validate(one).empty());
    Dfa bad = one;
    bad.num_states = 2;
    bad.delta = {{5, 1}};
    bad.accepting = {false, true};
    auto v = validate(bad);
    CHECK(v.size() == 1 && v[0].find("delta[0][0]") != std::string::npos);
    Dfa names = one;
    names.letter_names = std::vector<std::string>{"a", "b"};
    CHECK(validate(names).size() == 1 && validate(names)[0].find("letter_names") != std::string::npos);
    CHECK(validate(gen_bitsplitter(3)).empty() && validate(gen_cycle(6)).empty());

    // text format
    for (std::uint64_t s = 1; s <= 25; ++s) {
        Dfa d = gen_random_dfa(1 + (StateId)((s * 31) % 40), 1 + (LetterId)(s % 5), 0.1 * (s % 10), s);
        if (s % 3 == 0) d.initial.reset();
        if (s % 2 == 0) {
            std::vector<std::string> nm;
            for (LetterId a = 0; a < d.alphabet_size; ++a) nm.push_back("L" + std::to_string(a));
            d.letter_names = nm;
        }
        CHECK(read_dfa(write_dfa(d)) == d);
        CHECK(write_dfa(read_dfa(write_dfa(d))) == write_dfa(d));
    }
    CHECK(read_dfa(write_dfa(gen_bitsplitter(1))) == gen_bitsplitter(1));
    CHECK(read_dfa(write_dfa(gen_bitsplitter_ext(3))) == gen_bitsplitter_ext(3));
    CHECK(write_dfa(gen_bitsplitter(4)).find("initial -\n") != std::string::npos);
    Dfa spaced = one;
    spaced.num_states = 2;
    spaced.alphabet_size = 2;
    spaced.delta = {{1, 0}, {0, 0}};
    spaced.accepting = {false, true};
    spaced.letter_names = std::vector<std::string>{"hello, world", "b c"};
    CHECK(read_dfa(write_dfa(spaced)) == spaced);
    try {
        read_dfa("dfa 1\nstates 2\nalphabet 1\ninitial 0\naccepting 0\ntrans 0 0 1 1\n");
        CHECK(false);
    } catch (const ParseError& e) {
        CHECK(e.line() == 6);
    }
    CHECK(throws<ParseError>([] { read_dfa("dfa 2\nstates 1\n"); }));
    CHECK(throws<ParseError>([] { read_dfa("dfa 1\nstates 1\nalphabet 0\ninitial 0\naccepting 0\njunk\n"); }));
    CHECK(throws<ParseError>([] { read_dfa("dfa 1\nstates 1\nalphabet 1\ninitial 3\naccepting 0\ntrans 0 0\n"); }));
    CHECK(throws<ParseError>([] { read_dfa("dfa 1\nstates 3\nalphabet 0\ninitial -\naccepting 2 2 1\n"); }));

    // partitions, quotient, pruning, canonical forms
    CHECK(Partition::from_labels(std::vector<StateId>{7, 7, 3, 9, 3}).block_of == (std::vector<StateId>{0, 0, 1, 2, 1}));
    Dfa twins = one;
    twins.num_states = 2;
    twins.delta = {{0, 1}};
    twins.accepting = {true, true};
    Dfa q1 = quotient(twins, Partition::single_block(2));
    CHECK(q1.num_states == 1 && q1.accepting[0] && q1.delta[0][0] == 0);
    Dfa mixed = twins;
    mixed.accepting = {true, false};
    CHECK(throws<std::invalid_argument>([&] { quotient(mixed, Partition::single_block(2)); }));
    Dfa open3 = one;
    open3.num_states = 3;
    open3.delta = {{2, 1, 2}};
    open3.accepting = {false, false, true};
    CHECK(throws<std::invalid_argument>(
        [&] { quotient(open3, Partition::from_labels(std::vector<StateId>{0, 0, 1})); }));
    Dfa unreach = one;
    unreach.num_states = 3;
    unreach.delta = {{1, 0, 2}};
    unreach.accepting = {false, true, true};
    auto [pruned, map] = prune_unreachable(unreach);
    CHECK(pruned.num_states == 2 && map[2] == kNoState && map[0] == 0 && map[1] == 1);
    CHECK(throws<std::invalid_argument>([] { prune_unreachable(gen_bitsplitter(3)); }));
    Dfa r = prune_unreachable(gen_random_dfa(30, 2, 0.5, 8)).first;
    for (std::uint64_t s = 0; s < 5; ++s) CHECK(canonical_form(shuffled(r, s)) == canonical_form(r));
    CHECK(canonical_form(canonical_form(r)) == canonical_form(r));
    Dfa idq = quotient(gen_random_dfa(9, 2, 0.4, 11), Partition::identity(9));
    CHECK(write_dfa(canonical_form(prune_unreachable(idq).first)) ==
          write_dfa(canonical_form(prune_unreachable(gen_random_dfa(9, 2, 0.4, 11)).first)));

    // apartness
    CHECK(partition_from_apart(ApartMatrix(4)).num_blocks == 1);
    ApartMatrix all(3);
    for (StateId a = 0; a < 3; ++a)
        for (StateId b = a + 1; b < 3; ++b) all.set_apart(a, b);
    CHECK(partition_from_apart(all) == Partition::identity(3));
    ApartMatrix nt(3);
    nt.set_apart(0, 2);
    CHECK(throws<std::invalid_argument>([&] { partition_from_apart(nt); }));
    CHECK(throws<std::invalid_argument>([] { ApartMatrix m(2); m.set_apart(1, 1); }));

    // generators: parameter guards and budgets
    CHECK(throws<ResourceError>([] { gen_bitsplitter(20, 1000); }));
    CHECK(throws<ResourceError>([] { gen_cycle(40, 1000); }));
    CHECK(throws<ResourceError>([] { gen_memory_perfect(20, 1000); }));
    CHECK(throws<ResourceError>([] { fib_word(40, 1000); }));
    CHECK(throws<std::invalid_argument>([] { gen_cycle(1); }));
    CHECK(throws<std::invalid_argument>([] { gen_bitsplitter(0); }));
    CHECK(throws<std::invalid_argument>([] { gen_random_dfa(5, 2, 1.5, 1); }));
    CHECK(throws<std::invalid_argument>([] { gen_fib(1); }));
    CHECK(throws<std::invalid_argument>([] { gen_memory_forgetful(1); }));

    // .aut pipeline
    Lts l = load_aut("des (0, 1, 2)\n(0, \"a\", 1)\n");
    CHECK(l.num_states == 2 && l.transitions.size() == 1 && l.transitions[0].label == "a");
    Lts l2 = load_aut("des (0, 4, 3)\n(0, a, 1)\n(0, a, 1)\n(1, \"hello, world\", 2)\n(2, \"b c\", 0)\n");
    CHECK(l2.transitions.size() == 4 && l2.transitions[2].label == "hello, world" && l2.transitions[3].label == "b c");
    try {
        load_aut("des (0, 2, 2)\n(0, a, 1)\n");
        CHECK(false);
    } catch (const ParseError& e) {
        CHECK(e.line() == 3 && std::string(e.what()).find("mismatch") != std::string::npos);
    }
    CHECK(throws<ParseError>([] { load_aut("hello\n"); }));
    CHECK(throws<ParseError>([] { load_aut("des (5, 0, 2)\n"); }));
    CHECK(throws<ParseError>([] { load_aut("des (0, 1, 2)\n(0, a, 7)\n"); }));
    Lts nd;
    nd.num_states = 2;
    nd.transitions = {{0, "a", 0}, {0, "a", 1}};
    Lts det = determinize(nd);
    CHECK(det.num_states == 2 && complete_to_dfa(det).num_states == 3);
    Lts big;
    big.num_states = 12;
    for (StateId q = 0; q < 12; ++q) {
        big.transitions.push_back({q, "a", (q + 1) % 12});
        big.transitions.push_back({q, "a", (q * 5 + 3) % 12});
    }
    DeterminizeOptions o;
    o.max_states = 2;
    CHECK(throws<ResourceError>([&] { determinize(big, o); }));
    Lts empty;
    empty.num_states = 1;
    Dfa tiny = complete_to_dfa(empty);
    CHECK(tiny.num_states == 2 && tiny.accepting[0] && !tiny.accepting[1] && tiny.alphabet_size == 0);

    std::printf("OK %d\n", checks);
    return 0;
}
