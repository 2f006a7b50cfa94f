// dfakit_cli.cpp -- the `dfakit` command line (reference tools/dfakit_cli.cpp
// interface: subcommands generate / minimize / equiv / include / convert /
// bench, the same flags, CSV header and exit codes 0 ok, 1 counterexample,
// 2 operational error).  Minimisation and equivalence run on the GPU
// through libdfakit_b200.
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <sstream>
#include <thread>

#include "dfakit_b200.hpp"

using namespace dfakit;

namespace {

const char* const kHeader = "name,n,k,algo,output_size,refine_iters,closure_iters,mean_ms,status";

struct Args {
    std::vector<std::string> pos;
    std::multimap<std::string, std::string> opt;
    std::vector<std::string> flags;
    bool has(const std::string& f) const {
        for (auto& x : flags)
            if (x == f) return true;
        return false;
    }
    std::optional<std::string> get(const std::string& k) const {
        auto it = opt.find(k);
        if (it == opt.end()) return std::nullopt;
        return it->second;
    }
    std::vector<std::string> all(const std::string& k) const {
        std::vector<std::string> v;
        auto r = opt.equal_range(k);
        for (auto it = r.first; it != r.second; ++it) v.push_back(it->second);
        return v;
    }
};

// options that take a value; everything else starting with '-' is a flag
const char* const kValued[] = {"--word-index", "--n", "--k", "--accept-fraction", "--seed", "-o", "--out", "--algo",
                               "--policy", "--runs", "--timeout-s", "--mem-budget-mb", "--emit", "--name",
                               "--max-subset-states", "--suite", "--algos"};

Args parse(int argc, char** argv, int first) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string s = argv[i];
        bool valued = false;
        for (const char* v : kValued)
            if (s == v) valued = true;
        if (valued) {
            if (i + 1 >= argc) throw std::invalid_argument("option " + s + " needs a value");
            a.opt.emplace(s == "--out" ? "-o" : s, argv[++i]);
        } else if (s.size() > 1 && s[0] == '-') {
            a.flags.push_back(s);
        } else {
            a.pos.push_back(s);
        }
    }
    return a;
}

std::uint64_t to_u64(const std::string& s, const char* what) {
    std::size_t used = 0;
    unsigned long long v = std::stoull(s, &used);
    if (used != s.size()) throw std::invalid_argument(std::string("bad ") + what + " '" + s + "'");
    return v;
}

struct Budget {
    std::optional<double> mb;
    std::uint64_t visited() const {
        return mb ? std::max<std::uint64_t>(1, (std::uint64_t)(*mb * (1 << 20) / 24.0)) : kDefaultMaxVisited;
    }
    std::uint64_t pair_nodes() const {
        return mb ? std::max<std::uint64_t>(1, (std::uint64_t)std::sqrt(*mb * (1 << 20) * 8.0 / 2.0))
                  : kDefaultMaxPairNodes;
    }
    std::uint64_t transitions() const {
        return mb ? std::max<std::uint64_t>(1, (std::uint64_t)(*mb * (1 << 20) / 4.0)) : kDefaultMaxTransitions;
    }
};

Algorithm algo_of(const std::string& s) {
    static const std::map<std::string, Algorithm> m = {{"moore", Algorithm::moore}, {"trans", Algorithm::trans},
                                                       {"naive", Algorithm::naive_pr},
                                                       {"naive-fused", Algorithm::naive_pr_fused},
                                                       {"sort", Algorithm::sort_pr}, {"transpr", Algorithm::trans_pr}};
    auto it = m.find(s);
    if (it == m.end()) throw std::invalid_argument("unknown algorithm '" + s + "'");
    return it->second;
}

Dfa family(const std::string& fam, std::optional<std::uint32_t> word_index, std::optional<std::uint32_t> n,
           std::uint32_t k, double frac, std::uint64_t seed) {
    auto need = [&]() {
        if (!n) throw std::invalid_argument("family '" + fam + "' needs --n");
        return *n;
    };
    if (fam == "fib") {
        if (!word_index) throw std::invalid_argument("family 'fib' needs --word-index");
        return gen_fib(*word_index);
    }
    if (fam == "bitsplit") return gen_bitsplitter(need());
    if (fam == "bitsplit-ext") return gen_bitsplitter_ext(need());
    if (fam == "cycle") return gen_cycle(need());
    if (fam == "memory-perfect") return gen_memory_perfect(need());
    if (fam == "memory-forgetful") return gen_memory_forgetful(need());
    if (fam == "random") return gen_random_dfa(need(), k, frac, seed);
    throw std::invalid_argument("unknown family '" + fam + "'");
}

RefinementReport run_algo(const Dfa& d, Algorithm a, const ElectionPolicy& pol, const Budget& b) {
    switch (a) {
        case Algorithm::moore: return moore_minimize(d);
        case Algorithm::trans: return trans_minimize(d, b.pair_nodes()).report;
        case Algorithm::naive_pr: return naive_pr(d, pol);
        case Algorithm::naive_pr_fused: return naive_pr_fused(d);
        case Algorithm::sort_pr: return sort_pr(d);
        case Algorithm::trans_pr: return trans_pr(d, pol, b.transitions());
    }
    throw std::logic_error("unreachable");
}

struct Row {
    std::string name;
    StateId n = 0;
    LetterId k = 0;
    Algorithm algo = Algorithm::moore;
    std::optional<RefinementReport> rep;
    double mean_ms = 0;
    std::string status = "ok";
};

void print_row(std::ostream& o, const Row& r) {
    o << r.name << ',' << r.n << ',' << r.k << ',' << to_string(r.algo) << ',';
    if (r.status == "ok") {
        char ms[32];
        std::snprintf(ms, sizeof ms, "%.3f", r.mean_ms);
        o << r.rep->partition.num_blocks << ',' << r.rep->refining_iterations << ',' << r.rep->closure_iterations
          << ',' << ms;
    } else {
        o << ",,,";
    }
    o << ',' << r.status << '\n';
}

// R timed repetitions in a worker; a run exceeding the per-run budget marks
// the row "timeout" and the worker is left to finish on its own.
Row measure(const std::string& name, std::shared_ptr<const Dfa> d, Algorithm a, const ElectionPolicy& pol,
            std::uint32_t runs, double timeout_s, const Budget& b) {
    struct State {
        std::mutex mu;
        std::condition_variable cv;
        std::vector<double> ms;
        std::optional<RefinementReport> rep;
        std::string error;
        bool oom = false, failed = false, done = false;
    };
    auto st = std::make_shared<State>();
    Row row;
    row.name = name;
    row.n = d->num_states;
    row.k = d->alphabet_size;
    row.algo = a;
    std::thread w([st, d, a, pol, runs, b] {
        try {
            for (std::uint32_t i = 0; i < runs; ++i) {
                auto t0 = std::chrono::steady_clock::now();
                RefinementReport r = run_algo(*d, a, pol, b);
                auto t1 = std::chrono::steady_clock::now();
                std::lock_guard<std::mutex> lk(st->mu);
                st->ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
                st->rep = std::move(r);
                st->cv.notify_all();
            }
        } catch (const ResourceError& e) {
            std::lock_guard<std::mutex> lk(st->mu);
            st->oom = true;
            st->error = e.what();
        } catch (const std::exception& e) {
            std::lock_guard<std::mutex> lk(st->mu);
            st->failed = true;
            st->error = e.what();
        }
        std::lock_guard<std::mutex> lk(st->mu);
        st->done = true;
        st->cv.notify_all();
    });
    std::unique_lock<std::mutex> lk(st->mu);
    for (std::uint32_t i = 0; i < runs; ++i) {
        const auto until = std::chrono::steady_clock::now() +
                           std::chrono::duration_cast<std::chrono::steady_clock::duration>(
                               std::chrono::duration<double>(timeout_s));
        if (!st->cv.wait_until(lk, until, [&] { return st->ms.size() > i || st->done; })) {
            row.status = "timeout";
            lk.unlock();
            w.detach();
            return row;
        }
        if (st->done && st->ms.size() <= i) break;
    }
    lk.unlock();
    w.join();
    if (st->failed) throw std::runtime_error(st->error);
    if (st->oom) {
        row.status = "out-of-memory";
        std::cerr << name << ": " << st->error << "\n";
        return row;
    }
    double sum = 0;
    for (double x : st->ms) sum += x;
    row.mean_ms = sum / (double)st->ms.size();
    row.rep = std::move(st->rep);
    return row;
}

std::string slurp(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open " + path);
    std::ostringstream ss;
    ss << f.rdbuf();
    return ss.str();
}

int verdict_out(const Dfa& a, const ProductResult& r, bool stats, const char* ok) {
    if (r.verdict == Verdict::counterexample) {
        std::cout << "counterexample";
        for (LetterId l : r.counterexample)
            std::cout << ' ' << (a.letter_names ? (*a.letter_names)[l] : std::to_string(l));
        std::cout << '\n';
    } else {
        std::cout << ok << '\n';
    }
    if (stats) std::cout << "explored_states=" << r.explored_states << " levels=" << r.levels << '\n';
    return r.verdict == Verdict::counterexample ? 1 : 0;
}

int usage() {
    std::cerr << "usage: dfakit <generate|minimize|equiv|include|convert|bench> ...\n";
    return 2;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    try {
        Args a = parse(argc, argv, 2);
        Budget budget;
        if (const char* env = std::getenv("DFAKIT_MEM_BUDGET_MB")) budget.mb = std::atof(env);
        if (auto m = a.get("--mem-budget-mb")) budget.mb = std::stod(*m);

        if (cmd == "generate") {
            if (a.pos.empty()) throw std::invalid_argument("generate needs a family");
            std::optional<std::uint32_t> wi, n;
            if (auto v = a.get("--word-index")) wi = (std::uint32_t)to_u64(*v, "word index");
            if (auto v = a.get("--n")) n = (std::uint32_t)to_u64(*v, "n");
            const std::uint32_t k = a.get("--k") ? (std::uint32_t)to_u64(*a.get("--k"), "k") : 2;
            const double frac = a.get("--accept-fraction") ? std::stod(*a.get("--accept-fraction")) : 0.5;
            const std::uint64_t seed = a.get("--seed") ? to_u64(*a.get("--seed"), "seed") : 0;
            Dfa d = family(a.pos[0], wi, n, k, frac, seed);
            if (auto out = a.get("-o")) {
                write_dfa_file(d, *out);
                std::cerr << "wrote " << *out << " (" << d.num_states << " states, " << d.alphabet_size
                          << " letters)\n";
            } else {
                std::cout << write_dfa(d);
            }
            return 0;
        }
        if (cmd == "minimize") {
            if (a.pos.empty()) throw std::invalid_argument("minimize needs an input file");
            auto d = std::make_shared<const Dfa>(read_dfa_file(a.pos[0]));
            const std::string pol_s = a.get("--policy").value_or("min-index");
            ElectionPolicy pol = ElectionPolicy::min_index();
            if (pol_s == "arbitrary") pol = ElectionPolicy::arbitrary(a.get("--seed") ? to_u64(*a.get("--seed"), "seed") : 0);
            else if (pol_s != "min-index") throw std::invalid_argument("unknown policy '" + pol_s + "'");
            const std::string name = a.get("--name").value_or(std::filesystem::path(a.pos[0]).stem().string());
            const std::uint32_t runs = a.get("--runs") ? (std::uint32_t)to_u64(*a.get("--runs"), "runs") : 5;
            const double timeout = a.get("--timeout-s") ? std::stod(*a.get("--timeout-s")) : 300.0;
            Row row = measure(name, d, algo_of(a.get("--algo").value_or("naive")), pol, runs, timeout, budget);
            std::cout << kHeader << '\n';
            print_row(std::cout, row);
            if (auto emit = a.get("--emit"); emit && row.status == "ok") {
                const Partition& p = row.rep->partition;
                if (d->initial) {
                    auto [pruned, map] = prune_unreachable(*d);
                    std::vector<StateId> lab(pruned.num_states);
                    for (StateId q = 0; q < d->num_states; ++q)
                        if (map[q] != kNoState) lab[map[q]] = p.block_of[q];
                    write_dfa_file(quotient(pruned, Partition::from_labels(lab)), *emit);
                } else {
                    std::ofstream f(*emit);
                    if (!f) throw std::runtime_error("cannot open " + *emit);
                    std::vector<std::vector<StateId>> members(p.num_blocks);
                    for (StateId q = 0; q < d->num_states; ++q) members[p.block_of[q]].push_back(q);
                    f << "partition " << p.num_blocks << '\n';
                    for (StateId b = 0; b < p.num_blocks; ++b) {
                        f << "block " << b << ':';
                        for (StateId q : members[b]) f << ' ' << q;
                        f << '\n';
                    }
                }
            }
            return 0;
        }
        if (cmd == "equiv" || cmd == "include") {
            if (a.pos.size() < 2) throw std::invalid_argument(cmd + " needs two DFA files");
            Dfa x = read_dfa_file(a.pos[0]), y = read_dfa_file(a.pos[1]);
            ExploreOptions o;
            o.match_letters_by_name = a.has("--by-name");
            o.max_visited = budget.visited();
            if (cmd == "equiv") return verdict_out(x, check_equiv(x, y, o), a.has("--stats"), "equivalent");
            return verdict_out(x, check_inclusion(x, y, o), a.has("--stats"), "included");
        }
        if (cmd == "convert") {
            if (a.pos.size() < 2) throw std::invalid_argument("convert needs input and output paths");
            DeterminizeOptions o;
            if (auto v = a.get("--timeout-s")) o.timeout_s = std::stod(*v);
            if (auto v = a.get("--max-subset-states")) o.max_states = to_u64(*v, "max subset states");
            Dfa d = complete_to_dfa(determinize(load_aut(slurp(a.pos[0])), o));
            write_dfa_file(d, a.pos[1]);
            std::cout << "states=" << d.num_states << " alphabet=" << d.alphabet_size << '\n';
            return 0;
        }
        if (cmd == "bench") {
            auto suites = a.all("--suite");
            if (suites.empty()) throw std::invalid_argument("bench needs --suite family=lo..hi");
            std::vector<Algorithm> algos;
            std::stringstream ss(a.get("--algos").value_or("naive,sort,transpr"));
            for (std::string t; std::getline(ss, t, ',');)
                if (!t.empty()) algos.push_back(algo_of(t));
            if (algos.empty()) throw std::invalid_argument("--algos parsed to an empty list");
            const std::uint32_t runs = a.get("--runs") ? (std::uint32_t)to_u64(*a.get("--runs"), "runs") : 5;
            const double timeout = a.get("--timeout-s") ? std::stod(*a.get("--timeout-s")) : 300.0;
            const std::uint32_t k = a.get("--k") ? (std::uint32_t)to_u64(*a.get("--k"), "k") : 2;
            std::ofstream file;
            if (auto out = a.get("-o")) {
                file.open(*out);
                if (!file) throw std::runtime_error("cannot open " + *out);
            }
            std::ostream& o = file.is_open() ? file : std::cout;
            o << kHeader << '\n';
            for (const auto& spec : suites) {
                const auto eq = spec.find('='), dots = spec.find("..");
                if (eq == std::string::npos || dots == std::string::npos || dots < eq)
                    throw std::invalid_argument("suite spec must look like family=lo..hi, got '" + spec + "'");
                const std::string fam = spec.substr(0, eq);
                const std::uint32_t lo = (std::uint32_t)to_u64(spec.substr(eq + 1, dots - eq - 1), "suite bound");
                const std::uint32_t hi = (std::uint32_t)to_u64(spec.substr(dots + 2), "suite bound");
                if (hi < lo) throw std::invalid_argument("suite range is empty: '" + spec + "'");
                for (std::uint32_t p = lo; p <= hi; ++p) {
                    const std::string name = fam + "_" + std::to_string(p);
                    std::shared_ptr<const Dfa> d;
                    try {
                        if (fam == "fib") d = std::make_shared<const Dfa>(gen_fib(p));
                        else if (fam == "random") d = std::make_shared<const Dfa>(gen_random_dfa(p, k, 0.5, p));
                        else d = std::make_shared<const Dfa>(family(fam, std::nullopt, p, k, 0.5, p));
                    } catch (const ResourceError& e) {
                        std::cerr << name << ": " << e.what() << '\n';
                        for (Algorithm al : algos) {
                            Row r;
                            r.name = name;
                            r.algo = al;
                            r.status = "out-of-memory";
                            print_row(o, r);
                        }
                        continue;
                    }
                    for (Algorithm al : algos) {
                        print_row(o, measure(name, d, al, ElectionPolicy::min_index(), runs, timeout, budget));
                        o.flush();
                    }
                }
            }
            return 0;
        }
        return usage();
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    }
}
