// gpu_checks.cpp -- the C++ drop-in API on the GPU: concurrent callers (every
// thread gets its own device context, so calls run in parallel) and the
// dfakit::b200 extensions (per-thread device, multi-GPU sortPR at world size
// 1 over NCCL).  Prints "OK <n>" and exits 0, or the failing check and 1.
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include "dfakit/dfa.hpp"
#include "dfakit/equivalence.hpp"
#include "dfakit/generators.hpp"
#include "dfakit/minimize.hpp"
#include "dfakit_b200.hpp"

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

int main() {
    // reference results, one thread
    constexpr int kThreadsN = 8;
    std::vector<Dfa> in;
    std::vector<RefinementReport> want_sort, want_naive;
    std::vector<ProductResult> want_eq;
    for (int i = 0; i < kThreadsN; ++i) {
        in.push_back(gen_random_dfa(20000 + 977 * i, 3, 0.5, 100 + i));
        want_sort.push_back(sort_pr(in.back()));
        want_naive.push_back(naive_pr(in.back(), ElectionPolicy::arbitrary(i)));
        want_eq.push_back(check_equiv(in.back(), in.back()));
    }
    // the same calls from kThreadsN threads at once, several rounds each
    std::vector<int> ok(kThreadsN, 0), dev(kThreadsN, -1);
    std::vector<std::thread> ts;
    for (int i = 0; i < kThreadsN; ++i)
        ts.emplace_back([&, i] {
            bool good = true;
            for (int r = 0; r < 4; ++r) {
                const RefinementReport s = sort_pr(in[i]);
                const RefinementReport nv = naive_pr(in[i], ElectionPolicy::arbitrary(i));
                const ProductResult e = check_equiv(in[i], in[i]);
                good = good && s.partition == want_sort[i].partition &&
                       s.refining_iterations == want_sort[i].refining_iterations &&
                       nv.partition == want_naive[i].partition &&
                       nv.refining_iterations == want_naive[i].refining_iterations &&
                       e.verdict == want_eq[i].verdict && e.explored_states == want_eq[i].explored_states;
            }
            dev[i] = b200::current_device();
            ok[i] = good;
        });
    for (auto& t : ts) t.join();
    for (int i = 0; i < kThreadsN; ++i) {
        CHECK(ok[i]);
        CHECK(dev[i] >= 0);
    }
    // multi-GPU sortPR through the C++ extension at world size 1
    {
        const b200::CommId id = b200::sharded_unique_id();
        b200::ShardedComm comm(id, 1, 0, b200::current_device());
        CHECK(comm.world() == 1 && comm.rank() == 0);
        for (int i = 0; i < 3; ++i) {
            const RefinementReport r = b200::sort_pr_sharded(in[i], comm);
            CHECK(r.partition == want_sort[i].partition);
            CHECK(r.refining_iterations == want_sort[i].refining_iterations);
        }
    }
    std::printf("OK %d\n", checks);
    return 0;
}
