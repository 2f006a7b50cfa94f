"""GPU parity of the minimisers against the oracle and the reference's golden
vectors.  Bar: bit-exact partitions (canonical numbering) and identical
refining / closure pass counts -- for ElectionPolicy.arbitrary(seed) too:
the GPU draws the winners from the reference's own mt19937_64 stream
(refine_arbitrary.cu), so its pass counts are the reference's."""
import random

import numpy as np
import pytest

from conftest import digest, mkdfa

pytestmark = pytest.mark.gpu

ALGOS = {"moore": "moore_minimize", "sort": "sort_pr", "naive": "naive_pr", "naive-fused": "naive_pr_fused",
         "transpr": "trans_pr"}


def run(dk, algo, dfa, policy=None):
    if algo == "naive":
        return dk.naive_pr(dfa, policy or dk.ElectionPolicy.min_index())
    if algo == "transpr":
        return dk.trans_pr(dfa, policy or dk.ElectionPolicy.min_index())
    if algo == "trans":
        return dk.trans_minimize(dfa).report
    return getattr(dk, ALGOS[algo])(dfa)


def same(rep, want):
    return (np.array_equal(rep.partition.block_of, want.blocks) and rep.partition.num_blocks == want.num_blocks
            and rep.refining_iterations == want.refine_iters and rep.closure_iterations == want.closure_iters)


def test_random_sweep_all_minimisers(dk, oracle):
    """Acceptance criterion 1 shape: random DFAs n<=200, k<=4, every minimiser."""
    g = random.Random(1000)
    for i in range(250):
        n, k, frac, s = g.randint(1, 200), g.randint(1, 4), g.randint(0, 10) / 10, g.getrandbits(64)
        t = oracle.gen_random(n, k, frac, s)
        dfa = mkdfa(dk, t)
        for algo in ("moore", "sort", "naive", "naive-fused", "transpr") + (("trans",) if n <= 30 else ()):
            want = oracle.minimize(algo, t[0], t[1])
            got = run(dk, algo, dfa)
            assert same(got, want), (i, algo, n, k, frac, s, got.refining_iterations, want.refine_iters)
        staged = dk.sort_pr(dfa, grouping="staged")
        assert same(staged, oracle.minimize("sort", t[0], t[1])), (i, "staged")
        # arbitrary(seed): the reference's mt19937_64 winner stream, so the
        # pass counts match too (not only the winner-independent partition)
        for seed in (1, 2, 3):
            got = dk.naive_pr(dfa, dk.ElectionPolicy.arbitrary(seed))
            assert same(got, oracle.minimize("naive", t[0], t[1], policy=1, seed=seed)), (i, "arbitrary", seed)
        got = dk.trans_pr(dfa, dk.ElectionPolicy.arbitrary(5))
        assert same(got, oracle.minimize("transpr", t[0], t[1], policy=1, seed=5)), (i, "transpr arbitrary")


def test_golden_minimise_vectors(dk, oracle, golden):
    for e in golden["minimize"]:
        t = (oracle.gen_random(e["n"], e["k"], e["frac"], e["seed"]) if e["kind"] == "random"
             else oracle.gen_family(e["family"], e["param"]))
        dfa = mkdfa(dk, t)
        n = t[0].shape[1]
        for key, want in e["results"].items():
            algo, _, pol = key.partition("@arbitrary")
            if pol:
                rep = run(dk, algo, dfa, dk.ElectionPolicy.arbitrary(int(pol)))
            else:
                rep = run(dk, algo, dfa)
            blocks = [int(x) for x in rep.partition.block_of] if n <= 64 else digest(rep.partition.block_of)
            assert blocks == want["blocks"], (e, key)
            assert rep.partition.num_blocks == want["num_blocks"]
            assert (rep.refining_iterations, rep.closure_iterations) == \
                (want["refine_iters"], want["closure_iters"]), (e, key)


def test_bitsplitter_and_fibonacci_pass_counts(dk, oracle, golden):
    """Acceptance criteria 2 and 3 (the reference's own observed values)."""
    for n, want in golden["acceptance"]["bitsplit"].items():
        dfa = mkdfa(dk, oracle.gen_family("bitsplit", int(n)))
        for algo, iters in want.items():
            rep = run(dk, algo, dfa)
            assert rep.partition.num_blocks == 1 << int(n)
            assert rep.refining_iterations == iters, (n, algo)
    dfa = mkdfa(dk, oracle.gen_family("fib", 19))
    for algo, iters in golden["acceptance"]["fib19"].items():
        rep = run(dk, algo, dfa)
        assert rep.partition.num_blocks == 6765 and rep.refining_iterations == iters, algo
    rep = dk.naive_pr_fused(dfa)
    assert rep.refining_iterations == golden["acceptance"]["fib19"]["naive"]


def test_trans_minimize_matches_oracle(dk, oracle, golden):
    for m, (nb, ri, ci) in golden["acceptance"]["trans_closure"].items():
        res = dk.trans_minimize(mkdfa(dk, oracle.gen_family("fib", int(m))))
        assert (res.report.partition.num_blocks, res.report.refining_iterations,
                res.report.closure_iterations) == (nb, ri, ci)
    g = random.Random(7)
    for _ in range(20):
        n, k, frac, s = g.randint(1, 25), g.randint(1, 3), g.randint(0, 10) / 10, g.getrandbits(64)
        t = oracle.gen_random(n, k, frac, s)
        res = dk.trans_minimize(mkdfa(dk, t))
        assert np.array_equal(res.apart, oracle.trans_apart(t[0], t[1]).astype(bool))
        assert same(res.report, oracle.minimize("trans", t[0], t[1]))


def test_trans_minimize_budget_message(dk, oracle):
    with pytest.raises(dk.ResourceError, match=r"7921.*MiB"):
        dk.trans_minimize(mkdfa(dk, oracle.gen_family("fib", 10)), 1000)


def test_transitive_alphabet(dk, oracle, golden):
    for e in golden["transitive"]:
        t = oracle.gen_random(e["n"], e["k"], e["frac"], e["seed"])
        out = dk.build_transitive_alphabet(mkdfa(dk, t))
        assert out.alphabet_size == e["k_out"] and digest(out.delta) == e["delta"]
    chain = mkdfa(dk, oracle.gen_chain(10))
    closed = dk.build_transitive_alphabet(chain)
    assert closed.alphabet_size == 4 and closed.letter_names[3] == "a^8"
    assert closed.delta[3][0] == 8 and closed.delta[3][1] == 9
    with pytest.raises(dk.ResourceError):
        dk.build_transitive_alphabet(mkdfa(dk, oracle.gen_family("fib", 10)), 100)
    with pytest.raises(dk.ResourceError):
        dk.trans_pr(mkdfa(dk, oracle.gen_family("fib", 10)), max_transitions=100)


def test_edge_cases(dk):
    one = dk.Dfa(np.zeros((1, 1), np.uint32), np.array([1], np.uint8), 0)
    empty_alpha = dk.Dfa(np.zeros((0, 2), np.uint32), np.array([0, 1], np.uint8), None)
    none_acc = dk.Dfa(np.array([[1, 2, 0]], np.uint32), np.zeros(3, np.uint8), 0)
    all_acc = dk.Dfa(np.array([[1, 2, 0]], np.uint32), np.ones(3, np.uint8), 0)
    cyc4 = dk.Dfa(np.array([[1, 2, 3, 0]], np.uint32), np.array([1, 1, 0, 0], np.uint8), None)
    for f in (dk.moore_minimize, dk.sort_pr, dk.naive_pr, dk.naive_pr_fused, dk.trans_pr):
        r = f(one)
        assert r.partition.num_blocks == 1 and r.refining_iterations == 0
        r = f(empty_alpha)
        assert list(r.partition.block_of) == [0, 1] and r.refining_iterations == 0
        for d in (none_acc, all_acc):
            r = f(d)
            assert r.partition.num_blocks == 1 and r.refining_iterations == 0
    r = dk.sort_pr(cyc4)
    assert r.partition.num_blocks == 4 and r.refining_iterations == 1
    bad = dk.Dfa(np.array([[5, 1]], np.uint32), np.array([0, 1], np.uint8), None)
    with pytest.raises(ValueError):
        dk.sort_pr(bad)


def test_sort_exact_paths_and_collision_recovery(dk, oracle):
    """Packed, dense-packed, fingerprint, chunked-exact and forced-collision
    paths all give the oracle's partition and pass count."""
    g = random.Random(31)
    collisions = 0
    for i in range(16):
        n, k, s = g.randint(500, 20000), g.randint(5, 12), g.getrandbits(64)
        frac = 0.5 if i % 2 else 0.97   # skewed acceptance keeps blocks large for longer
        t = oracle.gen_random(n, k, frac, s)
        want = oracle.minimize("moore", t[0], t[1])
        dfa = mkdfa(dk, t)
        for kw in ({}, {"force_exact": True}, {"fingerprint_bits": 6}, {"grouping": "radix_sort"},
                   {"grouping": "radix_sort", "fingerprint_bits": 6}, {"grouping": "staged"},
                   {"grouping": "staged", "fingerprint_bits": 6}):
            rep = dk.sort_pr(dfa, **kw)
            assert same(rep, want), kw
            collisions += rep.hash_collisions
    assert collisions > 0, "the 6-bit fingerprint hook never produced a collision"


def copies(t, c):
    """c language-equal copies of a DFA, copy j stepping into copy j+1:
    every equivalence class has c members spread over the state space."""
    delta, acc, _ = t
    k, n0 = delta.shape
    out = np.empty((k, n0 * c), np.uint32)
    for j in range(c):
        out[:, j * n0:(j + 1) * n0] = delta + ((j + 1) % c) * n0
    return out, np.tile(acc, c), 0


def test_grouping_strategies(dk, oracle):
    """Large equivalence classes push passes through the counting table, the
    radix-bucket shared-memory hashing, the overflow (global table) fallback
    and the radix-sort grouping; all must agree with the oracle."""
    for n0, c, k in ((2000, 50, 8), (40, 1500, 8), (20, 6000, 8), (3000, 3, 12)):
        base = oracle.gen_random(n0, k, 0.5, n0 * 7 + c)
        t = copies(base, c)
        want = oracle.minimize("moore", t[0], t[1])
        dfa = mkdfa(dk, t)
        for kw in ({}, {"fingerprint_bits": 6}, {"force_exact": True}, {"grouping": "radix_sort"},
                   {"grouping": "staged"}, {"grouping": "staged", "fingerprint_bits": 6}):
            assert same(dk.sort_pr(dfa, **kw), want), (n0, c, k, kw)
        for algo in ("naive", "naive-fused"):
            assert same(run(dk, algo, dfa), oracle.minimize(algo, t[0], t[1])), (n0, c, algo)


@pytest.mark.slow
def test_config0_random_1M_k2(dk, oracle):
    """BASELINE configs[0]: random complete DFA, 1M states, |Sigma|=2."""
    t = oracle.gen_random(1_000_000, 2, 0.5, 7)
    want = oracle.minimize("moore", t[0], t[1])
    dfa = mkdfa(dk, t)
    rep = dk.sort_pr(dfa)
    assert same(rep, want)
    # the literal radix-sort grouping over ~330 sort tiles per digit (look-back chains)
    assert same(dk.sort_pr(dfa, grouping="radix_sort"), want)


@pytest.mark.slow
def test_config1_synth_10M_k10(dk, oracle):
    """BASELINE configs[1] size: 10M states x 10 letters = 100M transitions."""
    t = oracle.gen_synth(10_000_000, 10, 1)
    want = oracle.minimize("moore", t[0], t[1])
    dfa = mkdfa(dk, t)
    rep = dk.sort_pr(dfa)
    assert same(rep, want)
    # the partition is a congruence: successors of block-mates are block-mates
    blk = rep.partition.block_of
    first = np.full(rep.partition.num_blocks, -1, np.int64)
    order = np.arange(blk.size)
    first[blk[::-1]] = order[::-1]
    rep_of = first[blk]
    for a in range(t[0].shape[0]):
        assert np.array_equal(blk[t[0][a]], blk[t[0][a][rep_of]])


@pytest.mark.slow
def test_config2_chain_with_closure(dk, oracle):
    """BASELINE configs[2]: chain DFA with partial transitive closure, up to
    the 10M-state chain the bench times."""
    for n in (1000, 100_000, 10_000_000):
        t = oracle.gen_chain(n)
        want = oracle.minimize("transpr", t[0], t[1])
        rep = dk.trans_pr(mkdfa(dk, t))
        assert same(rep, want)
        assert rep.partition.num_blocks == n


def test_streamed_host_input(dk, oracle):
    """Host-buffer calls from 2^20 states stream delta in chunks and run pass 1
    as they land: same partition and pass count, and an out-of-range target in
    the last chunk is still rejected."""
    t = oracle.gen_random(1_500_000, 3, 0.5, 21)
    want = oracle.minimize("moore", t[0], t[1])
    for f in (dk.sort_pr, dk.moore_minimize):
        assert same(f(mkdfa(dk, t)), want), f
    bad = t[0].copy()
    bad[2][-1] = 1_500_000
    with pytest.raises(ValueError, match="out of range"):
        dk.sort_pr(dk.Dfa(bad, t[1], 0))


def test_streamed_host_input_sliced(dk, oracle, monkeypatch):
    """The streamed host-buffer path with every wide pass sliced (the
    1B-transition e2e shape, forced at 1.5M states)."""
    monkeypatch.setenv("DFAKIT_TEST_SLICE_BYTES", "200000")
    t = oracle.gen_synth(1_500_000, 10, 4)
    want = oracle.minimize("moore", t[0], t[1])
    assert same(dk.sort_pr(mkdfa(dk, t)), want)
    t = copies(oracle.gen_random(3000, 6, 0.5, 9), 400)
    assert same(dk.sort_pr(mkdfa(dk, t)), oracle.minimize("moore", t[0], t[1]))


def test_naive_kernel_paths(dk, oracle):
    """Leader election through each of its kernels: single CTA with delta in
    shared memory (n * k small), single CTA with delta from L1 (shared arrays
    fit, delta does not), and the persistent grid kernels (n * k > 2^16) --
    pass counts exact for min_index and arbitrary(seed)."""
    cases = [(900, 3, 0.5, 11),     # one CTA, delta in shared memory
             (4000, 12, 0.3, 12),   # one CTA, delta from global / L1
             (3000, 30, 0.5, 13),   # persistent grid kernels
             (2500, 40, 0.2, 14)]
    for n, k, frac, seed in cases:
        t = oracle.gen_random(n, k, frac, seed)
        dfa = mkdfa(dk, t)
        for algo in ("naive", "naive-fused"):
            want = oracle.minimize(algo, t[0], t[1])
            got = run(dk, algo, dfa)
            assert same(got, want), (n, k, algo, got.refining_iterations, want.refine_iters)
        got = dk.naive_pr(dfa, dk.ElectionPolicy.arbitrary(7))
        assert same(got, oracle.minimize("naive", t[0], t[1], policy=1, seed=7)), (n, k)


def test_first_pass_class_edge_cases_large(dk, oracle):
    """Large automata (past the small-m engine) whose first pass runs over
    every state before the class sizes are read: a singleton accepting class,
    a singleton rejecting class, all accepting, none accepting -- partition
    and pass counts exact against the oracle."""
    n, k = 300_000, 3
    delta, acc, _ = oracle.gen_random(n, k, 0.5, 77)
    for name in ("one_acc", "one_rej", "all_acc", "no_acc"):
        a = np.zeros(n, dtype=np.uint8)
        if name == "one_acc":
            a[12345] = 1
        elif name == "one_rej":
            a[:] = 1
            a[0] = 0
        elif name == "all_acc":
            a[:] = 1
        want = oracle.minimize("sort", delta, a)
        got = dk.sort_pr(dk.Dfa(delta, a, 0))
        assert same(got, want), (name, got.refining_iterations, want.refine_iters, got.partition.num_blocks,
                                 want.num_blocks)
    a = acc.copy()  # a nonzero flag other than 1 still means accepting
    a[a != 0] = 7
    want = oracle.minimize("sort", delta, acc)
    assert same(dk.sort_pr(dk.Dfa(delta, a, 0)), want)


def test_naive_persistent_grid_stride(dk, oracle):
    """More states than resident threads (every CTA loops over several
    states per pass): 2000 relabelled copies of a 200-state DFA, 400K states,
    through the persistent naive / fused kernels -- pass counts and
    partitions exact."""
    base = oracle.gen_random(200, 4, 0.5, 4242)
    t = copies(base, 2000)
    dfa = mkdfa(dk, t)
    for algo in ("naive", "naive-fused"):
        want = oracle.minimize(algo, t[0], t[1])
        got = run(dk, algo, dfa)
        assert same(got, want), (algo, got.refining_iterations, want.refine_iters)


def test_arbitrary_replay_path(dk, oracle, monkeypatch):
    """ElectionPolicy.arbitrary(seed): a draw libstdc++'s Lemire downscaling
    would reject (probability < c / 2^64) makes the pass replay sequentially
    from the pre-pass engine state.  The test hook sends EVERY pass through
    that replay kernel; winners, pass counts and partitions must still be
    the reference's."""
    monkeypatch.setenv("DFAKIT_TEST_ARB_REPLAY", "1")
    g = random.Random(4242)
    for i in range(12):
        n, k, frac, s = g.randint(2, 400), g.randint(1, 4), g.randint(1, 9) / 10, g.getrandbits(64)
        t = oracle.gen_random(n, k, frac, s)
        dfa = mkdfa(dk, t)
        for seed in (0, 9):
            got = dk.naive_pr(dfa, dk.ElectionPolicy.arbitrary(seed))
            assert same(got, oracle.minimize("naive", t[0], t[1], policy=1, seed=seed)), (i, seed)
    # a larger case with many writers per slot (copies: big classes)
    base = oracle.gen_random(300, 3, 0.5, 5)
    t = copies(base, 40)
    got = dk.naive_pr(mkdfa(dk, t), dk.ElectionPolicy.arbitrary(3))
    assert same(got, oracle.minimize("naive", t[0], t[1], policy=1, seed=3))
    monkeypatch.delenv("DFAKIT_TEST_ARB_REPLAY")
    got = dk.naive_pr(mkdfa(dk, t), dk.ElectionPolicy.arbitrary(3))
    assert same(got, oracle.minimize("naive", t[0], t[1], policy=1, seed=3))


def test_sliced_signature_passes(dk, oracle, monkeypatch):
    """Passes whose key labels exceed the L2 gather their labels in sweeps
    over slices of the label array and add partial keys (packed fields ORed,
    fingerprint terms summed).  A tiny slice size forces that path (up to 64
    slices) on small automata: partitions and pass counts stay the oracle's,
    through fingerprints, packed keys, forced collisions and heavy
    duplication."""
    monkeypatch.setenv("DFAKIT_TEST_SLICE_BYTES", "2048")
    g = random.Random(77)
    for i in range(6):
        n, k, s = g.randint(3000, 30000), g.randint(3, 12), g.getrandbits(64)
        t = oracle.gen_random(n, k, 0.5 if i % 2 else 0.95, s)
        want = oracle.minimize("moore", t[0], t[1])
        dfa = mkdfa(dk, t)
        for kw in ({}, {"fingerprint_bits": 6}, {"force_exact": True}):
            assert same(dk.sort_pr(dfa, **kw), want), (i, kw)
    for n0, c, k in ((2000, 50, 8), (20, 6000, 8)):
        t = copies(oracle.gen_random(n0, k, 0.5, n0 * 7 + c), c)
        assert same(dk.sort_pr(mkdfa(dk, t)), oracle.minimize("moore", t[0], t[1])), (n0, c)
    # more than 16 letters: the chunked sweep kernel instead of the all-letters one
    for n, k, s in ((9000, 20, 3), (12001, 17, 4)):
        t = oracle.gen_random(n, k, 0.5, s)
        want = oracle.minimize("moore", t[0], t[1])
        for kw in ({}, {"fingerprint_bits": 6}):
            assert same(dk.sort_pr(mkdfa(dk, t), **kw), want), (n, k, kw)


def test_speculative_second_pass(dk, oracle, monkeypatch):
    """Large automata queue their second pass (a fingerprint bucket pass over
    every state) behind the first before its counters are read; it is used
    when the first pass left every state active and dropped otherwise.  The
    threshold is lowered so small automata take that path: pass-1 fixed
    points, survivors that make it moot, collisions (6-bit fingerprints) and
    duplicates -- partitions and pass counts stay the oracle's."""
    monkeypatch.setenv("DFAKIT_TEST_SPEC_MIN", "1000")
    g = random.Random(91)
    for i in range(24):
        n, k, s = g.randint(1000, 40000), g.randint(1, 12), g.getrandbits(64)
        t = oracle.gen_random(n, k, [0.5, 0.9, 1.0, 0.0, 0.99][i % 5], s)
        want = oracle.minimize("moore", t[0], t[1])
        dfa = mkdfa(dk, t)
        for kw in ({}, {"fingerprint_bits": 6}):
            assert same(dk.sort_pr(dfa, **kw), want), (i, n, k, kw)
    for n0, c, k in ((2000, 50, 8), (20, 6000, 8), (3000, 3, 12)):
        t = copies(oracle.gen_random(n0, k, 0.5, n0 * 7 + c), c)
        assert same(dk.sort_pr(mkdfa(dk, t)), oracle.minimize("moore", t[0], t[1])), (n0, c)
    t = oracle.gen_synth(2_000_000, 10, 5)
    assert same(dk.sort_pr(mkdfa(dk, t)), oracle.minimize("moore", t[0], t[1]))


def with_duplicates(t, d, seed):
    """t plus d new states, each a duplicate (same row, same acceptance) of a
    random existing state: d small classes among otherwise distinct states."""
    delta, acc, _ = t
    k, n = delta.shape
    src = np.random.default_rng(seed).integers(0, n, d)
    return np.concatenate([delta, delta[:, src]], axis=1), np.concatenate([acc, acc[src]]), 0


@pytest.mark.parametrize("spec", [False, True], ids=["plain", "speculative"])
def test_deferred_pass_mixed_buckets(dk, oracle, monkeypatch, spec):
    """A big fingerprint pass whose buckets are mostly all-distinct (no
    records written, states taken from the entries) with a few holding
    equivalent states (records applied): random automata plus a few
    thousand duplicated states, past the small-automaton kernel's size so the
    bucket grouping defers its labels -- with the speculative second pass on
    the first pass's raw table keys too."""
    if spec:
        monkeypatch.setenv("DFAKIT_TEST_SPEC_MIN", "1000")
    for n0, d, k, s in ((400_000, 3000, 10, 5), (300_000, 40, 12, 6), (250_000, 20_000, 9, 7)):
        t = with_duplicates(oracle.gen_synth(n0, k, s), d, s)
        want = oracle.minimize("moore", t[0], t[1])
        assert want.num_blocks < n0 + d
        assert same(dk.sort_pr(mkdfa(dk, t)), want), (n0, d, k)


def test_speculative_sliced_packed_labels(dk, oracle, monkeypatch):
    """The speculative second pass on the first pass's raw table keys packed
    12 bits apiece five per 64-bit word (sliced -- tiny slice size) or 11
    bits back to back (unsliced): random automata, duplicates, forced
    collisions -- partitions and pass counts stay the oracle's, the packing
    kernels demonstrably ran, and the packing can be switched off."""
    monkeypatch.setenv("DFAKIT_TEST_SPEC_MIN", "1000")
    monkeypatch.setenv("DFAKIT_TEST_SLICE_BYTES", "4096")
    monkeypatch.setenv("DFAKIT_PACK12_MIN_MB", "0")
    g = random.Random(123)
    for i in range(10):
        n, k, s = g.randint(3000, 60000), g.randint(2, 12), g.getrandbits(64)
        t = oracle.gen_random(n, k, [0.5, 0.9, 0.3][i % 3], s)
        if i % 4 == 3:
            t = with_duplicates(t, 300, s)
        want = oracle.minimize("moore", t[0], t[1])
        dfa = mkdfa(dk, t)
        for kw in ({}, {"fingerprint_bits": 6}):
            assert same(dk.sort_pr(dfa, **kw), want), (i, n, k, kw)
    t = oracle.gen_synth(200_001, 10, 9)
    want = oracle.minimize("moore", t[0], t[1])
    dfa = mkdfa(dk, t)

    def kernels_of_run():
        import ctypes as C
        import json
        from paper_2508_20735_b200 import _native as nat
        ctx = dk.Context(0)
        nat.check(nat.lib.dfakit_profile_begin(ctx.handle))
        rep = dk.sort_pr(dfa, ctx=ctx)
        buf = C.create_string_buffer(1 << 16)
        nat.check(nat.lib.dfakit_profile_end(ctx.handle, buf, len(buf)))
        return rep, {x["name"] for x in json.loads(buf.value.decode())}

    rep, names = kernels_of_run()  # sliced: 12-bit fields
    assert same(rep, want) and "pack12_kernel" in names, names
    monkeypatch.delenv("DFAKIT_TEST_SLICE_BYTES")  # unsliced: 11-bit fields
    rep, names = kernels_of_run()
    assert same(rep, want) and "pack11_kernel" in names, names
    monkeypatch.setenv("DFAKIT_NO_PACK12", "1")
    rep, names = kernels_of_run()
    assert same(rep, want) and not any(x.startswith("pack1") for x in names), names
