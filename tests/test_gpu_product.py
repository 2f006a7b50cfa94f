"""GPU parity of equivalence / inclusion checking.  Naive Hopcroft-Karp
(explore_product): verdict, explored_states, levels and the counterexample
word must equal the reference's exactly.  Union-find Hopcroft-Karp: verdict
must equal, the witness must distinguish the languages."""
import random

import numpy as np
import pytest

from conftest import mkdfa

pytestmark = pytest.mark.gpu


def accepts(t, word):
    delta, acc, init = t
    q = init
    for a in word:
        q = delta[a][q]
    return bool(acc[q])


def same(r, o):
    return (r.verdict.name, r.explored_states, r.levels, r.counterexample) == \
        (o.verdict, o.explored, o.levels, o.counterexample)


def test_golden_products(dk, oracle, golden):
    for e in golden["products"]:
        if "fam_a" in e:
            A, B = oracle.gen_family(e["fam_a"], e["pa"]), oracle.gen_family(e["fam_b"], e["pb"])
        else:
            A = oracle.gen_random(e["na"], e["k"], e["frac"], e["sa"])
            B = A if e["same"] else oracle.gen_random(e["nb"], e["k"], e["frac"], e["sb"])
        r = dk.explore_product(mkdfa(dk, A), mkdfa(dk, B), dk.ExploreMode[e["mode"]])
        assert (r.verdict.name, r.explored_states, r.levels, r.counterexample) == \
            (e["verdict"], e["explored"], e["levels"], e["word"]), e


def test_random_products_vs_oracle(dk, oracle):
    g = random.Random(5000)
    for i in range(150):
        na, nb, k = g.randint(2, 100), g.randint(2, 100), g.randint(1, 3)
        frac = g.randint(0, 10) / 10
        A = oracle.gen_random(na, k, frac, g.getrandbits(64))
        B = A if i % 2 == 0 else oracle.gen_random(nb, k, frac, g.getrandbits(64))
        da, db = mkdfa(dk, A), mkdfa(dk, B)
        for mode in ("equivalence", "inclusion", "full"):
            r = dk.explore_product(da, db, dk.ExploreMode[mode])
            assert same(r, oracle.explore(mode, A, B)), (i, mode)
        u = dk.check_equiv_uf(da, db)
        e = oracle.explore("equivalence", A, B)
        assert u.verdict.name == e.verdict
        if u.verdict.name == "counterexample":
            assert accepts(A, u.counterexample) != accepts(B, u.counterexample)


@pytest.mark.parametrize("table", ["hash", "primary"])
def test_products_through_table_collisions(dk, oracle, monkeypatch, table):
    """A 64-slot first hash table (test hook): explorations run at load up to
    1/2, so keys collide on their home slots and go through the
    tile-cooperative windows, and the table grows and re-inserts the
    records; results must not change.  `hash`: every pair in the hash table
    (the primary table off); `primary` (the default): pairs whose first
    state's direct-mapped slot is taken go to the hash table, whose
    reservations run out mid-level -- the table grows and the level re-runs."""
    if table == "hash":
        monkeypatch.setenv("DFAKIT_BFS_NO_PRIMARY", "1")
    ctx = dk.default_context()
    A = oracle.gen_random(3000, 2, 0.5, 1)
    B = A if table == "hash" else oracle.gen_random(2500, 2, 0.5, 2)
    da, db = mkdfa(dk, A), mkdfa(dk, B)
    l0 = ctx.kernel_launches
    dk.explore_product(da, db, dk.ExploreMode["full"])
    plain = ctx.kernel_launches - l0
    monkeypatch.setenv("DFAKIT_TEST_TABLE_LOG2", "6")
    l0 = ctx.kernel_launches
    r = dk.explore_product(da, db, dk.ExploreMode["full"])
    assert same(r, oracle.explore("full", A, B))
    assert ctx.kernel_launches - l0 > plain + 2  # the 64-slot table grew: re-insertions, relaunches
    g = random.Random(77)
    for i in range(40):
        na, nb, k = g.randint(20, 800), g.randint(20, 800), g.randint(1, 4)
        frac = g.randint(1, 9) / 10
        A = oracle.gen_random(na, k, frac, g.getrandbits(64))
        B = A if i % 3 == 0 else oracle.gen_random(nb, k, frac, g.getrandbits(64))
        da, db = mkdfa(dk, A), mkdfa(dk, B)
        for mode in ("equivalence", "inclusion", "full"):
            assert same(dk.explore_product(da, db, dk.ExploreMode[mode]), oracle.explore(mode, A, B)), (i, mode)


def test_acceptance_product_sizes(dk, oracle, golden):
    """Acceptance criteria 5 and 6 (Table 4 / Table 5 state counts)."""
    acc = golden["acceptance"]
    for n, (v, e, lv) in acc["self_equiv_ext"].items():
        A = mkdfa(dk, oracle.gen_family("bitsplit-ext", int(n)))
        r = dk.check_equiv(A, A)
        assert (r.verdict.name, r.explored_states, r.levels) == (v, e, lv)
    for n, (v, e, lv) in acc["self_equiv_cycle"].items():
        A = mkdfa(dk, oracle.gen_family("cycle", int(n)))
        r = dk.check_equiv(A, A)
        assert (r.verdict.name, r.explored_states, r.levels) == (v, e, lv)
    for n, (v, e, lv) in acc["inclusion_memory"].items():
        r = dk.check_inclusion(mkdfa(dk, oracle.gen_family("memory-forgetful", int(n))),
                               mkdfa(dk, oracle.gen_family("memory-perfect", int(n))))
        assert (r.verdict.name, r.explored_states, r.levels) == (v, e, lv)


def test_empty_word_and_errors(dk, oracle):
    yes = mkdfa(dk, oracle.gen_random(5, 2, 1.0, 1))
    no = mkdfa(dk, oracle.gen_random(5, 2, 0.0, 1))
    r = dk.check_equiv(yes, no)
    assert r.verdict == dk.Verdict.counterexample and r.counterexample == [] and r.explored_states == 1
    assert r.levels == 0
    full = dk.explore_product(yes, no, dk.ExploreMode.full)
    assert full.verdict == dk.Verdict.counterexample and full.counterexample == [] and full.explored_states > 1
    nob = mkdfa(dk, oracle.gen_family("bitsplit", 3))
    with pytest.raises(ValueError):
        dk.check_equiv(nob, nob)
    with pytest.raises(ValueError):
        dk.check_equiv(mkdfa(dk, oracle.gen_random(4, 2, 0.5, 1)), mkdfa(dk, oracle.gen_random(4, 3, 0.5, 1)))
    big = mkdfa(dk, oracle.gen_family("memory-perfect", 8))
    with pytest.raises(dk.ResourceError):
        dk.check_equiv(big, big, dk.ExploreOptions(max_visited=10))


def test_budget_matches_reference_semantics(dk, oracle):
    A = oracle.gen_family("memory-perfect", 6)
    B = oracle.gen_family("memory-forgetful", 6)
    for mv in (1, 2, 3, 5, 9, 17, 40, 200):
        for mode in ("equivalence", "inclusion", "full"):
            try:
                want = oracle.explore(mode, A, B, max_visited=mv)
            except MemoryError:
                want = None
            if want is None:
                with pytest.raises(dk.ResourceError):
                    dk.explore_product(mkdfa(dk, A), mkdfa(dk, B), dk.ExploreMode[mode],
                                       dk.ExploreOptions(max_visited=mv))
            else:
                r = dk.explore_product(mkdfa(dk, A), mkdfa(dk, B), dk.ExploreMode[mode],
                                       dk.ExploreOptions(max_visited=mv))
                assert same(r, want), (mv, mode)


def test_letters_matched_by_name(dk, oracle):
    d, a, init = oracle.gen_family("memory-perfect", 3)
    A = dk.Dfa(d, a, init, ["f", "t"])
    B = dk.Dfa(d[::-1].copy(), a, init, ["t", "f"])
    assert dk.check_equiv(A, B).verdict == dk.Verdict.counterexample
    assert dk.check_equiv(A, B, dk.ExploreOptions(match_letters_by_name=True)).verdict == dk.Verdict.equivalent


@pytest.mark.slow
def test_large_equal_and_differing_pairs(dk, oracle):
    """BASELINE configs[3] shape at 1M states: a DFA against a relabelled copy
    (equal) and against a copy with one flipped accepting bit (differing)."""
    n, k = 1_000_000, 4
    d, a, _ = oracle.gen_synth(n, k, 3)
    perm = np.random.default_rng(1).permutation(n).astype(np.uint32)
    d2 = np.empty_like(d)
    for l in range(k):
        d2[l][perm] = perm[d[l]]
    a2 = np.empty_like(a)
    a2[perm] = a
    A, B = (d, a, 0), (d2, a2, int(perm[0]))
    r = dk.check_equiv(mkdfa(dk, A), mkdfa(dk, B))
    o = oracle.explore("equivalence", A, B)
    assert same(r, o) and r.verdict == dk.Verdict.equivalent
    u = dk.check_equiv_uf(mkdfa(dk, A), mkdfa(dk, B))
    assert u.verdict == dk.Verdict.equivalent
    a3 = a2.copy()
    a3[d2[0][perm[0]]] ^= 1
    C = (d2, a3, int(perm[0]))
    r = dk.check_equiv(mkdfa(dk, A), mkdfa(dk, C))
    o = oracle.explore("equivalence", A, C)
    assert same(r, o) and r.verdict == dk.Verdict.counterexample
    r = dk.check_inclusion(mkdfa(dk, A), mkdfa(dk, C))
    assert same(r, oracle.explore("inclusion", A, C))


@pytest.mark.slow
def test_config3_full_size_10M(dk, oracle):
    """BASELINE configs[3] at full size, the bench's shape: a 10M-state DFA
    over two letters against a relabelled copy (equal: ~8M product pairs, 42
    levels) and against the copy with the accepting bit flipped at the state
    30 letters-0 from the initial state (differing).  Verdict, explored pairs,
    levels and counterexample word identical to the oracle's."""
    n, k = 10_000_000, 2
    d, a, _ = oracle.gen_synth(n, k, 11)
    perm = np.random.default_rng(5).permutation(n).astype(np.uint32)
    d2 = np.empty_like(d)
    for l in range(k):
        d2[l][perm] = perm[d[l]]
    a2 = np.empty_like(a)
    a2[perm] = a
    A, B = (d, a, 0), (d2, a2, int(perm[0]))
    da, db = mkdfa(dk, A), mkdfa(dk, B)
    for mode in ("equivalence", "inclusion"):
        r = dk.explore_product(da, db, dk.ExploreMode[mode])
        assert same(r, oracle.explore(mode, A, B)), mode
    assert dk.check_equiv_uf(da, db).verdict == dk.Verdict.equivalent
    q = int(perm[0])
    for _ in range(30):
        q = int(d2[0][q])
    a3 = a2.copy()
    a3[q] ^= 1
    C = (d2, a3, int(perm[0]))
    dc = mkdfa(dk, C)
    for mode in ("equivalence", "inclusion"):
        r = dk.explore_product(da, dc, dk.ExploreMode[mode])
        assert same(r, oracle.explore(mode, A, C)), mode
    u = dk.check_equiv_uf(da, dc)
    assert u.verdict == dk.Verdict.counterexample and accepts(A, u.counterexample) != accepts(C, u.counterexample)
