"""Pins the C restatement (oracle/oracle.c) against the reference's own
outputs: golden vectors recorded from oracle/_ref (the reference sources
compiled in place) and, when the reference is present, a live sweep."""
import random

import numpy as np
import pytest

from conftest import digest


def _family(oracle, fam, p):
    return oracle.gen_family(fam, p)


def test_generators_match_reference(oracle, golden):
    for g in golden["generators"]:
        d, a, init = _family(oracle, g["family"], g["param"])
        assert (d.shape[1], d.shape[0], init) == (g["n"], g["k"], g["initial"]), g
        assert digest(d) == g["delta"] and digest(a) == g["acc"], g


def test_random_generator_is_libstdcxx_identical(oracle, golden):
    for g in golden["random"]:
        d, a, _ = oracle.gen_random(g["n"], g["k"], g["frac"], g["seed"])
        assert digest(d) == g["delta"] and digest(a) == g["acc"], g


def _case_dfa(oracle, e):
    if e["kind"] == "random":
        return oracle.gen_random(e["n"], e["k"], e["frac"], e["seed"])
    return oracle.gen_family(e["family"], e["param"])


def test_minimisers_match_reference(oracle, golden):
    for e in golden["minimize"]:
        d, a, _ = _case_dfa(oracle, e)
        n = d.shape[1]
        for key, want in e["results"].items():
            algo, _, pol = key.partition("@arbitrary")
            policy, seed = (1, int(pol)) if pol else (0, 0)
            r = oracle.minimize(algo, d, a, policy, seed)
            got_blocks = [int(x) for x in r.blocks] if n <= 64 else digest(r.blocks.astype(np.uint32))
            assert (r.num_blocks, r.refine_iters, r.closure_iters) == \
                (want["num_blocks"], want["refine_iters"], want["closure_iters"]), (e, key)
            assert got_blocks == want["blocks"], (e, key)


def test_transitive_alphabet_matches_reference(oracle, golden):
    for e in golden["transitive"]:
        d, a, _ = oracle.gen_random(e["n"], e["k"], e["frac"], e["seed"])
        t = oracle.transitive_alphabet(d, a)
        assert t.shape[0] == e["k_out"] and digest(t) == e["delta"]


def test_products_match_reference(oracle, golden):
    for e in golden["products"]:
        if "fam_a" in e:
            A, B = oracle.gen_family(e["fam_a"], e["pa"]), oracle.gen_family(e["fam_b"], e["pb"])
        else:
            A = oracle.gen_random(e["na"], e["k"], e["frac"], e["sa"])
            B = A if e["same"] else oracle.gen_random(e["nb"], e["k"], e["frac"], e["sb"])
        r = oracle.explore(e["mode"], A, B)
        assert (r.verdict, r.explored, r.levels, r.counterexample) == \
            (e["verdict"], e["explored"], e["levels"], e["word"]), e


def test_acceptance_numbers(oracle, golden):
    acc = golden["acceptance"]
    for n, want in acc["bitsplit"].items():
        d, a, _ = oracle.gen_family("bitsplit", int(n))
        for algo, it in want.items():
            assert oracle.minimize(algo, d, a).refine_iters == it
    for m, (nb, ri, ci) in acc["trans_closure"].items():
        d, a, _ = oracle.gen_family("fib", int(m))
        r = oracle.minimize("trans", d, a)
        assert (r.num_blocks, r.refine_iters, r.closure_iters) == (nb, ri, ci)
    for n, (v, e, lv) in acc["self_equiv_ext"].items():
        A = oracle.gen_family("bitsplit-ext", int(n))
        r = oracle.explore("equivalence", A, A)
        assert (r.verdict, r.explored, r.levels) == (v, e, lv)
    for n, (v, e, lv) in acc["inclusion_memory"].items():
        r = oracle.explore("inclusion", oracle.gen_family("memory-forgetful", int(n)),
                           oracle.gen_family("memory-perfect", int(n)))
        assert (r.verdict, r.explored, r.levels) == (v, e, lv)


def test_fib19_pass_counts(oracle, golden):
    d, a, _ = oracle.gen_family("fib", 19)
    for algo in ("naive", "sort", "transpr"):
        assert oracle.minimize(algo, d, a).refine_iters == golden["acceptance"]["fib19"][algo]


def test_live_sweep_against_reference(oracle, ref):
    """Criterion-1-style sweep: 300 random DFAs, every minimiser, both backends."""
    g = random.Random(2024)
    for _ in range(300):
        n, k, frac, s = g.randint(1, 200), g.randint(1, 4), g.randint(0, 10) / 10, g.getrandbits(64)
        d, a, _ = ref.gen_random(n, k, frac, s)
        for algo in ("moore", "sort", "naive", "naive-fused", "transpr") + (("trans",) if n <= 25 else ()):
            x, y = oracle.minimize(algo, d, a), ref.minimize(algo, d, a)
            assert np.array_equal(x.blocks, y.blocks) and x.refine_iters == y.refine_iters
            assert x.closure_iters == y.closure_iters


def test_synth_generator_properties(oracle):
    d, a, _ = oracle.gen_synth(1000, 3, 42)
    assert d.shape == (3, 1000) and d.max() < 1000 and set(np.unique(a)) <= {0, 1}
    d2, a2, _ = oracle.gen_synth(1000, 3, 42)
    assert np.array_equal(d, d2) and np.array_equal(a, a2)
    # roughly uniform successors and ~half accepting
    assert 300 < a.sum() < 700
