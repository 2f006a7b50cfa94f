#!/usr/bin/env python
"""Randomised parity sweep on the GPU against the oracle (a longer, seeded
version of the -m gpu tests' sweeps): sort_pr under the production paths
(speculative second pass, lazy apply, singleton buckets, packed labels,
sliced passes -- thresholds lowered so small automata take them) and the
product exploration (primary table, tiny hash table).

    python tools/parity_sweep.py [--cases 300] [--seed 1]
"""
import argparse
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--cases", type=int, default=300)
    p.add_argument("--seed", type=int, default=1)
    a = p.parse_args()
    bad = sweep(a.cases, a.seed)
    sys.exit(1 if bad else 0)


def sweep(cases, seed, log=print):
    """Returns the number of mismatches (each also logged)."""
    import numpy as np
    import paper_2508_20735_b200 as dk
    import pyoracle
    from conftest import mkdfa
    o = pyoracle.COracle()
    g = random.Random(seed)
    envs = [{}, {"DFAKIT_TEST_SPEC_MIN": "500"},
            {"DFAKIT_TEST_SPEC_MIN": "500", "DFAKIT_PACK12_MIN_MB": "0"},
            {"DFAKIT_TEST_SPEC_MIN": "500", "DFAKIT_PACK12_MIN_MB": "0", "DFAKIT_TEST_SLICE_BYTES": "2048"},
            {"DFAKIT_TEST_SLICE_BYTES": "2048"}]
    bad = 0
    for i in range(cases):
        n, k = g.randint(2, 40000), g.randint(1, 14)
        frac = g.choice([0.0, 0.1, 0.5, 0.9, 1.0])
        t = o.gen_random(n, k, frac, g.getrandbits(64))
        if g.random() < 0.3:  # duplicated states: small classes among distinct ones
            d, acc, _ = t
            src = np.random.default_rng(i).integers(0, n, max(1, n // 50))
            t = (np.concatenate([d, d[:, src]], axis=1), np.concatenate([acc, acc[src]]), 0)
        want = o.minimize("moore", t[0], t[1])
        env = envs[i % len(envs)]
        fp = {"fingerprint_bits": 6} if g.random() < 0.2 else {}
        try:
            for key, val in env.items():
                os.environ[key] = val
            r = dk.sort_pr(mkdfa(dk, t), **fp)
        finally:
            for key in env:
                os.environ.pop(key, None)
        ok = (np.array_equal(r.partition.block_of, want.blocks) and r.refining_iterations == want.refine_iters)
        if not ok:
            bad += 1
            log(f"MISMATCH sort_pr {i} {n} {k} {frac} {env} {fp}")
        if i % 3 == 0:  # product exploration against the oracle
            A = t
            if g.random() < 0.5:  # a different pair: small, so the product stays within the pair budget
                A = o.gen_random(g.randint(2, 3000), k, frac, g.getrandbits(64))
                B = o.gen_random(g.randint(2, 3000), k, frac, g.getrandbits(64))
            else:
                B = t
            tiny = g.random() < 0.3
            mode = g.choice(["equivalence", "inclusion", "full"])
            try:
                if tiny:
                    os.environ["DFAKIT_TEST_TABLE_LOG2"] = "6"
                rr = dk.explore_product(mkdfa(dk, A), mkdfa(dk, B), dk.ExploreMode[mode])
            finally:
                os.environ.pop("DFAKIT_TEST_TABLE_LOG2", None)
            oo = o.explore(mode, A, B)
            if (rr.verdict.name, rr.explored_states, rr.levels, rr.counterexample) != \
                    (oo.verdict, oo.explored, oo.levels, oo.counterexample):
                bad += 1
                log(f"MISMATCH explore {i} {mode}")
    log(f"parity sweep: {cases} cases, {bad} mismatches")
    return bad


if __name__ == "__main__":
    main()
