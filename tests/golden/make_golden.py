"""Generate tests/golden/reference_vectors.json from the reference itself.

Runs HERE (where /root/reference exists): builds oracle/_ref (the unmodified
reference sources compiled in place, see oracle/Makefile) and records its
outputs.  The GPU box never runs this; it only reads the committed JSON.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.json")


def digest(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()[:32]


def blocks_entry(res, n):
    return [int(x) for x in res.blocks] if n <= 64 else digest(res.blocks.astype(np.uint32))


def random_cases(count: int, seed: int, nmax: int = 200, kmax: int = 4):
    g = random.Random(seed)
    out = []
    for _ in range(count):
        n = g.randint(1, nmax)
        k = g.randint(1, kmax)
        frac = g.randint(0, 10) / 10
        s = g.getrandbits(64)
        out.append((n, k, frac, s))
    return out


def main() -> None:
    pyoracle.build()
    ref = pyoracle.RefLib()
    data = {"source": "reference sources /root/reference/proj/src compiled by oracle/Makefile",
            "generators": [], "random": [], "minimize": [], "products": [], "transitive": [], "acceptance": {}}

    # --- generator outputs (src/generators.cpp) ---
    fams = [("fib", range(2, 20)), ("bitsplit", range(1, 16)), ("bitsplit-ext", range(1, 12)),
            ("cycle", range(2, 26)), ("memory-perfect", range(1, 12)), ("memory-forgetful", range(2, 12))]
    for fam, ps in fams:
        for p in ps:
            d, a, init = ref.gen_family(fam, p)
            data["generators"].append({"family": fam, "param": p, "n": int(d.shape[1]), "k": int(d.shape[0]),
                                       "initial": init, "delta": digest(d), "acc": digest(a)})
    for (n, k, frac, s) in random_cases(60, 11, 3000, 6):
        d, a, _ = ref.gen_random(n, k, frac, s)
        data["random"].append({"n": n, "k": k, "frac": frac, "seed": s, "delta": digest(d), "acc": digest(a)})

    # --- minimisers (src/minimize.cpp) on random DFAs and families ---
    algos = ["moore", "sort", "naive", "naive-fused", "transpr"]
    cases = [("random", c) for c in random_cases(120, 1234)]
    cases += [("family", ("fib", m)) for m in (2, 5, 9, 12, 16)]
    cases += [("family", ("bitsplit", m)) for m in (1, 2, 5, 8, 10)]
    cases += [("family", ("bitsplit-ext", m)) for m in (1, 3, 6)]
    cases += [("family", ("cycle", m)) for m in (5, 9, 13)]
    cases += [("family", ("memory-perfect", m)) for m in (1, 4, 7)]
    cases += [("family", ("memory-forgetful", m)) for m in (2, 4, 7)]
    for kind, spec in cases:
        if kind == "random":
            n, k, frac, s = spec
            d, a, init = ref.gen_random(n, k, frac, s)
            tag = {"kind": "random", "n": n, "k": k, "frac": frac, "seed": s}
        else:
            d, a, init = ref.gen_family(*spec)
            tag = {"kind": "family", "family": spec[0], "param": spec[1]}
        n = int(d.shape[1])
        entry = dict(tag)
        entry["results"] = {}
        for algo in algos + (["trans"] if n <= 30 else []):
            pols = [(0, 0)]
            if algo in ("naive", "transpr"):
                pols.append((1, 7))
            for pol, sd in pols:
                r = ref.minimize(algo, d, a, pol, sd)
                key = algo if pol == 0 else f"{algo}@arbitrary{sd}"
                entry["results"][key] = {"num_blocks": r.num_blocks, "refine_iters": r.refine_iters,
                                         "closure_iters": r.closure_iters, "blocks": blocks_entry(r, n)}
        data["minimize"].append(entry)
        if kind == "random" and len(data["transitive"]) < 30:
            t = ref.transitive_alphabet(d, a)
            data["transitive"].append({"n": spec[0], "k": spec[1], "frac": spec[2], "seed": spec[3],
                                       "k_out": int(t.shape[0]), "delta": digest(t)})

    # --- product exploration (src/equivalence.cpp) ---
    g = random.Random(99)
    for i in range(120):
        na, nb = g.randint(1, 80), g.randint(1, 80)
        k = g.randint(1, 3)
        frac = g.randint(0, 10) / 10
        sa, sb = g.getrandbits(64), g.getrandbits(64)
        A = ref.gen_random(na, k, frac, sa)
        B = ref.gen_random(nb, k, frac, sb) if i % 3 else A
        for mode in ("equivalence", "inclusion", "full"):
            r = ref.explore(mode, A, B)
            data["products"].append({"na": na, "nb": nb, "k": k, "frac": frac, "sa": sa, "sb": sb,
                                     "same": i % 3 == 0, "mode": mode, "verdict": r.verdict,
                                     "explored": r.explored, "levels": r.levels, "word": r.counterexample})
    for (fa, pa, fb, pb) in [("memory-forgetful", 5, "memory-perfect", 5), ("memory-perfect", 3, "memory-forgetful", 3),
                             ("bitsplit-ext", 5, "bitsplit-ext", 5), ("memory-perfect", 2, "memory-perfect", 2)]:
        A, B = ref.gen_family(fa, pa), ref.gen_family(fb, pb)
        for mode in ("equivalence", "inclusion", "full"):
            r = ref.explore(mode, A, B)
            data["products"].append({"fam_a": fa, "pa": pa, "fam_b": fb, "pb": pb, "mode": mode,
                                     "verdict": r.verdict, "explored": r.explored, "levels": r.levels,
                                     "word": r.counterexample})

    # --- the reference's acceptance numbers (tests/acceptance.cpp) ---
    acc = data["acceptance"]
    acc["bitsplit"] = {}
    for n in range(10, 16):
        d, a, _ = ref.gen_family("bitsplit", n)
        acc["bitsplit"][str(n)] = {al: ref.minimize(al, d, a, want_blocks=False).refine_iters
                                   for al in ("naive", "sort", "transpr")}
    d, a, _ = ref.gen_family("fib", 19)
    acc["fib19"] = {al: ref.minimize(al, d, a, want_blocks=False).refine_iters for al in ("naive", "sort", "transpr")}
    acc["trans_closure"] = {}
    for m in (5, 6, 7, 8, 9):
        d, a, _ = ref.gen_family("fib", m)
        r = ref.minimize("trans", d, a)
        acc["trans_closure"][str(m)] = [r.num_blocks, r.refine_iters, r.closure_iters]
    acc["self_equiv_ext"] = {}
    for n in range(5, 15):
        A = ref.gen_family("bitsplit-ext", n)
        r = ref.explore("equivalence", A, A)
        acc["self_equiv_ext"][str(n)] = [r.verdict, r.explored, r.levels]
    acc["self_equiv_cycle"] = {}
    for n in (20, 30, 31):
        A = ref.gen_family("cycle", n)
        r = ref.explore("equivalence", A, A)
        acc["self_equiv_cycle"][str(n)] = [r.verdict, r.explored, r.levels]
    acc["inclusion_memory"] = {}
    for n in range(5, 11):
        r = ref.explore("inclusion", ref.gen_family("memory-forgetful", n), ref.gen_family("memory-perfect", n))
        acc["inclusion_memory"][str(n)] = [r.verdict, r.explored, r.levels]

    with open(OUT, "w") as f:
        json.dump(data, f, separators=(",", ":"))
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
