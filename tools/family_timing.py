#!/usr/bin/env python
"""Times the GPU minimisers on the reference's benchmark families (the
inputs of the reference CLI's `bench --suite`) beside the reference's own
sequential implementation (oracle/_ref).  Prints one JSON line per case."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    import numpy as np
    import paper_2508_20735_b200 as dk
    import pyoracle
    ref = pyoracle.RefLib()
    gen = pyoracle.COracle()
    cases = [("fib", 15), ("fib", 19), ("fib", 23), ("bitsplit", 12), ("bitsplit", 16), ("memory-perfect", 12)]
    for fam, p in cases:
        d, a, init = gen.gen_family(fam, p)
        dfa = dk.Dfa(d, a, None if init < 0 else init)
        for algo, fn in (("sort", dk.sort_pr), ("naive", dk.naive_pr)):
            fn(dfa)  # warm-up
            t0 = time.perf_counter()
            rep = fn(dfa)
            g = time.perf_counter() - t0
            t0 = time.perf_counter()
            want = ref.minimize(algo, d, a, want_blocks=False)
            r = time.perf_counter() - t0
            print(json.dumps({"family": fam, "param": p, "n": int(d.shape[1]), "k": int(d.shape[0]), "algo": algo,
                              "passes": rep.refining_iterations, "ref_passes": want.refine_iters,
                              "gpu_ms": g * 1e3, "ref_cpu_ms": r * 1e3}), flush=True)


if __name__ == "__main__":
    main()
