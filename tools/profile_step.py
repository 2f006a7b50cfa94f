#!/usr/bin/env python
"""Short device-resident workload for ncu captures (one GPU, no timing).

    python tools/profile_step.py [--algo sort_pr] [--states N] [--alphabet K] [--reps R] [--workload synth|chain|equiv]

Runs R minimisations (or product explorations) of the bench's synthetic
input so `ncu -k regex:<kernel> -s <skip> -c <count>` can pick launches
after the first (warm-up) repetition.  Numbers printed under ncu are never
bench values.
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--algo", default="sort_pr")
    p.add_argument("--workload", default="synth", choices=["synth", "chain", "equiv"])
    p.add_argument("--states", type=int, default=10_000_000)
    p.add_argument("--alphabet", type=int, default=10)
    p.add_argument("--reps", type=int, default=2)
    a = p.parse_args()
    import torch
    import paper_2508_20735_b200 as dk
    from paper_2508_20735_b200 import _native as nat

    ctx = dk.Context(0)
    n, k = a.states, (1 if a.workload == "chain" else a.alphabet)
    delta = torch.empty(k * n, dtype=torch.int32, device="cuda")
    acc = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    if a.workload == "chain":
        nat.check(nat.lib.dfakit_gen_chain_device(ctx.handle, n, delta.data_ptr(), acc.data_ptr(), ctx.stream))
        algo = "trans_pr"
    else:
        nat.check(nat.lib.dfakit_gen_synth_device(ctx.handle, n, k, 1, delta.data_ptr(), acc.data_ptr(), ctx.stream))
        algo = a.algo
    torch.cuda.synchronize()
    view = nat.CDfa(n, k, delta.data_ptr(), acc.data_ptr(), 0)
    if a.workload == "equiv":
        d2 = torch.empty(k * n, dtype=torch.int32, device="cuda")
        a2 = torch.empty(n, dtype=torch.uint8, device="cuda")
        init2 = C.c_uint32()
        nat.check(nat.lib.dfakit_permute_states_device(ctx.handle, n, k, 5, delta.data_ptr(), acc.data_ptr(),
                                                       d2.data_ptr(), a2.data_ptr(), C.byref(init2), ctx.stream))
        vb = nat.CDfa(n, k, d2.data_ptr(), a2.data_ptr(), int(init2.value))
        res = nat.CProduct()
        for _ in range(a.reps):
            nat.check(nat.lib.dfakit_explore_product_device(ctx.handle, C.byref(view), C.byref(vb), 0, None, 1 << 32,
                                                            None, 0, C.byref(res), ctx.stream))
        print("explored", res.explored_states, "levels", res.levels)
        return
    opts = nat.COptions(0, 0, 0, 1 << 40, 0, 64, 0)
    rep = nat.CReport()
    for _ in range(a.reps):
        nat.check(nat.lib.dfakit_minimize_device(ctx.handle, C.byref(view), int(dk.Algorithm[algo]), C.byref(opts),
                                                 out.data_ptr(), C.byref(rep), ctx.stream))
    torch.cuda.synchronize()
    print("passes", rep.passes, "blocks", rep.num_blocks, "launches", ctx.kernel_launches)


if __name__ == "__main__":
    main()
