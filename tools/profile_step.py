#!/usr/bin/env python
"""Short device-resident workloads for ncu captures (one GPU, no timing).

    python tools/profile_step.py [--workload W] [--states N] [--alphabet K] [--reps R]

workloads:
  synth     sort_pr on the bench automaton (10M x 10)          [default]
  radix     sort_pr with grouping=radix_sort (literal Alg. 4)
  naive     naive_pr + naive_pr_fused on 100K x 10
  chain     trans_pr on a 10M-state chain (pointer doubling)
  equiv     equivalence + inclusion (hash-set product BFS) and union-find HK, 10M x 2
  sharded   the native sharded engine at world size 1 (NCCL), 10M x 10
  trans     trans_minimize (CH92) on Fibonacci 12
  fib       naive_pr / naive_pr_fused (single-CTA kernels) and sort_pr (persistent small-m engine) on Fibonacci 19
  calib     the random-gather calibration probe

Numbers printed under ncu are never bench values.
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--workload", default="synth",
                   choices=["synth", "radix", "naive", "chain", "equiv", "sharded", "trans", "calib", "fib"])
    p.add_argument("--states", type=int, default=None)
    p.add_argument("--alphabet", type=int, default=10)
    p.add_argument("--reps", type=int, default=2)
    a = p.parse_args()
    import torch
    import paper_2508_20735_b200 as dk
    from paper_2508_20735_b200 import _native as nat

    ctx = dk.Context(0)
    w = a.workload
    n = a.states or {"naive": 100_000, "trans": 0}.get(w, 10_000_000)
    k = {"chain": 1, "equiv": 2}.get(w, a.alphabet)

    def minimize(view, algo, out, grouping=0):
        rep = nat.CReport()
        opts = nat.COptions(0, 0, 0, 1 << 40, 1 << 24, 64, grouping)
        nat.check(nat.lib.dfakit_minimize_device(ctx.handle, C.byref(view), int(dk.Algorithm[algo]), C.byref(opts),
                                                 out.data_ptr(), C.byref(rep), ctx.stream))
        return rep

    if w == "calib":
        r = C.c_double()
        for _ in range(a.reps):
            nat.check(nat.lib.dfakit_calibrate_gather(ctx.handle, n, 4, 100_000_000, C.byref(r)))
        print("gathers/s", r.value)
        return
    if w == "fib":
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle
        d, acc, _ = pyoracle.COracle().gen_family("fib", 19)
        dfa = dk.Dfa(d, acc, 0)
        for fn in (dk.naive_pr, dk.naive_pr_fused, dk.sort_pr):
            res = fn(dfa, ctx=ctx)
        print("passes", res.refining_iterations)
        return
    if w == "trans":
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle
        d, acc, _ = pyoracle.COracle().gen_family("fib", 12)
        dfa = dk.Dfa(d, acc, 0)
        for _ in range(a.reps):
            res = dk.trans_minimize(dfa, max_pair_nodes=1 << 24)
        print("blocks", res.report.partition.num_blocks)
        return
    delta = torch.empty(k * n, dtype=torch.int32, device="cuda")
    acc = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    if w == "chain":
        nat.check(nat.lib.dfakit_gen_chain_device(ctx.handle, n, delta.data_ptr(), acc.data_ptr(), ctx.stream))
    else:
        nat.check(nat.lib.dfakit_gen_synth_device(ctx.handle, n, k, 1, delta.data_ptr(), acc.data_ptr(), ctx.stream))
    torch.cuda.synchronize()
    view = nat.CDfa(n, k, delta.data_ptr(), acc.data_ptr(), 0)
    if w == "equiv":
        d2 = torch.empty(k * n, dtype=torch.int32, device="cuda")
        a2 = torch.empty(n, dtype=torch.uint8, device="cuda")
        init2 = C.c_uint32()
        nat.check(nat.lib.dfakit_permute_states_device(ctx.handle, n, k, 5, delta.data_ptr(), acc.data_ptr(),
                                                       d2.data_ptr(), a2.data_ptr(), C.byref(init2), ctx.stream))
        vb = nat.CDfa(n, k, d2.data_ptr(), a2.data_ptr(), int(init2.value))
        res = nat.CProduct()
        for mode in (0, 1):
            nat.check(nat.lib.dfakit_explore_product_device(ctx.handle, C.byref(view), C.byref(vb), mode, None,
                                                            1 << 32, None, 0, C.byref(res), ctx.stream))
        nat.check(nat.lib.dfakit_check_equiv_uf_device(ctx.handle, C.byref(view), C.byref(vb), None, 0,
                                                       C.byref(res), ctx.stream))
        print("explored", res.explored_states, "levels", res.levels)
        return
    if w == "sharded":
        import torch.distributed as dist
        from paper_2508_20735_b200 import sharded
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        ncomm = sharded.NativeComm(ctx)  # the native C++ driver (owner-bucket layout)
        for _ in range(a.reps):
            blocks, rep = sharded.sort_pr_sharded_native(ctx, ncomm, delta, acc, n, k)
        print("passes", rep.passes, "blocks", rep.num_blocks)
        ncomm.close()
        dist.destroy_process_group()
        return
    if w == "naive":
        for algo in ("naive_pr", "naive_pr_fused"):
            rep = minimize(view, algo, out)
        print("passes", rep.passes, "blocks", rep.num_blocks)
        return
    algo = "trans_pr" if w == "chain" else "sort_pr"
    for _ in range(a.reps):
        rep = minimize(view, algo, out, 1 if w == "radix" else 0)
    torch.cuda.synchronize()
    print("passes", rep.passes, "blocks", rep.num_blocks, "launches", ctx.kernel_launches)


if __name__ == "__main__":
    main()
