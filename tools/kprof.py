#!/usr/bin/env python
"""Wall time and live per-kernel breakdown (the library's CUDA-event
profiler) of one workload -- a development aid for picking what to optimise.

    python tools/kprof.py chain [--states N] [--reps R]
    python tools/kprof.py synth | fib | equiv
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("workload", choices=["synth", "chain", "fib", "naive", "equiv", "sharded"])
    p.add_argument("--states", type=int, default=None)
    p.add_argument("--alphabet", type=int, default=10)
    p.add_argument("--param", type=int, default=19)
    p.add_argument("--algo", default=None)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--grouping", type=int, default=0, help="dfakit_options.grouping (1 = radix_sort)")
    p.add_argument("--host", action="store_true", help="synth: through dfakit_minimize with pinned host buffers")
    a = p.parse_args()
    import torch
    import paper_2508_20735_b200 as dk
    from paper_2508_20735_b200 import _native as nat

    ctx = dk.Context(0)
    w = a.workload
    if w == "fib":
        import pyoracle
        d, acc, _ = pyoracle.COracle().gen_family("fib", a.param)
        n, k = len(acc), 1
        delta = torch.from_numpy(d.astype("int32").reshape(-1)).cuda()
        accd = torch.from_numpy(acc.astype("uint8")).cuda()
    else:
        n = a.states or {"naive": 100_000}.get(w, 10_000_000)
        k = {"chain": 1, "equiv": 2}.get(w, a.alphabet)
        delta = torch.empty(k * n, dtype=torch.int32, device="cuda")
        accd = torch.empty(n, dtype=torch.uint8, device="cuda")
        if w == "chain":
            nat.check(nat.lib.dfakit_gen_chain_device(ctx.handle, n, delta.data_ptr(), accd.data_ptr(), ctx.stream))
        else:
            nat.check(nat.lib.dfakit_gen_synth_device(ctx.handle, n, k, 1, delta.data_ptr(), accd.data_ptr(),
                                                      ctx.stream))
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    view = nat.CDfa(n, k, delta.data_ptr(), accd.data_ptr(), 0)
    algo = a.algo or {"chain": "trans_pr", "naive": "naive_pr"}.get(w, "sort_pr")
    if algo == "uf":
        algo = "sort_pr"  # (report label only; the equiv workload reads a.algo)

    def run():
        rep = nat.CReport()
        opts = nat.COptions(0, 0, 0, 1 << 40, 1 << 24, 64, a.grouping)
        nat.check(nat.lib.dfakit_minimize_device(ctx.handle, C.byref(view), int(dk.Algorithm[algo]), C.byref(opts),
                                                 out.data_ptr(), C.byref(rep), ctx.stream))
        return rep

    if a.host and w == "synth":
        hd = torch.empty(k * n, dtype=torch.int32, pin_memory=True)
        ha = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        hb = torch.empty(n, dtype=torch.int32, pin_memory=True)
        hd.copy_(delta.cpu())
        ha.copy_(accd.cpu())
        hview = nat.CDfa(n, k, hd.data_ptr(), ha.data_ptr(), -1)

        def run():  # noqa: F811
            rep = nat.CReport()
            opts = nat.COptions(0, 0, 0, 1 << 40, 1 << 24, 64, a.grouping)
            nat.check(nat.lib.dfakit_minimize(ctx.handle, C.byref(hview), int(dk.Algorithm[algo]), C.byref(opts),
                                              hb.data_ptr(), C.byref(rep)))
            return rep

    if w == "sharded":  # the native sharded engine at world size 1 (NCCL)
        import socket
        import torch.distributed as dist
        from paper_2508_20735_b200 import sharded
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
        sk.close()
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        ncomm = sharded.NativeComm(ctx)

        def run():  # noqa: F811
            _, r = sharded.sort_pr_sharded_native(ctx, ncomm, delta, accd, n, k, out=out)
            rep = nat.CReport()
            rep.passes, rep.num_blocks = r.passes, r.num_blocks
            return rep

    if w == "equiv":
        d2 = torch.empty(k * n, dtype=torch.int32, device="cuda")
        a2 = torch.empty(n, dtype=torch.uint8, device="cuda")
        init2 = C.c_uint32()
        nat.check(nat.lib.dfakit_permute_states_device(ctx.handle, n, k, 5, delta.data_ptr(), accd.data_ptr(),
                                                       d2.data_ptr(), a2.data_ptr(), C.byref(init2), ctx.stream))
        v2 = nat.CDfa(n, k, d2.data_ptr(), a2.data_ptr(), init2.value)

        def run():  # noqa: F811
            r = nat.CProduct()
            cex = (C.c_uint32 * 4096)()
            if a.algo == "uf":  # union-find Hopcroft-Karp
                nat.check(nat.lib.dfakit_check_equiv_uf_device(ctx.handle, C.byref(view), C.byref(v2), cex, 4096,
                                                               C.byref(r), ctx.stream))
                return r
            nat.check(nat.lib.dfakit_explore_product_device(ctx.handle, C.byref(view), C.byref(v2), 0, None,
                                                            1 << 40, cex, 4096, C.byref(r), ctx.stream))
            return r

    run()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(a.reps):
        rep = run()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) * 1000 / a.reps
    print(f"{w} n={n} k={k} {algo}: {ms:.3f} ms/run (wall)")
    if hasattr(rep, "passes"):
        print("passes", rep.passes, "blocks", rep.num_blocks)
    nat.check(nat.lib.dfakit_profile_begin(ctx.handle))
    for _ in range(a.reps):
        run()
    buf = C.create_string_buffer(1 << 16)
    nat.check(nat.lib.dfakit_profile_end(ctx.handle, buf, len(buf)))
    allk = json.loads(buf.value.decode())
    ks = sorted((x for x in allk if not x["name"].startswith("#")), key=lambda x: -x["ms"])
    for x in allk:
        if x["name"].startswith("#pass"):
            print(f"  {x['name']:10s} {x['ms'] / a.reps:9.3f} ms  {x['bytes'] / a.reps / 1e6:9.1f} MB algorithmic")
    tot = sum(x["ms"] for x in ks)
    for x in ks[:15]:
        print(f"  {x['name'][:40]:40s} {x['ms'] / a.reps:9.3f} ms  x{x['launches'] / a.reps:.1f}  {100 * x['ms'] / tot:5.1f}%")
    print(f"  kernels total {tot / a.reps:.3f} ms/run")


if __name__ == "__main__":
    main()
