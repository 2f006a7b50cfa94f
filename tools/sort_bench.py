#!/usr/bin/env python
"""Per-digit timing of the LSD radix sort (dfakit_radix_sort_pairs_device) on
m random (64-bit key, 32-bit value) pairs -- the onesweep kernel alone.

    python tools/sort_bench.py [--m 10000000] [--bits 64] [--reps 5]
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--m", type=int, default=10_000_000)
    p.add_argument("--bits", type=int, default=64)
    p.add_argument("--reps", type=int, default=5)
    a = p.parse_args()
    import torch
    import paper_2508_20735_b200 as dk
    from paper_2508_20735_b200 import _native as nat
    ctx = dk.Context(0)
    g = torch.Generator(device="cuda").manual_seed(1)
    src = torch.randint(-(1 << 62), 1 << 62, (a.m,), dtype=torch.int64, device="cuda", generator=g)
    k0, v0 = torch.empty_like(src), torch.arange(a.m, dtype=torch.int32, device="cuda")
    k1, v1 = torch.empty_like(k0), torch.empty_like(v0)
    fl = C.c_int32()

    def run():
        k0.copy_(src)
        torch.cuda.synchronize()
        nat.check(nat.lib.dfakit_radix_sort_pairs_device(ctx.handle, k0.data_ptr(), v0.data_ptr(), k1.data_ptr(),
                                                         v1.data_ptr(), a.m, a.bits, C.byref(fl), ctx.stream))
    run()
    nat.check(nat.lib.dfakit_profile_begin(ctx.handle))
    for _ in range(a.reps):
        run()
    buf = C.create_string_buffer(1 << 16)
    nat.check(nat.lib.dfakit_profile_end(ctx.handle, buf, len(buf)))
    for x in sorted(json.loads(buf.value.decode()), key=lambda x: -x["ms"]):
        per = x["ms"] / x["launches"]
        gbs = x["bytes"] / (x["ms"] / 1e3) / 1e9 if x["bytes"] else 0
        print(f"  {x['name'][:40]:40s} {per * 1000:8.1f} us/launch  x{x['launches'] / a.reps:.0f}  {gbs:7.0f} GB/s")
    # calibration: torch.sort (CUB device radix sort, 64-bit keys + 64-bit
    # indices) on the same keys, whole sort
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for stable in (True,):
        torch.sort(src, stable=stable)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            torch.sort(src, stable=stable)
        e1.record()
        torch.cuda.synchronize()
        print(f"  torch.sort(int64, stable={stable}) {e0.elapsed_time(e1) / a.reps * 1000:8.1f} us per sort")


if __name__ == "__main__":
    main()
