#!/usr/bin/env python
"""Benchmark: sort-based DFA minimisation (sortPR) on B200.

Step = one full sort_pr minimisation (every refinement pass up to and
including the confirming pass) of a synthetic random DFA resident in HBM.
Default workload (BASELINE.json configs[1]): 10M states x |Sigma| = 10 =
100M transitions.  metric = transitions refined / s = n * k * passes / time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 (torchrun): every rank minimises its own independent 100M-transition
DFA (independent objects, no data-path collective; "scaling": "weak"); the
step time is the max over ranks.

--impl reference times the reference's own CPU sort_pr (oracle/_ref, the
unmodified reference sources compiled in place) on a bounded sample of the
same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "transitions refined/sec"
UNIT = "transitions/s"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--states", type=int, default=10_000_000)
    p.add_argument("--alphabet", type=int, default=10)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--no-extras", action="store_true", help="skip the secondary configs")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_name(n, k):
    return f"sort_pr random DFA {n // 1_000_000}M states x |Sigma|={k} ({n * k // 1_000_000}M transitions)"


# --------------------------------------------------------------------------
# clocks: NVML sampled every few ms in a background thread during timing
# --------------------------------------------------------------------------

class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons = [], set()
        self.ok = False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel: str):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            j = json.load(f)
        return j["kernels"][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


# --------------------------------------------------------------------------
# CPU baseline: the reference's own sort_pr (oracle/_ref) on a bounded sample
# --------------------------------------------------------------------------

def reference_sample(n: int, k: int, seed: int):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    try:
        lib = pyoracle.RefLib()
        kind = "reference"
    except Exception:
        lib = pyoracle.COracle()
        kind = "port"
    gen = pyoracle.COracle()
    d, a, _ = gen.gen_synth(n, k, seed)
    return lib, kind, d, a


def time_reference_once(lib, d, a):
    t0 = time.perf_counter()
    r = lib.minimize("sort", d, a, want_blocks=False) if lib.kind == "reference" else lib.minimize("sort", d, a)
    dt = time.perf_counter() - t0
    n, k = d.shape[1], d.shape[0]
    return n * k * (r.refine_iters + 1) / dt, dt, r


def cpu_baseline(k: int, seed: int, budget_s: float = 20.0):
    n = 250_000
    lib, kind, d, a = reference_sample(n, k, seed)
    v, dt, r = time_reference_once(lib, d, a)
    # grow the sample toward ~budget/2 seconds of reference work
    while dt < budget_s / 6 and n < 4_000_000:
        n *= 2
        lib, kind, d, a = reference_sample(n, k, seed)
        v, dt, r = time_reference_once(lib, d, a)
    return {"value": v, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"reference sort_pr on synth DFA {n} states x |Sigma|={k} (same generator), "
                      f"{r.refine_iters + 1} passes, {dt:.2f} s, single-threaded (the reference is sequential)"}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    k = args.alphabet
    n = min(args.states, 1_000_000)
    lib, kind, d, a = reference_sample(n, k, args.seed)
    for _ in range(args.warmup):
        time_reference_once(lib, d, a)
    vals, secs = [], 0.0
    for _ in range(args.steps):
        v, dt, r = time_reference_once(lib, d, a)
        vals.append(v)
        secs += dt
    value = float(np.mean(vals))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * secs / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic", "impl": "reference",
            "config": {"workload": workload_name(args.states, k), "sample_states": n, "alphabet": k,
                       "passes": r.refine_iters + 1},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": kind,
                             "sample": f"reference sort_pr on synth DFA {n} states x |Sigma|={k} per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# B200 arm
# --------------------------------------------------------------------------

def run_b200(args, rank, world, local):
    import torch
    import paper_2508_20735_b200 as dk
    from paper_2508_20735_b200 import _native as nat

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ctx = dk.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream)
    n, k = args.states, args.alphabet
    delta = torch.empty(k * n, dtype=torch.int32, device="cuda")
    acc = torch.empty(n, dtype=torch.uint8, device="cuda")
    blocks = torch.empty(n, dtype=torch.int32, device="cuda")
    nat.check(nat.lib.dfakit_gen_synth_device(ctx.handle, n, k, args.seed + rank, delta.data_ptr(), acc.data_ptr(),
                                              ctx.stream))
    torch.cuda.synchronize()
    view = nat.CDfa(n, k, delta.data_ptr(), acc.data_ptr(), -1)
    opts = nat.COptions(0, 0, 0, 0, 0, 64, 0)
    rep = nat.CReport()

    def step():
        nat.check(nat.lib.dfakit_minimize_device(ctx.handle, C.byref(view), int(dk.Algorithm.sort_pr), C.byref(opts),
                                                 blocks.data_ptr(), C.byref(rep), ctx.stream))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = ctx.kernel_launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    barrier()
    launches = ctx.kernel_launches - launches0
    ms_total = max_over_ranks(ev0.elapsed_time(ev1))
    ms_step = ms_total / args.steps
    passes = int(rep.passes)
    transitions = n * k * passes
    value = transitions * world / (ms_step / 1000.0)

    # live per-kernel profile (event-bracketed launches on the library stream)
    # of the same steps, for the roofline of the dominant kernel
    nat.check(nat.lib.dfakit_profile_begin(ctx.handle))
    for _ in range(args.steps):
        step()
    buf = C.create_string_buffer(1 << 16)
    nat.check(nat.lib.dfakit_profile_end(ctx.handle, buf, len(buf)))
    kernels = json.loads(buf.value.decode())
    kernels.sort(key=lambda x: -x["ms"])
    top = kernels[0]
    peak, peak_src = measured_peaks()
    achieved = top["bytes"] / (top["ms"] / 1000.0) / 1e9 if top["ms"] > 0 else 0.0
    prof_ms = sum(x["ms"] for x in kernels)
    roofline = {"bound": "hbm", "kernel": top["name"], "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu_traffic(top["name"]),
                "algorithmic_bytes_per_launch": top["bytes"] / max(top["launches"], 1),
                "avg_launch_ms": top["ms"] / max(top["launches"], 1), "share_of_step": top["ms"] / prof_ms,
                "peak_source": peak_src,
                "kernels": [{"name": x["name"], "ms_per_step": x["ms"] / args.steps,
                             "launches_per_step": x["launches"] / args.steps,
                             "GBps": (x["bytes"] / (x["ms"] / 1000.0) / 1e9) if x["ms"] > 0 and x["bytes"] else None}
                            for x in kernels[:8]]}

    # end to end through the public host-buffer API (H2D + compute + D2H)
    h_delta = torch.empty(k * n, dtype=torch.int32, pin_memory=True)
    h_acc = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_blocks = torch.empty(n, dtype=torch.int32, pin_memory=True)
    h_delta.copy_(delta.cpu())
    h_acc.copy_(acc.cpu())
    hview = nat.CDfa(n, k, h_delta.data_ptr(), h_acc.data_ptr(), -1)

    def e2e_step():
        nat.check(nat.lib.dfakit_minimize(ctx.handle, C.byref(hview), int(dk.Algorithm.sort_pr), C.byref(opts),
                                          h_blocks.data_ptr(), C.byref(rep)))

    for _ in range(max(1, args.warmup)):
        e2e_step()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = max_over_ranks(time.perf_counter() - t0) / args.steps
    e2e = {"value": transitions * world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 4 * k * n + n,
           "d2h_bytes_per_step": 4 * n, "ms_per_step": e2e_s * 1000.0,
           "api": "dfakit_minimize (host buffers, pinned)"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": workload_name(n, k), "states": n, "alphabet": k, "transitions": n * k,
                       "algorithm": "sort_pr", "passes": passes, "refining_iterations": int(rep.refining_iterations),
                       "num_blocks": int(rep.num_blocks), "wall_ms_to_minimal_dfa": ms_step,
                       "states_sorted_per_step": int(rep.states_sorted),
                       "l2": "inputs larger than L2 (delta 400 MB per rank > 126 MB L2)",
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
            "roofline": roofline, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks.summary()}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(k, args.seed)
    if rank == 0 and world == 1 and not args.no_extras:
        line["extra"] = extras(dk, nat, ctx, torch)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def extras(dk, nat, ctx, torch):
    """Secondary BASELINE configs, device-resident, timed with CUDA events."""
    out = {}

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            r = fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps, r

    # configs[1]: sort vs naive splitting (naive needs ~0.4 n passes on random
    # DFAs, so it is measured on a 100K-state instance)
    n, k = 100_000, 10
    d = torch.empty(k * n, dtype=torch.int32, device="cuda")
    a = torch.empty(n, dtype=torch.uint8, device="cuda")
    b = torch.empty(n, dtype=torch.int32, device="cuda")
    nat.check(nat.lib.dfakit_gen_synth_device(ctx.handle, n, k, 7, d.data_ptr(), a.data_ptr(), ctx.stream))
    view = nat.CDfa(n, k, d.data_ptr(), a.data_ptr(), -1)
    for algo in ("sort_pr", "naive_pr", "naive_pr_fused"):
        rep = nat.CReport()
        opts = nat.COptions(0, 0, 0, 0, 0, 64, 0)

        def f():
            nat.check(nat.lib.dfakit_minimize_device(ctx.handle, C.byref(view), int(dk.Algorithm[algo]),
                                                     C.byref(opts), b.data_ptr(), C.byref(rep), ctx.stream))
            return rep

        s, r = timed(f, 2)
        out[f"{algo}_100K_k10"] = {"ms": s * 1000, "passes": int(r.passes), "blocks": int(r.num_blocks),
                                   "transitions_per_s": n * k * int(r.passes) / s}
    # configs[2]: chain DFA (n-pass worst case) with partial transitive closure
    n = 10_000_000
    d = torch.empty(n, dtype=torch.int32, device="cuda")
    a = torch.empty(n, dtype=torch.uint8, device="cuda")
    b = torch.empty(n, dtype=torch.int32, device="cuda")
    nat.check(nat.lib.dfakit_gen_chain_device(ctx.handle, n, d.data_ptr(), a.data_ptr(), ctx.stream))
    view = nat.CDfa(n, 1, d.data_ptr(), a.data_ptr(), 0)
    rep = nat.CReport()
    opts = nat.COptions(0, 0, 0, 1 << 40, 0, 64, 0)

    def g():
        nat.check(nat.lib.dfakit_minimize_device(ctx.handle, C.byref(view), int(dk.Algorithm.trans_pr),
                                                 C.byref(opts), b.data_ptr(), C.byref(rep), ctx.stream))
        return rep

    s, r = timed(g, 2)
    out["trans_pr_chain_10M"] = {"ms": s * 1000, "passes": int(r.passes), "closure_iterations": int(r.closure_iterations),
                                 "blocks": int(r.num_blocks)}
    # configs[3]: equivalence / inclusion of two 10M-state DFAs
    n, k = 10_000_000, 2
    d = torch.empty(k * n, dtype=torch.int32, device="cuda")
    a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(k * n, dtype=torch.int32, device="cuda")
    a2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    nat.check(nat.lib.dfakit_gen_synth_device(ctx.handle, n, k, 11, d.data_ptr(), a.data_ptr(), ctx.stream))
    init2 = C.c_uint32()
    nat.check(nat.lib.dfakit_permute_states_device(ctx.handle, n, k, 5, d.data_ptr(), a.data_ptr(), d2.data_ptr(),
                                                   a2.data_ptr(), C.byref(init2), ctx.stream))
    torch.cuda.synchronize()
    va = nat.CDfa(n, k, d.data_ptr(), a.data_ptr(), 0)
    vb = nat.CDfa(n, k, d2.data_ptr(), a2.data_ptr(), int(init2.value))
    cex = np.zeros(1 << 16, np.uint32)
    for name, fn in (("naive_hk", nat.lib.dfakit_explore_product_device),):
        res = nat.CProduct()

        def h():
            nat.check(fn(ctx.handle, C.byref(va), C.byref(vb), 0, None, 1 << 32, cex.ctypes.data, len(cex),
                         C.byref(res), ctx.stream))
            return res

        s, r = timed(h, 1)
        out[f"equiv_{name}_10M_equal"] = {"ms": s * 1000, "verdict": int(r.verdict),
                                          "explored_pairs": int(r.explored_states), "levels": int(r.levels),
                                          "pairs_per_s": int(r.explored_states) * k / s}
    res = nat.CProduct()

    def u():
        nat.check(nat.lib.dfakit_check_equiv_uf_device(ctx.handle, C.byref(va), C.byref(vb), cex.ctypes.data,
                                                       len(cex), C.byref(res), ctx.stream))
        return res

    s, r = timed(u, 1)
    out["equiv_union_find_10M_equal"] = {"ms": s * 1000, "verdict": int(r.verdict), "unions": int(r.explored_states),
                                         "levels": int(r.levels)}
    return out


def main():
    args = parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    run_b200(args, rank, world, local)


if __name__ == "__main__":
    main()
