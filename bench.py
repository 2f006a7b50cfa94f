#!/usr/bin/env python
"""Benchmark: sort-based DFA minimisation (sortPR) on B200.

Step = one full sort_pr minimisation (every refinement pass up to and
including the confirming pass) of a synthetic random DFA resident in HBM.
Default workload (BASELINE.json configs[1]): 10M states x |Sigma| = 10 =
100M transitions.  metric = transitions refined / s = n * k * passes / time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N = 1: the single-GPU engine (dfakit_minimize_device).  N > 1: one rank per
GPU over NCCL -- launched by the driver under torchrun, or, when WORLD_SIZE
is unset, by this script re-executing itself under torch.distributed.run --
the native sharded engine on ONE automaton of N x 10M states (weak scaling:
100M transitions per GPU); per pass the label slices are allgathered and the
wide-key entries exchanged all-to-all over NVLink; the step time is the max
over ranks.  Beside the headline, `strong_scaling` times BASELINE configs[4]:
one fixed 100M x 10 (1B-transition) automaton on all N GPUs.

--impl reference times the reference's own CPU sort_pr (oracle/_ref, the
unmodified reference sources compiled in place) on a bounded sample of the
same workload, one independent minimisation per host core, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import re
import os
import socket
import subprocess
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
    p.add_argument("--engine", choices=["auto", "single", "sharded", "sharded-py"], default="auto",
                   help="auto: single-GPU engine at N = 1, the native (C++ / NCCL) sharded engine at N > 1")
    p.add_argument("--states", type=int, default=10_000_000, help="states per GPU")
    p.add_argument("--alphabet", type=int, default=10)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--no-extras", action="store_true", help="skip the secondary configs")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-strong", action="store_true", help="skip the configs[4] strong-scaling record")
    p.add_argument("--dry-run", action="store_true",
                   help="launcher check only (CPU, gloo): spawn / rendezvous / max-over-ranks, no device work")
    return p.parse_args()


def ensure_ranks(args):
    """`bench.py --gpus N` outside torchrun re-executes itself under
    torch.distributed.run with N ranks (one per GPU); under torchrun the
    world size must equal --gpus.  Returns only in a correctly sized rank."""
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None:
        if args.gpus <= 1:
            return
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
        sys.exit(subprocess.call(cmd, env=env))
    if int(world_env) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env} (launch one rank per GPU)")


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_name(n, k, world=1):
    s = f"sort_pr random DFA {n / 1e6:g}M states x |Sigma|={k} ({n * k / 1e6:g}M transitions)"
    return s + (f", sharded over {world} GPUs" if world > 1 else "")


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
    """DRAM bytes per launch of `kernel` from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            j = json.load(f)
        def norm(s):
            for tok in re.findall(r"[A-Za-z_]\w*", s):
                if tok.endswith("_kernel"):
                    return tok
            return s
        ks = {norm(name): v for name, v in j["kernels"].items()}
        k = ks[norm(kernel)]
        return k["dram_bytes_per_launch"], f"profiles/ncu_summary.json ({j['tag']}, {k['workload']} workload)"
    except Exception:
        return None, None


# --------------------------------------------------------------------------
# CPU side: the reference's own sort_pr (oracle/_ref) on bounded samples
# --------------------------------------------------------------------------

def reference_sample(n: int, k: int, seed: int):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    try:
        lib = pyoracle.RefLib()
    except Exception:
        lib = pyoracle.COracle()
    gen = pyoracle.COracle()
    d, a, _ = gen.gen_synth(n, k, seed)
    return lib, d, a


def time_reference_once(lib, d, a):
    t0 = time.perf_counter()
    r = lib.minimize("sort", d, a, want_blocks=False) if lib.kind == "reference" else lib.minimize("sort", d, a)
    dt = time.perf_counter() - t0
    n, k = d.shape[1], d.shape[0]
    return n * k * (r.refine_iters + 1), dt, r


def cpu_baseline(k: int, seed: int, budget_s: float = 20.0):
    """Single-threaded reference on one sample grown toward ~budget/6 s."""
    n = 250_000
    lib, d, a = reference_sample(n, k, seed)
    work, dt, r = time_reference_once(lib, d, a)
    while dt < budget_s / 6 and n < 4_000_000:
        n *= 2
        lib, d, a = reference_sample(n, k, seed)
        work, dt, r = time_reference_once(lib, d, a)
    return {"value": work / dt, "unit": UNIT, "cores": 1, "kind": lib.kind,
            "sample": f"reference sort_pr on synth DFA {n} states x |Sigma|={k} (same generator), "
                      f"{r.refine_iters + 1} passes, {dt:.2f} s, one thread (the reference is sequential)"}


def _ref_worker(args):
    n, k, seed, reps = args
    lib, d, a = reference_sample(n, k, seed)
    out = []
    for _ in range(reps):
        out.append(time_reference_once(lib, d, a)[:2])
    return lib.kind, out


def run_reference_arm(args, rank, world):
    """The reference sort_pr is sequential: every host core minimises its own
    1M-state sample of the workload concurrently; value = all transitions
    refined / wall time of the timed steps."""
    if rank != 0:
        return
    import multiprocessing as mp
    k = args.alphabet
    n = min(args.states, 1_000_000)
    cores = max(1, min(len(os.sched_getaffinity(0)), 64))
    with mp.get_context("fork").Pool(cores) as pool:
        pool.map(_ref_worker, [(n, k, args.seed + c, max(1, args.warmup)) for c in range(cores)])
        t0 = time.perf_counter()
        res = pool.map(_ref_worker, [(n, k, args.seed + c, args.steps) for c in range(cores)])
        wall = time.perf_counter() - t0
    kind = res[0][0]
    work = sum(w for _, runs in res for w, _ in runs)
    value = work / wall
    passes = int(round(res[0][1][0][0] / (n * k)))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * wall / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic", "impl": "reference",
            "config": {"workload": workload_name(args.states * max(1, args.gpus), k, args.gpus), "sample_states": n,
                       "alphabet": k, "passes": passes, "cores": cores},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": f"reference sort_pr, one {n}-state x |Sigma|={k} synth DFA per core per step "
                                       f"({cores} concurrent processes)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# B200 arm
# --------------------------------------------------------------------------

def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def profile_kernels(nat, ctx, run, steps):
    """Live per-kernel profile (CUDA events around every library launch on
    its stream) over `steps` repetitions of `run`."""
    nat.check(nat.lib.dfakit_profile_begin(ctx.handle))
    for _ in range(steps):
        run()
    buf = C.create_string_buffer(1 << 16)
    nat.check(nat.lib.dfakit_profile_end(ctx.handle, buf, len(buf)))
    kernels = json.loads(buf.value.decode())
    kernels.sort(key=lambda x: -x["ms"])
    return kernels


def split_passes(kernels):
    """The profiler's per-kernel entries and its per-pass sums ("#pass N")."""
    return ([x for x in kernels if not x["name"].startswith("#")],
            sorted((x for x in kernels if x["name"].startswith("#pass")), key=lambda x: int(x["name"].split()[1])))


def roofline_of(kernels, steps, gather_peak, n):
    kernels, passes = split_passes(kernels)
    top = kernels[0]
    peak, peak_src = measured_peaks()
    achieved = top["bytes"] / (top["ms"] / 1000.0) / 1e9 if top["ms"] > 0 else 0.0
    prof_ms = sum(x["ms"] for x in kernels)
    g = [x for x in kernels if x.get("units")]
    gather = None
    if g and gather_peak:
        gk = g[0]
        rate = gk["units"] / (gk["ms"] / 1000.0)
        gather = {"kernel": gk["name"], "achieved_gathers_per_s": rate, "peak_gathers_per_s": gather_peak,
                  "frac": rate / gather_peak,
                  "peak_source": f"dfakit_calibrate_gather: random 32-bit gathers from an {n}-entry table, "
                                 "every SM busy, measured in this run",
                  "all_gather_kernels": [{"name": x["name"], "gathers_per_s": x["units"] / (x["ms"] / 1000.0),
                                          "frac": x["units"] / (x["ms"] / 1000.0) / gather_peak} for x in g]}
    traffic, traffic_src = ncu_traffic(top["name"])
    return {"bound": "hbm", "kernel": top["name"], "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
            "algorithmic_bytes_per_launch": top["bytes"] / max(top["launches"], 1),
            "avg_launch_ms": top["ms"] / max(top["launches"], 1), "share_of_step": top["ms"] / prof_ms,
            "peak_source": peak_src,
            "binding_resource": "L1TEX/L2 line rate of the random block-label gathers (one 128-byte line per "
                                "lane); see gather_roofline and profiles/",
            "gather_roofline": gather,
            # north_star's target is per refinement pass: algorithmic bytes of
            # the pass's kernels / their summed device time (host gaps excluded)
            "per_pass": [{"pass": int(x["name"].split()[1]), "ms": x["ms"] / steps,
                          "algorithmic_bytes": x["bytes"] / steps,
                          "GBps": x["bytes"] / (x["ms"] / 1000.0) / 1e9 if x["ms"] > 0 else None,
                          "frac_hbm": x["bytes"] / (x["ms"] / 1000.0) / 1e9 / peak if x["ms"] > 0 else None,
                          "gathers_per_s": x["units"] / (x["ms"] / 1000.0) if x["ms"] > 0 else None,
                          "frac_gather_ceiling": (x["units"] / (x["ms"] / 1000.0) / gather_peak
                                                  if x["ms"] > 0 and gather_peak else None)}
                         for x in passes],
            "kernels": [{"name": x["name"], "ms_per_step": x["ms"] / steps, "launches_per_step": x["launches"] / steps,
                         "GBps": (x["bytes"] / (x["ms"] / 1000.0) / 1e9) if x["ms"] > 0 and x["bytes"] else None}
                        for x in kernels[:10]]}


def run_b200(args, rank, world, local):
    import torch
    import paper_2508_20735_b200 as dk
    from paper_2508_20735_b200 import _native as nat
    from paper_2508_20735_b200 import sharded

    if torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: --gpus {world} needs {world} visible devices, found {torch.cuda.device_count()}")
    torch.cuda.set_device(local)
    engine = args.engine if args.engine != "auto" else ("single" if world == 1 else "sharded")
    import torch.distributed as dist
    if world > 1 or engine.startswith("sharded"):
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        use_dist = True
    else:
        use_dist = False

    def barrier():
        if use_dist:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if not use_dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ctx = dk.Context(local)
    lib_stream = torch.cuda.ExternalStream(ctx.stream)
    k = args.alphabet
    sharded_engine = engine.startswith("sharded")
    n = args.states * (world if sharded_engine else 1)
    delta = torch.empty(k * n, dtype=torch.int32, device="cuda")
    acc = torch.empty(n, dtype=torch.uint8, device="cuda")
    blocks = torch.empty(n, dtype=torch.int32, device="cuda")
    # the same automaton on every rank (replicated input of the sharded engine);
    # the single-GPU engine's replicas minimise their own seeds
    gseed = args.seed if sharded_engine else args.seed + rank
    nat.check(nat.lib.dfakit_gen_synth_device(ctx.handle, n, k, gseed, delta.data_ptr(), acc.data_ptr(), ctx.stream))
    torch.cuda.synchronize()
    opts = nat.COptions(0, 0, 0, 0, 0, 64, 0)
    rep = nat.CReport()
    state = {}

    if engine == "single":
        view = nat.CDfa(n, k, delta.data_ptr(), acc.data_ptr(), -1)

        def step():
            nat.check(nat.lib.dfakit_minimize_device(ctx.handle, C.byref(view), int(dk.Algorithm.sort_pr),
                                                     C.byref(opts), blocks.data_ptr(), C.byref(rep), ctx.stream))
            state["passes"], state["iters"], state["blocks"] = int(rep.passes), int(rep.refining_iterations), \
                int(rep.num_blocks)
    elif engine == "sharded":
        ncomm = sharded.NativeComm(ctx)

        def step():
            b, r = sharded.sort_pr_sharded_native(ctx, ncomm, delta, acc, n, k, out=blocks)
            state["passes"], state["iters"], state["blocks"] = r.passes, r.refining_iterations, r.num_blocks
            state["exchanged"] = r.exchanged_entries
            state["out"] = b
    else:
        comm = sharded.TorchComm()
        ops = sharded.CudaShardOps(ctx, delta, acc, n, k)

        def step():
            b, r = sharded.sort_pr_sharded(ops, comm, n, k)
            state["passes"], state["iters"], state["blocks"] = r.passes, r.refining_iterations, r.num_blocks
            state["exchanged"] = r.exchanged_entries
            state["out"] = b

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = ctx.kernel_launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    timing_stream = lib_stream if engine == "single" else torch.cuda.current_stream()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        ev0.record(timing_stream)
        for _ in range(args.steps):
            step()
        ev1.record(timing_stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    barrier()
    launches = (ctx.kernel_launches - launches0)
    ms_total = max_over_ranks(ev0.elapsed_time(ev1))
    ms_step = ms_total / args.steps
    passes = state["passes"]
    transitions = n * k * passes  # the whole automaton's transitions, every pass
    value = transitions * (1 if sharded_engine else world) / (ms_step / 1000.0)

    # measured ceiling of the random label gathers, then the live per-kernel profile
    gather_peak = C.c_double(0)
    nat.check(nat.lib.dfakit_calibrate_gather(ctx.handle, n, 4, 200_000_000, C.byref(gather_peak)))
    kernels = profile_kernels(nat, ctx, step, args.steps)
    roofline = roofline_of(kernels, args.steps, gather_peak.value, n)

    # end to end through the public API with host buffers (H2D + compute + D2H)
    h_delta = torch.empty(k * n, dtype=torch.int32, pin_memory=True)
    h_acc = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_blocks = torch.empty(n, dtype=torch.int32, pin_memory=True)
    h_delta.copy_(delta.cpu())
    h_acc.copy_(acc.cpu())
    if engine == "single":
        hview = nat.CDfa(n, k, h_delta.data_ptr(), h_acc.data_ptr(), -1)

        def e2e_step():
            nat.check(nat.lib.dfakit_minimize(ctx.handle, C.byref(hview), int(dk.Algorithm.sort_pr), C.byref(opts),
                                              h_blocks.data_ptr(), C.byref(rep)))
        h2d, d2h, api = 4 * k * n + n, 4 * n, "dfakit_minimize (host buffers, pinned)"
    else:
        def e2e_step():
            delta.copy_(h_delta, non_blocking=True)
            acc.copy_(h_acc, non_blocking=True)
            step()
            if rank == 0:
                h_blocks.copy_(state["out"], non_blocking=True)
            torch.cuda.synchronize()
        h2d, d2h, api = 4 * k * n + n, 4 * n if rank == 0 else 0, \
            f"sharded engine ({engine}; inputs copied from pinned host memory on every rank)"
    for _ in range(max(1, args.warmup)):
        e2e_step()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0) / args.steps
    e2e_transitions = transitions * (1 if sharded_engine else world)
    e2e = {"value": e2e_transitions / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "ms_per_step": e2e_s * 1000.0, "api": api}
    if rank == 0:
        e2e["pcie"] = pcie_bound(torch, h_delta, delta, h_blocks, blocks, h2d, d2h, e2e_s)

    cfg = {"workload": workload_name(n, k, world if sharded_engine else 1), "states": n, "alphabet": k,
           "transitions": n * k, "algorithm": "sort_pr", "engine": engine, "passes": passes,
           "refining_iterations": state["iters"], "num_blocks": state["blocks"], "wall_ms_to_minimal_dfa": ms_step,
           "l2": f"inputs larger than L2 (delta {4 * k * n / 1e6:.0f} MB per rank > 126 MB L2)",
           "parallelism": (f"sharded x{world} (NCCL all-to-all + label allgather per pass)" if sharded_engine
                           else (f"replicas x{world}" if world > 1 else "single GPU"))}
    if sharded_engine:
        ex = state.get("exchanged", 0)
        # per rank and step over NVLink: 16 B out + 4 B back per exchanged entry,
        # plus the label allgather (4 B per state and pass, all but the own slice)
        nv_bytes = 20 * ex + 4 * n * (world - 1) / world * max(state["iters"], 1)
        cfg["entries_exchanged_per_step_rank0"] = ex
        if world > 1:
            cfg["nvlink"] = {"bytes_per_rank_per_step": nv_bytes, "GBps_per_rank": nv_bytes / (ms_step / 1000.0) / 1e9,
                             "peak_GBps": 770.0, "frac": nv_bytes / (ms_step / 1000.0) / 1e9 / 770.0,
                             "peak_source": "B200_PROFILING.md measured peer copy per direction"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic", "config": cfg, "roofline": roofline, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clocks.summary()}

    # free the headline automaton before the configs[4] record
    del delta, acc, blocks, h_delta, h_acc, h_blocks
    if sharded_engine:
        state.pop("out", None)
    if engine == "sharded":
        ncomm.close()
    torch.cuda.empty_cache()
    if not args.no_strong:
        line["strong_scaling"] = strong_scaling_1b(args, dk, nat, sharded, torch, ctx, rank, world, barrier,
                                                   max_over_ranks)

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(k, args.seed)
    if rank == 0 and world == 1 and not args.no_extras:
        line["extra"] = extras(dk, nat, ctx, torch, sharded, args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.destroy_process_group()


def strong_scaling_1b(args, dk, nat, sharded, torch, ctx, rank, world, barrier, max_over_ranks):
    """BASELINE configs[4]: ONE fixed 1B-transition automaton (100M states x
    |Sigma| = 10, the bench generator) minimised on all N GPUs -- strong
    scaling.  N = 1: the single-GPU engine (and the native sharded engine at
    world size 1 beside it); N > 1: the native sharded engine over NCCL, the
    automaton replicated on every rank, states sharded in contiguous ranges.
    Device time with CUDA events, max over ranks."""
    n, k = 100_000_000, 10
    steps = max(1, min(args.steps, 5))
    d = torch.empty(k * n, dtype=torch.int32, device="cuda")
    a = torch.empty(n, dtype=torch.uint8, device="cuda")
    b = torch.empty(n, dtype=torch.int32, device="cuda")
    nat.check(nat.lib.dfakit_gen_synth_device(ctx.handle, n, k, args.seed, d.data_ptr(), a.data_ptr(), ctx.stream))
    torch.cuda.synchronize()
    st = {}
    rep = nat.CReport()
    opts = nat.COptions(0, 0, 0, 0, 0, 64, 0)
    view = nat.CDfa(n, k, d.data_ptr(), a.data_ptr(), -1)

    def single():
        nat.check(nat.lib.dfakit_minimize_device(ctx.handle, C.byref(view), int(dk.Algorithm.sort_pr), C.byref(opts),
                                                 b.data_ptr(), C.byref(rep), ctx.stream))
        st["passes"], st["iters"], st["blocks"] = int(rep.passes), int(rep.refining_iterations), int(rep.num_blocks)

    ncomm = sharded.NativeComm(ctx) if world > 1 else None

    def shard(comm):
        def f():
            _, r = sharded.sort_pr_sharded_native(ctx, comm, d, a, n, k, out=b)
            st["passes"], st["iters"], st["blocks"] = r.passes, r.refining_iterations, r.num_blocks
            st["exchanged"] = r.exchanged_entries
        return f

    stream = torch.cuda.ExternalStream(ctx.stream)

    def timeit(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1)) / steps

    out = {"workload": "sort_pr random DFA 100M states x |Sigma|=10 (1000M transitions), BASELINE configs[4]",
           "scaling": "strong", "n_gpus": world, "steps": steps, "warmup": 2}
    if world == 1:
        ms = timeit(single)
        out["engine"] = "single"
        import torch.distributed as dist
        own_pg = not dist.is_initialized()
        if own_pg:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ["MASTER_PORT"] = str(free_port())
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", ctx.device))
        c1 = sharded.NativeComm(ctx)
        out["sharded_native_world1_ms"] = timeit(shard(c1))
        c1.close()
        if own_pg:
            dist.destroy_process_group()
    else:
        ms = timeit(shard(ncomm))
        out["engine"] = "sharded (native, NCCL)"
        ex = st.get("exchanged", 0)
        nv = 20 * ex + 4 * n * (world - 1) / world * max(st["iters"], 1)
        out["nvlink"] = {"bytes_per_rank_per_step": nv, "GBps_per_rank": nv / (ms / 1000.0) / 1e9, "peak_GBps": 770.0,
                         "frac": nv / (ms / 1000.0) / 1e9 / 770.0,
                         "peak_source": "B200_PROFILING.md measured peer copy per direction"}
        ncomm.close()
    out.update({"ms_per_step": ms, "passes": st["passes"], "refining_iterations": st["iters"],
                "num_blocks": st["blocks"], "value": n * k * st["passes"] / (ms / 1000.0), "unit": UNIT})
    del d, a, b
    torch.cuda.empty_cache()
    return out


def pcie_bound(torch, h_in, d_in, h_out, d_out, h2d, d2h, e2e_s):
    """The e2e step's transfer floor, measured in the same run: plain pinned
    copies of the step's input (H2D) and result (D2H) buffers, CUDA events on
    a side stream.  ms_floor = the step's bytes at those rates; frac = floor /
    e2e step time (how much of the e2e step is the PCIe link itself)."""
    s = torch.cuda.Stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    best_in = best_out = float("inf")
    with torch.cuda.stream(s):
        for _ in range(3):
            ev[0].record(s)
            d_in.copy_(h_in, non_blocking=True)
            ev[1].record(s)
            h_out.copy_(d_out, non_blocking=True)
            ev[2].record(s)
            ev[2].synchronize()
            best_in = min(best_in, ev[0].elapsed_time(ev[1]))
            best_out = min(best_out, ev[1].elapsed_time(ev[2]))
    h2d_gbps = h_in.numel() * h_in.element_size() / (best_in / 1000.0) / 1e9
    d2h_gbps = h_out.numel() * h_out.element_size() / (best_out / 1000.0) / 1e9
    floor_ms = (h2d / h2d_gbps + d2h / d2h_gbps) / 1e6
    return {"h2d_GBps": h2d_gbps, "d2h_GBps": d2h_gbps, "transfer_floor_ms": floor_ms,
            "frac_of_e2e_step": floor_ms / (e2e_s * 1000.0)}


def extras(dk, nat, ctx, torch, sharded, args):
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

    def minimize(view, algo, b, opts=None):
        rep = nat.CReport()
        opts = opts or nat.COptions(0, 0, 0, 1 << 40, 0, 64, 0)

        def f():
            nat.check(nat.lib.dfakit_minimize_device(ctx.handle, C.byref(view), int(dk.Algorithm[algo]),
                                                     C.byref(opts), b.data_ptr(), C.byref(rep), ctx.stream))
            return rep
        return f

    # configs[0]: random complete DFA, 1M states, |Sigma| = 2, from the
    # reference's own generator (gen_random, libstdc++ mt19937_64), minimised
    # on the GPU and by the reference (oracle/_ref, one thread) -- same input,
    # same partition
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    gen = pyoracle.COracle()
    hd, ha, _ = gen.gen_random(1_000_000, 2, 0.5, 7)
    n, k = hd.shape[1], hd.shape[0]
    d = torch.from_numpy(np.ascontiguousarray(hd).view(np.int32).reshape(-1)).cuda()
    a = torch.from_numpy(np.ascontiguousarray(ha)).cuda()
    b = torch.empty(n, dtype=torch.int32, device="cuda")
    view = nat.CDfa(n, k, d.data_ptr(), a.data_ptr(), -1)
    s, r = timed(minimize(view, "sort_pr", b), 5)
    c0 = {"ms": s * 1000, "passes": int(r.passes), "refining_iterations": int(r.refining_iterations),
          "blocks": int(r.num_blocks), "transitions_per_s": n * k * int(r.passes) / s}
    try:
        ref = pyoracle.RefLib()
        t0 = time.perf_counter()
        rr = ref.minimize("sort", hd, ha)
        c0["reference_ms"] = (time.perf_counter() - t0) * 1000
        c0["reference_kind"] = "reference (oracle/_ref, one thread)"
        c0["same_partition"] = bool(np.array_equal(b.cpu().numpy().view(np.uint32), rr.blocks)
                                    and rr.refine_iters == int(r.refining_iterations))
        c0["speedup_vs_reference"] = c0["reference_ms"] / c0["ms"]
    except Exception as e:  # the compiled reference is optional on the box
        c0["reference_ms"] = None
        c0["reference_note"] = f"oracle/_ref unavailable: {e}"
    out["sort_pr_config0_1M_k2"] = c0
    del d, a, b
    # configs[1] at full size: the literal Alg. 4 grouping (full LSD radix sort
    # of the keys + adjacent difference + scan) beside the default
    n, k = args.states, args.alphabet
    d = torch.empty(k * n, dtype=torch.int32, device="cuda")
    a = torch.empty(n, dtype=torch.uint8, device="cuda")
    b = torch.empty(n, dtype=torch.int32, device="cuda")
    nat.check(nat.lib.dfakit_gen_synth_device(ctx.handle, n, k, args.seed, d.data_ptr(), a.data_ptr(), ctx.stream))
    view = nat.CDfa(n, k, d.data_ptr(), a.data_ptr(), -1)
    s, r = timed(minimize(view, "sort_pr", b, nat.COptions(0, 0, 0, 0, 0, 64, 1)), 3)
    out["sort_pr_radix_sort_grouping_10M_k10"] = {"ms": s * 1000, "passes": int(r.passes),
                                                  "transitions_per_s": n * k * int(r.passes) / s}
    # the sharded engines at world size 1 (their per-pass exchange logic, no peers)
    import torch.distributed as dist
    own_pg = not dist.is_initialized()
    if own_pg:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(free_port())
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", ctx.device))
    comm = sharded.TorchComm()
    ops = sharded.CudaShardOps(ctx, d, a, n, k)
    s, (bl, rr) = timed(lambda: sharded.sort_pr_sharded(ops, comm, n, k), 3)
    out["sort_pr_sharded_py_world1_10M_k10"] = {"ms": s * 1000, "passes": rr.passes,
                                                "transitions_per_s": n * k * rr.passes / s}
    ncomm = sharded.NativeComm(ctx)
    s, (bl, rr) = timed(lambda: sharded.sort_pr_sharded_native(ctx, ncomm, d, a, n, k, out=b), 3)
    out["sort_pr_sharded_native_world1_10M_k10"] = {"ms": s * 1000, "passes": rr.passes,
                                                    "transitions_per_s": n * k * rr.passes / s}
    ncomm.close()
    if own_pg:
        dist.destroy_process_group()
    del d, a, b, ops
    torch.cuda.empty_cache()
    # configs[1]: sort vs naive splitting (naive needs ~0.4 n passes on random
    # DFAs, so it is measured on a 100K-state instance)
    n, k = 100_000, 10
    d = torch.empty(k * n, dtype=torch.int32, device="cuda")
    a = torch.empty(n, dtype=torch.uint8, device="cuda")
    b = torch.empty(n, dtype=torch.int32, device="cuda")
    nat.check(nat.lib.dfakit_gen_synth_device(ctx.handle, n, k, 7, d.data_ptr(), a.data_ptr(), ctx.stream))
    view = nat.CDfa(n, k, d.data_ptr(), a.data_ptr(), -1)
    for algo in ("sort_pr", "naive_pr", "naive_pr_fused"):
        s, r = timed(minimize(view, algo, b), 2)
        out[f"{algo}_100K_k10"] = {"ms": s * 1000, "passes": int(r.passes), "blocks": int(r.num_blocks),
                                   "transitions_per_s": n * k * int(r.passes) / s}
    # ... and at 20K states through the compiled reference too (one thread),
    # sort vs naive on identical input (the reference's naive_pr at 100K
    # states would take minutes)
    n, k = 20_000, 10
    hd, ha, _ = gen.gen_synth(n, k, 7)
    d = torch.from_numpy(np.ascontiguousarray(hd).view(np.int32).reshape(-1)).cuda()
    a = torch.from_numpy(np.ascontiguousarray(ha)).cuda()
    b = torch.empty(n, dtype=torch.int32, device="cuda")
    view = nat.CDfa(n, k, d.data_ptr(), a.data_ptr(), -1)
    for algo, ralgo in (("sort_pr", "sort"), ("naive_pr", "naive"), ("naive_pr_fused", "naive-fused")):
        s, r = timed(minimize(view, algo, b), 2)
        e = {"ms": s * 1000, "passes": int(r.passes)}
        try:
            t0 = time.perf_counter()
            rr = pyoracle.RefLib().minimize(ralgo, hd, ha)
            e["reference_ms"] = (time.perf_counter() - t0) * 1000
            e["same_partition"] = bool(np.array_equal(b.cpu().numpy().view(np.uint32), rr.blocks)
                                       and rr.refine_iters == int(r.refining_iterations))
            e["speedup_vs_reference"] = e["reference_ms"] / e["ms"]
        except Exception as ex:
            e["reference_note"] = f"oracle/_ref unavailable: {ex}"
        out[f"{algo}_20K_k10_vs_reference"] = e
    del d, a, b
    # configs[2]: chain DFA (n-pass worst case) with partial transitive closure
    n = 10_000_000
    d = torch.empty(n, dtype=torch.int32, device="cuda")
    a = torch.empty(n, dtype=torch.uint8, device="cuda")
    b = torch.empty(n, dtype=torch.int32, device="cuda")
    nat.check(nat.lib.dfakit_gen_chain_device(ctx.handle, n, d.data_ptr(), a.data_ptr(), ctx.stream))
    view = nat.CDfa(n, 1, d.data_ptr(), a.data_ptr(), 0)
    s, r = timed(minimize(view, "trans_pr", b), 2)
    out["trans_pr_chain_10M"] = {"ms": s * 1000, "passes": int(r.passes),
                                 "closure_iterations": int(r.closure_iterations), "blocks": int(r.num_blocks)}
    # configs[2] shape at 1M states on both sides: trans_pr on the GPU and the
    # reference's trans_pr (oracle/_ref, one thread) on the same chain
    hd, ha, _ = gen.gen_chain(1_000_000)
    n1 = hd.shape[1]
    d = torch.from_numpy(np.ascontiguousarray(hd).view(np.int32).reshape(-1)).cuda()
    a = torch.from_numpy(np.ascontiguousarray(ha)).cuda()
    b = torch.empty(n1, dtype=torch.int32, device="cuda")
    view = nat.CDfa(n1, 1, d.data_ptr(), a.data_ptr(), 0)
    s, r = timed(minimize(view, "trans_pr", b), 3)
    c2 = {"ms": s * 1000, "passes": int(r.passes), "closure_iterations": int(r.closure_iterations),
          "blocks": int(r.num_blocks)}
    try:
        t0 = time.perf_counter()
        rr = pyoracle.RefLib().minimize("transpr", hd, ha)
        c2["reference_ms"] = (time.perf_counter() - t0) * 1000
        c2["reference_kind"] = "reference (oracle/_ref, one thread)"
        c2["same_partition"] = bool(np.array_equal(b.cpu().numpy().view(np.uint32), rr.blocks)
                                    and rr.refine_iters == int(r.refining_iterations))
        c2["speedup_vs_reference"] = c2["reference_ms"] / c2["ms"]
    except Exception as e:
        c2["reference_note"] = f"oracle/_ref unavailable: {e}"
    out["trans_pr_chain_1M_vs_reference"] = c2
    del d, a, b
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
    for mode, name in ((0, "equivalence"), (1, "inclusion")):
        res = nat.CProduct()

        def h():
            nat.check(nat.lib.dfakit_explore_product_device(ctx.handle, C.byref(va), C.byref(vb), mode, None, 1 << 32,
                                                            cex.ctypes.data, len(cex), C.byref(res), ctx.stream))
            return res

        s, r = timed(h, 1)
        out[f"{name}_naive_hk_10M_equal"] = {"ms": s * 1000, "verdict": int(r.verdict),
                                             "explored_pairs": int(r.explored_states), "levels": int(r.levels),
                                             "pairs_per_s": int(r.explored_states) / s}
    # the same pair through the reference's explore_product (oracle/_ref, one
    # thread): pairs / s on identical inputs, verdict and counts compared
    try:
        ref = pyoracle.RefLib()
        hA = (d.cpu().numpy().view(np.uint32).reshape(k, n), a.cpu().numpy(), 0)
        hB = (d2.cpu().numpy().view(np.uint32).reshape(k, n), a2.cpu().numpy(), int(init2.value))
        t0 = time.perf_counter()
        ro = ref.explore("equivalence", hA, hB)
        dt = time.perf_counter() - t0
        g = out["equivalence_naive_hk_10M_equal"]
        out["equivalence_reference_10M_equal"] = {
            "ms": dt * 1000, "verdict": ro.verdict, "explored_pairs": ro.explored, "levels": ro.levels,
            "pairs_per_s": ro.explored / dt, "kind": "reference (oracle/_ref, one thread)",
            "same_result": ro.explored == g["explored_pairs"] and ro.levels == g["levels"] and g["verdict"] == 0,
            "gpu_speedup": dt * 1000 / g["ms"]}
    except Exception as e:  # the compiled reference is optional on the box
        out["equivalence_reference_10M_equal"] = {"note": f"oracle/_ref unavailable: {e}"}
    res = nat.CProduct()

    def u():
        nat.check(nat.lib.dfakit_check_equiv_uf_device(ctx.handle, C.byref(va), C.byref(vb), cex.ctypes.data,
                                                       len(cex), C.byref(res), ctx.stream))
        return res

    s, r = timed(u, 1)
    out["equiv_union_find_10M_equal"] = {"ms": s * 1000, "verdict": int(r.verdict), "unions": int(r.explored_states),
                                         "levels": int(r.levels), "pairs_per_s": int(r.explored_states) / s}
    # ... and differing: B's flag flipped at the state 30 letters-0 from its
    # initial state (so a counterexample of length <= 30 exists)
    qb = int(init2.value)
    for _ in range(30):
        qb = int(d2[qb].item())
    a2[qb] ^= 1
    torch.cuda.synchronize()
    for mode, name in ((0, "equivalence"), (1, "inclusion")):
        res = nat.CProduct()

        def h():
            nat.check(nat.lib.dfakit_explore_product_device(ctx.handle, C.byref(va), C.byref(vb), mode, None, 1 << 32,
                                                            cex.ctypes.data, len(cex), C.byref(res), ctx.stream))
            return res

        s, r = timed(h, 1)
        out[f"{name}_naive_hk_10M_differing"] = {"ms": s * 1000, "verdict": int(r.verdict),
                                                 "explored_pairs": int(r.explored_states), "levels": int(r.levels),
                                                 "counterexample_len": int(r.counterexample_len),
                                                 "pairs_per_s": int(r.explored_states) / s}
    s, r = timed(u, 1)
    out["equiv_union_find_10M_differing"] = {"ms": s * 1000, "verdict": int(r.verdict),
                                             "unions": int(r.explored_states), "levels": int(r.levels),
                                             "pairs_per_s": int(r.explored_states) / s}
    return out


def run_dry(args, rank, world):
    """Launcher check without a device: every rank joins a gloo group, the
    step time is reduced MAX over ranks, rank 0 prints the line skeleton."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    t0 = time.perf_counter()
    time.sleep(0.01 * (rank + 1))
    ms = torch.tensor([(time.perf_counter() - t0) * 1000.0], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": float(ms[0]), "impl": args.impl, "dry_run": True}),
              flush=True)


def main():
    # one JSON line on stdout: keep NCCL's version banner off it
    if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"
    args = parse_args()
    ensure_ranks(args)
    rank, world, local = dist_env()
    if args.dry_run:
        run_dry(args, rank, world)
        return
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    run_b200(args, rank, world, local)


if __name__ == "__main__":
    main()
