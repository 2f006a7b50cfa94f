"""Sharded sort_pr on the GPU: the sm_100a shard primitives (CudaShardOps,
C ABI) under the sharded driver, against the oracle -- identical canonical
partition and refining-pass count.  World size 1 runs over NCCL; world size
2 runs two ranks on the one available GPU over gloo with host-staged
collectives (the NCCL path is the same driver with device tensors)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

CASES = [
    ("random", 300, 2, 0.5, 11),
    ("random", 5000, 3, 0.5, 12),
    ("random", 4000, 6, 0.9, 13),
    ("random", 20000, 10, 0.5, 14),
    ("copies", 400, 8, 0.5, 15),
    ("family", 7, 0, 0.0, 0),
    ("family", 12, 0, 0.0, 1),
    ("synth", 1_000_000, 10, 0.0, 3),
    # stable initial split {F, Q \ F}: refine_iters == 0 (the first pass is a
    # table pass that reaches the fixed point before any label exchange)
    ("random", 5000, 3, 1.0, 16),
    ("parity", 3000, 4, 0.0, 0),
    # classes of 3000 members: sub-buckets overflow (global-table fallback)
    ("bigcopies", 40, 8, 0.5, 17),
]


def make_case(case):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    o = pyoracle.COracle()
    kind, n, k, frac, seed = case
    if kind == "random":
        d, a, _ = o.gen_random(n, k, frac, seed)
    elif kind == "synth":
        d, a, _ = o.gen_synth(n, k, seed)
    elif kind == "parity":  # n copies of the 2-state parity automaton over k letters
        q = np.arange(2 * n, dtype=np.uint32)
        d = np.tile(q, (k, 1))
        d[0] ^= 1
        a = (q & 1).astype(np.uint8)
    elif kind in ("copies", "bigcopies"):
        base, acc0, _ = o.gen_random(n, k, frac, seed)
        c = 30 if kind == "copies" else 3000
        d = np.empty((k, n * c), np.uint32)
        for j in range(c):
            d[:, j * n:(j + 1) * n] = base + ((j + 1) % c) * n
        a = np.tile(acc0, c)
    else:
        d, a, _ = o.gen_family("bitsplit" if seed == 0 else "fib", n)
    return d, a, o.minimize("moore", d, a)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_cases(comm, dk, sharded):
    ctx = dk.Context(0)
    out = []
    for case in CASES:
        d, a, want = make_case(case)
        k, n = d.shape
        delta = torch.from_numpy(np.ascontiguousarray(d).view(np.int32).reshape(-1)).cuda()
        acc = torch.from_numpy(np.ascontiguousarray(a)).cuda()
        ops = sharded.CudaShardOps(ctx, delta, acc, n, k)
        blocks, rep = sharded.sort_pr_sharded(ops, comm, n, k)
        got = blocks.cpu().numpy().view(np.uint32)
        out.append((case, bool(np.array_equal(got, want.blocks)), rep.num_blocks == want.num_blocks,
                    rep.refining_iterations, want.refine_iters, rep.table_passes, rep.passes))
    return out


def check(rows):
    for case, same, nb, got, want, *_ in rows:
        assert same and nb and got == want, (case, got, want)
    assert any(tp > 0 for *_a, tp, p in rows) and any(p > tp for *_a, tp, p in rows)


def test_sharded_world1_nccl(dk):
    from paper_2508_20735_b200 import sharded
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        check(run_cases(sharded.TorchComm(), dk, sharded))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("peer", ["2", "0"], ids=["peer", "collectives"])
def test_sharded_native_driver_world1(dk, monkeypatch, peer):
    """The C++ pass loop over NCCL (dfakit_sort_pr_sharded), world size 1:
    peer mode (the comm's own buffers as the one peer) and the collective
    exchanges."""
    from paper_2508_20735_b200 import sharded
    monkeypatch.setenv("DFAKIT_SHARD_PEER", peer)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        ctx = dk.Context(0)
        comm = sharded.NativeComm(ctx)
        for case in CASES:
            d, a, want = make_case(case)
            k, n = d.shape
            delta = torch.from_numpy(np.ascontiguousarray(d).view(np.int32).reshape(-1)).cuda()
            acc = torch.from_numpy(np.ascontiguousarray(a)).cuda()
            blocks, rep = sharded.sort_pr_sharded_native(ctx, comm, delta, acc, n, k)
            got = blocks.cpu().numpy().view(np.uint32)
            assert np.array_equal(got, want.blocks) and rep.num_blocks == want.num_blocks, case
            assert rep.refining_iterations == want.refine_iters, (case, rep.refining_iterations, want.refine_iters)
        comm.close()
    finally:
        dist.destroy_process_group()


def worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        sys.path.insert(0, ROOT)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2508_20735_b200 as dk
        from paper_2508_20735_b200 import sharded
        q.put((rank, run_cases(sharded.TorchComm(stage_cpu=True), dk, sharded)))
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc()))


def test_sharded_world2_one_gpu(dk):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert not isinstance(res[r], str), res[r]
        check(res[r])


def run_hub(dk, world, d, a):
    """The native driver at `world` ranks as threads of this process (each
    with its own context on the one GPU, collectives through the in-process
    hub); returns every rank's (block_of, refining_iterations, num_blocks)."""
    import ctypes as C
    import threading
    from paper_2508_20735_b200 import _native as nat
    k, n = d.shape
    hub = C.c_void_p()
    nat.check(nat.lib.dfakit_local_hub_create(world, C.byref(hub)))
    out, errs = [None] * world, []

    def rank_main(r):
        try:
            ctx = dk.Context(0)
            comm = C.c_void_p()
            nat.check(nat.lib.dfakit_comm_init_local(hub, r, C.byref(comm)))
            delta = torch.from_numpy(np.ascontiguousarray(d).view(np.int32).reshape(-1)).cuda()
            acc = torch.from_numpy(np.ascontiguousarray(a)).cuda()
            blocks = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
            torch.cuda.synchronize()
            view = nat.CDfa(n, k, delta.data_ptr() if k else None, acc.data_ptr(), -1)
            rep = nat.CReport()
            nat.check(nat.lib.dfakit_sort_pr_sharded(ctx.handle, comm, C.byref(view), blocks.data_ptr(),
                                                     C.byref(rep), None, None))
            out[r] = (blocks[:n].cpu().numpy().view(np.uint32), int(rep.refining_iterations), int(rep.num_blocks))
            nat.lib.dfakit_comm_destroy(comm)
        except Exception as e:  # pragma: no cover - reported below
            errs.append((r, repr(e)))

    threads = [threading.Thread(target=rank_main, args=(r,), daemon=True) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    nat.lib.dfakit_local_hub_destroy(hub)
    assert not errs, (world, errs)
    return out


def check_hub(out, want, tag):
    for r, (blocks, iters, nb) in enumerate(out):
        assert np.array_equal(blocks, want.blocks) and nb == want.num_blocks, (tag, r)
        assert iters == want.refine_iters, (tag, r, iters, want.refine_iters)


@pytest.mark.parametrize("layout", ["owner", "owner-nccl", "staged", "owner-sliced"])
def test_native_driver_multirank_local_hub(dk, layout, monkeypatch):
    """The native C++ pass loop with world sizes 2 and 3 (ranks as threads on
    the one GPU; NCCL refuses two ranks on one device).  Every rank must
    return the oracle's partition and pass count -- through the owner-bucket
    layout in peer mode (the default: entries stored into the owners' receive
    regions and results into the senders' labels by the kernels themselves,
    here required), the owner layout with both exchanges as collectives, the
    staged-entries protocol, and sliced passes."""
    monkeypatch.setenv("DFAKIT_SHARD_PEER", "2")
    if layout == "owner-nccl":
        monkeypatch.setenv("DFAKIT_SHARD_PEER", "0")
    if layout == "staged":
        monkeypatch.setenv("DFAKIT_SHARD_STAGED", "1")
    if layout == "owner-sliced":  # signature passes gathered in label slices
        monkeypatch.setenv("DFAKIT_TEST_SLICE_BYTES", "4096")
    cases = [c for c in CASES if c[0] != "synth"] + [("synth", 300_000, 10, 0.0, 5)]
    for world in (2, 3):
        for case in cases:
            d, a, want = make_case(case)
            check_hub(run_hub(dk, world, d, a), want, (layout, world, case))


def test_native_driver_wide_worlds(dk, monkeypatch):
    """World sizes 5 and 8 (the owner-bucket layout's largest: sub-buckets of
    2048 / 8 = 256 slots, so heavy classes overflow into the fallback; peer
    mode required) and 9 (past it: the staged protocol)."""
    monkeypatch.setenv("DFAKIT_SHARD_PEER", "2")
    cases = [("random", 20000, 10, 0.5, 14), ("bigcopies", 40, 8, 0.5, 17), ("copies", 400, 8, 0.5, 15),
             ("family", 12, 0, 0.0, 1), ("synth", 200_000, 10, 0.0, 7)]
    for world in (5, 8, 9):
        for case in cases:
            d, a, want = make_case(case)
            check_hub(run_hub(dk, world, d, a), want, (world, case))


def test_cuda_ipc_mapping_two_processes(tmp_path):
    """The CUDA IPC calls of peer mode between two processes (on the one GPU
    here; between GPUs the same mapping rides NVLink): a buffer exported by
    one process is written by a kernel of the other through
    cudaIpcOpenMemHandle(..., cudaIpcMemLazyEnablePeerAccess)."""
    import subprocess
    exe = str(tmp_path / "ipc_check")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-o", exe,
                    os.path.join(ROOT, "tests", "cpp", "ipc_check.cu")], check=True)
    f = str(tmp_path / "handle")
    server = subprocess.Popen([exe, "serve", f], stdout=subprocess.PIPE, text=True)
    writer = subprocess.run([exe, "write", f], capture_output=True, text=True, timeout=180)
    out, _ = server.communicate(timeout=180)
    assert writer.returncode == 0 and writer.stdout.startswith("OK"), writer.stdout + writer.stderr
    assert server.returncode == 0 and out.startswith("OK"), out


def test_native_driver_tiny_automata_odd_worlds(dk, monkeypatch):
    """Peer mode at world sizes 4, 6 and 7 on automata smaller than the world
    (empty shards on some ranks) and on a few small odd shapes."""
    monkeypatch.setenv("DFAKIT_SHARD_PEER", "2")
    cases = [("random", 1, 1, 1.0, 21), ("random", 3, 2, 0.5, 22), ("random", 50, 3, 0.5, 23),
             ("copies", 5, 2, 0.5, 24), ("random", 3001, 7, 0.7, 25)]
    for world in (4, 6, 7):
        for case in cases:
            d, a, want = make_case(case)
            check_hub(run_hub(dk, world, d, a), want, (world, case))


def test_native_driver_packed_labels(dk, monkeypatch):
    """Wide passes gathering the carried 16-bit ranks packed 12 bits apiece
    (forced on small automata; sliced too): peer mode at worlds 1, 2 and 3."""
    monkeypatch.setenv("DFAKIT_SHARD_PEER", "2")
    monkeypatch.setenv("DFAKIT_PACK12_MIN_MB", "0")
    cases = [("random", 5000, 3, 0.5, 12), ("random", 20000, 10, 0.5, 14), ("copies", 400, 8, 0.5, 15),
             ("synth", 300_000, 10, 0.0, 5)]
    for world in (1, 2, 3):
        for case in cases:
            d, a, want = make_case(case)
            check_hub(run_hub(dk, world, d, a), want, (world, case))
    monkeypatch.setenv("DFAKIT_TEST_SLICE_BYTES", "4096")
    for case in cases[1:]:
        d, a, want = make_case(case)
        check_hub(run_hub(dk, 2, d, a), want, ("sliced", case))
