"""BASELINE configs[4] size, pinned to the oracle bit-exactly: a
1B-transition automaton (100M states x |Sigma| = 10) whose minimal partition
is known exactly without running the oracle at 100M states.

The automaton is c = 10 relabelled copies of the 10M x 10 bench automaton
(oracle generator `or_gen_synth`, seed 1): copy j's state q is state
j * n0 + pi_j(q) (pi_0 = identity, pi_j random permutations), and copy j
steps into copy j + 1 (mod c).  Every copy accepts the same language from
"the same" state, so the equivalence classes are the base's classes lifted
to all copies, every refinement round of the copied automaton is the base's
round lifted (identical refining-pass count), and -- because copy 0 holds
the smallest state ids, in base order -- its canonical numbering (minimum
state id per block, first-occurrence order) is the base's:
    block_of[j * n0 + pi_j(q)] == base_block_of[q].
The oracle therefore runs only on the 10M-state base.  An engine that
over-splits (separates copies) or under-splits fails the comparison.

Checked: the single-GPU engine (default grouping and the literal radix-sort
grouping), the native sharded engine at world size 1 over NCCL, and at world
sizes 2 and 4 with the ranks as threads sharing the one GPU (collectives
through the in-process hub, entries and results through peer memory)."""
import ctypes as C
import os
import socket
import threading

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N0, K, COPIES, SEED = 10_000_000, 10, 10, 1


@pytest.fixture(scope="module")
def instance(oracle):
    d0, a0, _ = oracle.gen_synth(N0, K, SEED)
    want = oracle.minimize("moore", d0, a0)
    dev = torch.device("cuda", 0)
    base_d = torch.from_numpy(np.ascontiguousarray(d0).view(np.int32)).to(dev).long()   # [K, N0]
    base_a = torch.from_numpy(np.ascontiguousarray(a0)).to(dev)
    base_b = torch.from_numpy(np.ascontiguousarray(want.blocks).view(np.int32)).to(dev)
    g = torch.Generator(device=dev)
    perms = [torch.arange(N0, device=dev)]
    for j in range(1, COPIES):
        g.manual_seed(1000 + j)
        perms.append(torch.randperm(N0, generator=g, device=dev))
    n = N0 * COPIES
    delta = torch.empty((K, n), dtype=torch.int32, device=dev)
    acc = torch.empty(n, dtype=torch.uint8, device=dev)
    expect = torch.empty(n, dtype=torch.int32, device=dev)
    for j in range(COPIES):
        nxt = (j + 1) % COPIES
        idx = j * N0 + perms[j]
        acc[idx] = base_a
        expect[idx] = base_b
        for a in range(K):
            delta[a][idx] = (nxt * N0 + perms[nxt][base_d[a]]).int()
    del base_d, perms
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    assert want.num_blocks < n  # non-trivial: every class has COPIES members
    return delta.reshape(-1), acc, expect, want.num_blocks, want.refine_iters


def _single(dk, delta, acc, n, grouping=0):
    from paper_2508_20735_b200 import _native as nat
    ctx = dk.Context(0)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    view = nat.CDfa(n, K, delta.data_ptr(), acc.data_ptr(), -1)
    rep = nat.CReport()
    opts = nat.COptions(0, 0, 0, 0, 0, 64, grouping)
    nat.check(nat.lib.dfakit_minimize_device(ctx.handle, C.byref(view), int(dk.Algorithm.sort_pr), C.byref(opts),
                                             out.data_ptr(), C.byref(rep), ctx.stream))
    torch.cuda.synchronize()
    return out, int(rep.refining_iterations), int(rep.num_blocks)


@pytest.mark.parametrize("grouping", [0, 1], ids=["default", "radix_sort"])
def test_config4_single_gpu_exact(dk, instance, grouping):
    delta, acc, expect, nb, iters = instance
    got, it, b = _single(dk, delta, acc, expect.numel(), grouping)
    assert b == nb and it == iters
    assert torch.equal(got, expect)


def test_config4_sharded_native_world1_nccl_exact(dk, instance):
    import torch.distributed as dist
    from paper_2508_20735_b200 import sharded
    delta, acc, expect, nb, iters = instance
    n = expect.numel()
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
    sk.close()
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        ctx = dk.Context(0)
        comm = sharded.NativeComm(ctx)
        got, r = sharded.sort_pr_sharded_native(ctx, comm, delta, acc, n, K)
        torch.cuda.synchronize()
        comm.close()
        assert r.num_blocks == nb and r.refining_iterations == iters
        assert torch.equal(got, expect)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_config4_sharded_native_hub_exact(dk, instance, world, monkeypatch):
    """World sizes 2 and 4 of the native driver: ranks are threads of this
    process sharing the GPU (and the read-only automaton), each with its own
    context; every rank must return the whole exact partition."""
    from paper_2508_20735_b200 import _native as nat
    monkeypatch.setenv("DFAKIT_SHARD_PEER", "2")  # the peer-memory exchange, required
    delta, acc, expect, nb, iters = instance
    n = expect.numel()
    hub = C.c_void_p()
    nat.check(nat.lib.dfakit_local_hub_create(world, C.byref(hub)))
    out, errs = [None] * world, []

    def rank_main(r):
        try:
            ctx = dk.Context(0)
            comm = C.c_void_p()
            nat.check(nat.lib.dfakit_comm_init_local(hub, r, C.byref(comm)))
            blocks = torch.empty(n, dtype=torch.int32, device="cuda")
            torch.cuda.synchronize()
            view = nat.CDfa(n, K, delta.data_ptr(), acc.data_ptr(), -1)
            rep = nat.CReport()
            nat.check(nat.lib.dfakit_sort_pr_sharded(ctx.handle, comm, C.byref(view), blocks.data_ptr(),
                                                     C.byref(rep), None, None))
            torch.cuda.synchronize()
            out[r] = (torch.equal(blocks, expect), int(rep.refining_iterations), int(rep.num_blocks))
            del blocks
            nat.lib.dfakit_comm_destroy(comm)
        except Exception as e:  # pragma: no cover - reported below
            errs.append((r, repr(e)))

    threads = [threading.Thread(target=rank_main, args=(r,), daemon=True) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=900)
    nat.lib.dfakit_local_hub_destroy(hub)
    torch.cuda.empty_cache()
    assert not errs, errs
    for r in range(world):
        same, it, b = out[r]
        assert same and it == iters and b == nb, (world, r, same, it, b)
