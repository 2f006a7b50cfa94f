"""Sharded sort_pr protocol on CPU: world-size 1, 2 and 3 gloo process groups
running paper_2508_20735_b200.sharded.sort_pr_sharded over the test-only numpy
pass primitives (tests/shard_cpu_ops.py).  Checked against the oracle: the
identical canonical partition and refining-pass count for every shard count,
through counting-table passes, packed and fingerprint all-to-all passes and
forced fingerprint collisions (retries with a new salt on every rank)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

CASES = [
    # (kind, n, k, frac, seed, fp_bits)
    ("random", 300, 2, 0.5, 11, 64),        # table passes only (small keys)
    ("random", 5000, 3, 0.5, 12, 64),       # packed 64-bit keys -> all-to-all
    ("random", 4000, 6, 0.9, 13, 64),       # dense table passes, then fingerprints
    ("random", 3000, 5, 0.97, 14, 6),       # 6-bit fingerprints: forced collisions + retries
    ("copies", 400, 8, 0.5, 15, 64),        # large equivalence classes (heavy key duplication)
    ("family", 7, 0, 0.0, 0, 64),           # bit-splitter 7
    ("family", 11, 0, 0.0, 1, 64),          # Fibonacci 11 (one pass per state pair)
]


def make_case(case):
    sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
    import pyoracle
    o = pyoracle.COracle()
    kind, n, k, frac, seed, _ = case
    if kind == "random":
        d, a, _ = o.gen_random(n, k, frac, seed)
    elif kind == "copies":
        base, acc0, _ = o.gen_random(n, k, frac, seed)
        c = 30
        d = np.empty((k, n * c), np.uint32)
        for j in range(c):
            d[:, j * n:(j + 1) * n] = base + ((j + 1) % c) * n
        a = np.tile(acc0, c)
    else:
        d, a, _ = o.gen_family("bitsplit" if seed == 0 else "fib", n)
    want = o.minimize("moore", d, a)
    return d, a, want


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        sys.path.insert(0, os.path.dirname(HERE))
        from paper_2508_20735_b200.sharded import TorchComm, sort_pr_sharded
        from shard_cpu_ops import NumpyShardOps
        comm = TorchComm()
        out = []
        for case in CASES:
            d, a, want = make_case(case)
            ops = NumpyShardOps(d, a, fp_bits=case[5])
            blocks, rep = sort_pr_sharded(ops, comm, d.shape[1], d.shape[0])
            ok = (np.array_equal(blocks.numpy().view(np.uint32), want.blocks)
                  and rep.num_blocks == want.num_blocks and rep.refining_iterations == want.refine_iters)
            out.append((case, ok, rep.refining_iterations, want.refine_iters, rep.collisions, rep.table_passes,
                        rep.passes, rep.exchanged_entries))
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc()))


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_protocol_matches_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(results[r], str), results[r]
        for case, ok, got, want, *_ in results[r]:
            assert ok, (world, r, case, got, want)
    rows = results[0]
    # every path of the protocol was exercised
    assert any(coll > 0 for (_, _, _, _, coll, *_r) in rows), "no forced collision was retried"
    assert any(tp > 0 for (_, _, _, _, _, tp, *_r) in rows), "no counting-table pass"
    assert any(p > tp for (_, _, _, _, _, tp, p, _) in rows), "no all-to-all pass"
