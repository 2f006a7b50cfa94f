"""Sharded sort_pr: one process per GPU, states sharded across ranks.

The single-GPU engine's pass (reference src/minimize.cpp:354-419, paper
Alg. 4) split over W ranks:

* states are sharded in contiguous ranges ``[lo, hi)`` of ``S = ceil(n / W)``;
  delta and the accepting flags are replicated (read-only, 4 B per
  transition -- 4 GB at 1B transitions, a small part of 180 GB of HBM), and
  so is the block-label array, re-assembled after every pass by one NCCL
  allgather of the label slices (the "block-ID allgather" of the design);
* a pass whose keys pack into <= 20 bits builds a local (run minimum, run
  size) counting table over the rank's active states and allreduces it (MIN
  / SUM) -- every rank then relabels its own states;
* wider passes partition each rank's (key, state) entries by owner rank
  (top hash bits), exchange them with one all-to-all, group them at the
  owner (shared-memory radix buckets; fingerprint groups verified tuple by
  tuple -- the owner can read any delta row and label), and return one word
  per entry (new min-state label | survivor bit) by the reverse all-to-all:
  the global merge-and-renumber;
* the fixed-point test B' = B - A + R uses allreduced counts, so every rank
  takes the same branch; a fingerprint collision anywhere re-runs the pass
  on every rank with a new salt.

Results are identical to the single-GPU engine and the reference: the same
partition under canonical numbering and the same refining-pass count.

The loop is written against two small interfaces: ``ops`` (local pass
primitives; :class:`CudaShardOps` calls the sm_100a kernels through the C
ABI) and ``comm`` (:class:`TorchComm`, torch.distributed collectives --
NCCL over NVLink in production).  The gloo CPU tests of the protocol plug a
numpy ``ops`` implemented under tests/; the product has no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from ._native import CDfa as _CDfa, Context, CPassPlan, check, lib

PLAN_TABLE, PLAN_PACKED, PLAN_FINGERPRINT, PLAN_CHUNKED = 0, 1, 2, 3
KEYLAB_BITS = 255  # PassPlan.keylab_bytes tag: one bit per state
BIT_LABELS_MIN_STATES = 1 << 25  # refine.cuh kBitLabelsMinStates
_SALT0 = 0x5EED5EED5EED


def plan_pass(n: int, k: int, num_blocks: int, active_states: int, collisions: int = 0) -> CPassPlan:
    """Key plan of one pass (dfakit_plan_pass; host only, same on every rank)."""
    p = CPassPlan()
    check(lib.dfakit_plan_pass(n, k, num_blocks, active_states, collisions, 0, C.byref(p)))
    if p.strategy == PLAN_CHUNKED:
        # the sharded engine retries fingerprints with fresh salts instead
        p.strategy, p.field_bits, p.key_bits, p.keylab_bytes = PLAN_FINGERPRINT, 0, 64, 0
    return p


def _mix64(z: int) -> int:
    m = (1 << 64) - 1
    z = (z + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


@dataclass
class ShardReport:
    num_blocks: int
    refining_iterations: int
    passes: int
    collisions: int
    exchanged_entries: int      # entries sent by this rank over all passes
    table_passes: int


class TorchComm:
    """Collectives through torch.distributed.  ``stage_cpu`` runs them on host
    copies (gloo with CUDA tensors, e.g. two ranks sharing one GPU in tests)."""

    def __init__(self, group=None, stage_cpu: bool = False):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.stage_cpu = stage_cpu
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)

    def _host(self, t):
        return t.cpu() if self.stage_cpu else t

    def allreduce_(self, t, op: str):
        import torch
        o = {"sum": self.dist.ReduceOp.SUM, "min": self.dist.ReduceOp.MIN}[op]
        h = self._host(t)
        if op == "min" and h.dtype == torch.int32:
            # unsigned MIN on int32 storage: flip the sign bit around the reduction
            h = h ^ torch.tensor(-(1 << 31), dtype=torch.int32, device=h.device)
            self.dist.all_reduce(h, op=o, group=self.group)
            h = h ^ torch.tensor(-(1 << 31), dtype=torch.int32, device=h.device)
        else:
            self.dist.all_reduce(h, op=o, group=self.group)
        if h is not t:
            t.copy_(h)
        return t

    def all_to_all_counts(self, counts):
        import torch
        h = self._host(counts.to(torch.int64))
        out = torch.empty_like(h)
        self.dist.all_to_all_single(out, h, group=self.group)
        return out

    def all_to_all_v(self, send, send_counts, recv_counts):
        import torch
        h = self._host(send)
        out = torch.empty((int(sum(recv_counts)),) + tuple(h.shape[1:]), dtype=h.dtype, device=h.device)
        self.dist.all_to_all_single(out, h, output_split_sizes=[int(x) for x in recv_counts],
                                    input_split_sizes=[int(x) for x in send_counts], group=self.group)
        return out.to(send.device) if self.stage_cpu else out

    def allgather_slices_(self, full, shard: int):
        """full[r*shard:(r+1)*shard] of every rank r -> full on every rank
        (on byte views: int16 / uint8 label arrays travel on every backend)."""
        import torch
        h = self._host(full)
        es = h.element_size()
        h8 = h.view(torch.uint8)
        mine = h8[self.rank * shard * es:(self.rank + 1) * shard * es].clone()
        if self.backend == "nccl":
            self.dist.all_gather_into_tensor(h8, mine, group=self.group)
        else:
            parts = list(h8.split(shard * es))
            self.dist.all_gather(parts, mine, group=self.group)
            h8.copy_(torch.cat(parts))
        if h is not full:
            full.copy_(h)
        return full


class CudaShardOps:
    """Local pass primitives of one rank: the sm_100a kernels via the C ABI.

    ``delta`` (int32 view of uint32, letter-major k*n) and ``acc`` (uint8, n)
    are full, replicated CUDA tensors on this rank's device."""

    def __init__(self, ctx: Context, delta, acc, n: int, k: int):
        import torch
        self.torch = torch
        self.ctx = ctx
        self.delta, self.acc = delta, acc
        self.n, self.k = n, k
        self.device = delta.device if k else acc.device
        self.view = _CDfa(n, k, delta.data_ptr() if k else None, acc.data_ptr(), -1)
        self._scratch = {}

    @property
    def stream(self):
        """every primitive runs on torch's current stream: collectives and
        kernels are ordered without cross-stream waits"""
        # 0 (torch's default stream) would mean "the context's stream" at the
        # C ABI: pass cudaStreamLegacy, the same NULL stream, explicitly
        return self.torch.cuda.current_stream(self.device).cuda_stream or 1

    # buffers reused across passes
    def _buf(self, name, count, dtype):
        b = self._scratch.get(name)
        if b is None or b.numel() < count or b.dtype != dtype:
            b = self.torch.empty(max(count, 1), dtype=dtype, device=self.device)
            self._scratch[name] = b
        return b[:count]

    def init(self, lab, act, lo, hi):
        B, A, M = C.c_uint32(), C.c_uint32(), C.c_uint64()
        check(lib.dfakit_shard_init(self.ctx.handle, C.byref(self.view), lo, hi, lab.data_ptr(), act.data_ptr(),
                                    C.byref(B), C.byref(A), C.byref(M), self.stream))
        return int(B.value), int(A.value), int(M.value)

    def keylab(self, lab, plan, num_blocks):
        if not plan.keylab_bytes:
            return lab
        if plan.keylab_bytes == 1 and num_blocks <= 2 and self.n >= BIT_LABELS_MIN_STATES:
            plan.keylab_bytes = KEYLAB_BITS  # two blocks, large n: one bit per state
        if plan.keylab_bytes == KEYLAB_BITS:
            out = self._buf("keylab_bits", (self.n + 31) // 32, self.torch.int32)
        else:
            dt = {1: self.torch.uint8, 2: self.torch.int16, 4: self.torch.int32}[plan.keylab_bytes]
            out = self._buf(f"keylab{plan.keylab_bytes}", self.n, dt)
        check(lib.dfakit_shard_keylab(self.ctx.handle, lab.data_ptr(), self.n, num_blocks, C.byref(plan),
                                      out.data_ptr(), self.stream))
        return out

    def table_signature(self, keylab, plan, lst, m, base=0):
        t = self.torch
        tsize = 1 << plan.key_bits
        keys32 = self._buf("keys32", m, t.int32)
        tmin = t.empty(tsize, dtype=t.int32, device=self.device)
        tcnt = t.empty(tsize, dtype=t.int32, device=self.device)
        check(lib.dfakit_shard_table_signature(self.ctx.handle, C.byref(self.view), keylab.data_ptr(), C.byref(plan),
                                               _ptr(lst), base, m, keys32.data_ptr(), tmin.data_ptr(),
                                               tcnt.data_ptr(), self.stream))
        return keys32, tmin, tcnt

    def table_apply(self, plan, lst, keys32, m, tmin, tcnt, lab, act, next_keylab=None, base=0):
        ctr = self.torch.empty(4, dtype=self.torch.int32, device=self.device)
        check(lib.dfakit_shard_table_apply(self.ctx.handle, C.byref(plan), _ptr(lst), base, keys32.data_ptr(), m,
                                           tmin.data_ptr(), tcnt.data_ptr(), lab.data_ptr(), act.data_ptr(),
                                           next_keylab.data_ptr() if next_keylab is not None else None,
                                           ctr.data_ptr(), self.stream))
        return ctr

    def partition(self, keylab, plan, salt, lst, m, world, base=0):
        t = self.torch
        send = self._buf("send", 4 * m, t.int32).view(-1, 4) if m else t.empty((0, 4), dtype=t.int32,
                                                                                   device=self.device)
        counts = t.empty(world, dtype=t.int32, device=self.device)
        check(lib.dfakit_shard_partition(self.ctx.handle, C.byref(self.view), keylab.data_ptr(), C.byref(plan),
                                         salt, _ptr(lst), base, m, world, send.data_ptr() if m else None,
                                         counts.data_ptr(), self.stream))
        return send, counts

    def group(self, lab, plan, recv):
        t = self.torch
        cnt = recv.shape[0]
        res = self._buf("res", cnt, t.int32)
        ctr = t.empty(4, dtype=t.int32, device=self.device)
        check(lib.dfakit_shard_group(self.ctx.handle, C.byref(self.view), lab.data_ptr(), C.byref(plan),
                                     recv.data_ptr() if cnt else None, cnt, res.data_ptr(), ctr.data_ptr(),
                                     self.stream))
        return res, ctr

    def apply(self, send, results, lab, act):
        check(lib.dfakit_shard_apply(self.ctx.handle, send.data_ptr() if send.shape[0] else None,
                                     results.data_ptr(), send.shape[0], lab.data_ptr(), act.data_ptr(), self.stream))

    def compact(self, act, lo, hi):
        t = self.torch
        lst = t.empty(max(hi - lo, 1), dtype=t.int32, device=self.device)
        cnt = t.zeros(1, dtype=t.int32, device=self.device)
        check(lib.dfakit_shard_compact(self.ctx.handle, act.data_ptr(), lo, hi, lst.data_ptr(), cnt.data_ptr(),
                                       self.stream))
        m = int(cnt.item())
        # a shard whose states are all active travels as the identity range
        return (None if m == hi - lo else lst[:m]), m

    def canonical(self, lab):
        t = self.torch
        out = t.empty(max(self.n, 1), dtype=t.int32, device=self.device)
        nb = C.c_uint32()
        check(lib.dfakit_shard_canonical(self.ctx.handle, lab.data_ptr(), self.n, out.data_ptr(), C.byref(nb),
                                         self.stream))
        return out[: self.n], int(nb.value)


def _ptr(t):
    return None if t is None else t.data_ptr()


def sort_pr_sharded(ops, comm, n: int, k: int, max_collision_retries: int = 16):
    """Runs the sharded sortPR loop; every rank returns (block_of tensor on the
    ops device, canonical numbering, ShardReport)."""
    import torch
    rank, world = comm.rank, comm.world
    shard = max(1, -(-n // world))
    lo, hi = min(n, rank * shard), min(n, (rank + 1) * shard)
    dev = ops.device
    lab = torch.zeros(world * shard, dtype=torch.int32, device=dev)
    act = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
    rep = ShardReport(0, 0, 0, 0, 0, 0)
    if n == 0:
        return torch.zeros(0, dtype=torch.int32, device=dev), rep
    B, A, m_total = ops.init(lab, act, lo, hi)
    lst, m = ops.compact(act, lo, hi)
    salt, strikes = _SALT0, 0
    carried = None  # (key labels of the current partition, bytes): ranks of a full table pass
    while m_total > 0:
        rep.passes += 1
        plan = plan_pass(n, k, B, m_total, min(strikes, 2))
        if plan.keylab_bytes and carried is not None:
            keylab, plan.keylab_bytes = carried
        else:
            keylab = ops.keylab(lab, plan, B)
        carried = None
        next_kl = None
        if plan.strategy == PLAN_TABLE:
            rep.table_passes += 1
            keys32, tmin, tcnt = ops.table_signature(keylab, plan, lst, m, base=lo)
            comm.allreduce_(tmin, "min")
            comm.allreduce_(tcnt, "sum")
            act[lo:hi].zero_()
            if m_total == n:
                # every block of the next partition is one table key: the
                # ranks of the occupied entries are its compact block ids
                next_kl = torch.zeros(world * shard, dtype=torch.int16 if plan.key_bits <= 16 else torch.int32,
                                      device=dev)
            ctr = ops.table_apply(plan, lst, keys32, m, tmin, tcnt, lab, act, next_kl, base=lo).to(torch.int64)
            comm.allreduce_(ctr, "sum")
            runs, ablk, surv, _ = (int(x) for x in ctr.tolist())
        else:
            send, counts = ops.partition(keylab, plan, salt, lst, m, world, base=lo)
            send_counts = counts.to(torch.int64).cpu().tolist()
            recv_counts = comm.all_to_all_counts(counts).cpu().tolist()
            recv = comm.all_to_all_v(send, send_counts, recv_counts)
            rep.exchanged_entries += int(send.shape[0])
            res, ctr = ops.group(lab, plan, recv)
            ctr = ctr.to(torch.int64)
            comm.allreduce_(ctr, "sum")
            runs, ablk, surv, coll = (int(x) for x in ctr.tolist())
            if coll:
                # a verified fingerprint collision on some owner: nothing was
                # applied anywhere; every rank re-runs the pass with a new salt
                rep.collisions += 1
                rep.passes -= 1
                strikes += 1
                if strikes > max_collision_retries:
                    raise RuntimeError("sharded sort_pr: repeated fingerprint collisions")
                salt = _mix64(salt + 0x1234567)
                continue
            if B - A + runs == B:
                break  # fixed point: no block split (reference l.411)
            back = comm.all_to_all_v(res.view(-1, 1), recv_counts, send_counts).view(-1)
            act[lo:hi].zero_()
            ops.apply(send, back, lab, act)
        strikes = 0
        new_b = B - A + runs
        if new_b == B:
            break
        rep.refining_iterations += 1
        B, A, m_total = new_b, ablk, surv
        comm.allgather_slices_(lab, shard)
        if next_kl is not None:
            comm.allgather_slices_(next_kl, shard)
            carried = (next_kl, next_kl.element_size())
        lst, m = ops.compact(act, lo, hi)
    blocks, nb = ops.canonical(lab)
    rep.num_blocks = nb
    return blocks, rep


class NativeComm:
    """An NCCL communicator owned by the library (dfakit_comm_init): rank 0's
    NCCL unique id travels to the other ranks by a torch.distributed
    broadcast; the pass loop then runs in C++ (dfakit_sort_pr_sharded)."""

    def __init__(self, ctx: Context, group=None):
        import torch
        import torch.distributed as dist
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        uid = torch.zeros(128, dtype=torch.uint8)
        if self.rank == 0:
            check(lib.dfakit_comm_unique_id(uid.data_ptr()))
        t = uid.cuda() if dist.get_backend(group) == "nccl" else uid
        dist.broadcast(t, src=0, group=group)
        uid = t.cpu().contiguous()
        h = C.c_void_p()
        check(lib.dfakit_comm_init(ctx.handle, uid.data_ptr(), self.world, self.rank, C.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            lib.dfakit_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def sort_pr_sharded_native(ctx: Context, comm: NativeComm, delta, acc, n: int, k: int, out=None):
    """The sharded pass loop in C++ over NCCL (same protocol as
    sort_pr_sharded).  delta / acc: full automaton on this rank's device.
    Returns (block_of tensor, ShardReport)."""
    import torch
    from ._native import CReport
    dev = acc.device
    if out is None:
        out = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    view = _CDfa(n, k, delta.data_ptr() if k else None, acc.data_ptr(), -1)
    rep = CReport()
    sent = C.c_uint64()
    stream = torch.cuda.current_stream(dev).cuda_stream or 1
    check(lib.dfakit_sort_pr_sharded(ctx.handle, comm.handle, C.byref(view), out.data_ptr(), C.byref(rep),
                                     C.byref(sent), stream))
    r = ShardReport(int(rep.num_blocks), int(rep.refining_iterations), int(rep.passes), int(rep.hash_collisions),
                    int(sent.value), 0)
    return out[:n], r
