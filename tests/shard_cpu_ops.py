"""Test-only CPU implementation of the sharded engine's local pass primitives.

Same interface and semantics as paper_2508_20735_b200.sharded.CudaShardOps,
written with numpy on CPU torch tensors, so the pass protocol of
sort_pr_sharded (all-to-all, allreduce, allgather, collision retries, fixed
point) can run in world-size-2 gloo process groups without a GPU.  This is
test infrastructure: the product calls the CUDA kernels only.
"""
import numpy as np
import torch

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def mix64(z):
    z = z.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def u32(t):
    return t.numpy().view(np.uint32)


class NumpyShardOps:
    def __init__(self, delta: np.ndarray, acc: np.ndarray, fp_bits: int = 64):
        # fp_bits < 64 narrows the fingerprints of every pass's FIRST attempt
        # (initial salt) so collisions are forced and the retry (new salt,
        # full width) path of the protocol runs
        self.delta = np.ascontiguousarray(delta, dtype=np.uint32)  # (k, n)
        self.acc = np.ascontiguousarray(acc, dtype=np.uint8)
        self.k, self.n = self.delta.shape
        self.device = torch.device("cpu")
        self.fp_mask = np.uint64((1 << fp_bits) - 1) if fp_bits < 64 else M64

    def init(self, lab, act, lo, hi):
        acc = self.acc
        ia, ir = np.flatnonzero(acc), np.flatnonzero(acc == 0)
        la = ia[0] if ia.size else 0
        lr = ir[0] if ir.size else 0
        L = u32(lab)
        L[: self.n] = np.where(acc != 0, la, lr)
        A = act.numpy()
        keep_a, keep_r = ia.size >= 2, ir.size >= 2
        A[lo:hi] = np.where(acc[lo:hi] != 0, keep_a, keep_r)
        B = int(ia.size > 0) + int(ir.size > 0)
        return B, int(keep_a) + int(keep_r), (ia.size if keep_a else 0) + (ir.size if keep_r else 0)

    def keylab(self, lab, plan, num_blocks):
        if not plan.keylab_bytes:
            return lab
        L = u32(lab)[: self.n]
        heads = (L == np.arange(self.n, dtype=np.uint32)).astype(np.int64)
        pos = np.cumsum(heads) - heads
        return torch.from_numpy(pos[L].astype(np.uint32).view(np.int32))

    def _tuples(self, keylab, qs):
        L = {torch.int32: lambda t: u32(t), torch.int16: lambda t: t.numpy().view(np.uint16)}.get(
            keylab.dtype, lambda t: t.numpy())(keylab)
        L = L[: self.n].astype(np.uint64)
        return L[qs], [L[self.delta[a][qs]] for a in range(self.k)]

    def _keys(self, keylab, plan, salt, qs):
        lead, succ = self._tuples(keylab, qs)
        if plan.strategy == 2:  # fingerprint
            h = mix64(np.uint64(salt) ^ (lead * np.uint64(0xD6E8FEB86659FD93)))
            for a, s in enumerate(succ):
                h = mix64((h + np.uint64(a)) ^ (s * np.uint64(0xD6E8FEB86659FD93)))
            from paper_2508_20735_b200.sharded import _SALT0
            return h & self.fp_mask if salt == _SALT0 else h
        fb = np.uint64(plan.field_bits)
        key = lead.copy()
        for s in succ:
            key = (key << fb) | s
        return key

    @staticmethod
    def _states(lst, m, base):
        return np.arange(base, base + m, dtype=np.uint32) if lst is None else u32(lst)[:m]

    def table_signature(self, keylab, plan, lst, m, base=0):
        qs = self._states(lst, m, base)
        keys = self._keys(keylab, plan, 0, qs).astype(np.int64)
        tsize = 1 << plan.key_bits
        tmin = np.full(tsize, 0xFFFFFFFF, np.uint64)
        tcnt = np.zeros(tsize, np.int64)
        np.minimum.at(tmin, keys, qs.astype(np.uint64))
        np.add.at(tcnt, keys, 1)
        return (torch.from_numpy(keys.astype(np.uint32).view(np.int32)),
                torch.from_numpy(tmin.astype(np.uint32).view(np.int32)),
                torch.from_numpy(tcnt.astype(np.int32)))

    def table_apply(self, plan, lst, keys32, m, tmin, tcnt, lab, act, next_keylab=None, base=0):
        qs = self._states(lst, m, base)
        keys = u32(keys32)[:m].astype(np.int64)
        rep = u32(tmin)[keys]
        multi = tcnt.numpy()[keys] >= 2
        if next_keylab is not None:
            occ = (tcnt.numpy() > 0).astype(np.int64)
            rank = np.cumsum(occ) - occ
            nk = next_keylab.numpy().view(np.uint16 if next_keylab.dtype == torch.int16 else np.uint32)
            nk[qs] = rank[keys]
        u32(lab)[qs] = rep
        act.numpy()[qs] = multi
        heads = rep == qs
        return torch.tensor([heads.sum(), (heads & multi).sum(), multi.sum(), 0], dtype=torch.int32)

    def partition(self, keylab, plan, salt, lst, m, world, base=0):
        qs = self._states(lst, m, base)
        key = self._keys(keylab, plan, salt, qs)
        hk = key if plan.strategy == 2 else mix64(key)
        dest = ((hk >> np.uint64(32)) * np.uint64(world)) >> np.uint64(32)
        order = np.argsort(dest, kind="stable")
        ent = np.zeros((m, 4), np.uint32)
        ent[:, 0] = (hk & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        ent[:, 1] = (hk >> np.uint64(32)).astype(np.uint32)
        ent[:, 2] = qs
        ent = ent[order]
        counts = np.bincount(dest.astype(np.int64), minlength=world).astype(np.int32)
        return torch.from_numpy(ent.view(np.int32)), torch.from_numpy(counts)

    def group(self, lab, plan, recv):
        e = recv.numpy().view(np.uint32).reshape(-1, 4)
        cnt = e.shape[0]
        if cnt == 0:
            return torch.zeros(0, dtype=torch.int32), torch.zeros(4, dtype=torch.int32)
        hk = (e[:, 1].astype(np.uint64) << np.uint64(32)) | e[:, 0].astype(np.uint64)
        qs = e[:, 2]
        uniq, inv = np.unique(hk, return_inverse=True)
        rep = np.full(uniq.size, 0xFFFFFFFF, np.uint64)
        np.minimum.at(rep, inv, qs.astype(np.uint64))
        size = np.bincount(inv, minlength=uniq.size)
        r = rep[inv].astype(np.uint32)
        multi = size[inv] >= 2
        heads = r == qs
        coll = 0
        if plan.strategy == 2:
            L = u32(lab)[: self.n]
            nh = ~heads
            a_q, a_r = qs[nh], r[nh]
            same = L[a_q] == L[a_r]
            for a in range(self.k):
                same &= L[self.delta[a][a_q]] == L[self.delta[a][a_r]]
            coll = int(not same.all())
        res = (r.astype(np.uint64) | (multi.astype(np.uint64) << np.uint64(31))).astype(np.uint32)
        ctr = [heads.sum(), (heads & multi).sum(), multi.sum(), coll]
        return torch.from_numpy(res.view(np.int32)), torch.tensor(ctr, dtype=torch.int32)

    def apply(self, send, results, lab, act):
        e = send.numpy().view(np.uint32).reshape(-1, 4)
        r = results.numpy().view(np.uint32)
        u32(lab)[e[:, 2]] = r & np.uint32(0x7FFFFFFF)
        act.numpy()[e[:, 2]] = (r >> np.uint32(31)).astype(np.uint8)

    def compact(self, act, lo, hi):
        idx = (np.flatnonzero(act.numpy()[lo:hi]) + lo).astype(np.uint32)
        if idx.size == hi - lo:
            return None, int(idx.size)
        return torch.from_numpy(idx.view(np.int32).copy()), int(idx.size)

    def canonical(self, lab):
        L = u32(lab)[: self.n]
        heads = (L == np.arange(self.n, dtype=np.uint32)).astype(np.int64)
        pos = np.cumsum(heads) - heads
        out = pos[L].astype(np.uint32)
        return torch.from_numpy(out.view(np.int32)), int(heads.sum())
