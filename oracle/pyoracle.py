"""ctypes bindings for the test-only checkers in oracle/.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, by __graft_entry__.smoke() and
by bench.py's cpu_baseline / --impl reference legs -- never by the product
package.  Two backends share one numpy-level API:

* ``COracle``  -- oracle/liboracle.so, the C restatement (oracle.c)
* ``RefLib``   -- oracle/_ref/libdfakit_ref.so, the unmodified reference
                  sources compiled in place (oracle/Makefile) + ref_shim.cpp

A DFA is passed as ``(delta, acc, initial)`` with ``delta`` a C-contiguous
uint32 array of shape (k, n) -- letter-major like the reference's
``delta[a][q]`` -- ``acc`` uint8 of shape (n,), and ``initial`` an int
(-1 = absent).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ALGOS = {"moore": 0, "trans": 1, "naive": 2, "naive-fused": 3, "sort": 4, "transpr": 5}
MODES = {"equivalence": 0, "inclusion": 1, "full": 2}
VERDICTS = {0: "equivalent", 1: "included", 2: "counterexample"}
FAMILIES = {"random": 0, "fib": 1, "bitsplit": 2, "bitsplit-ext": 3, "cycle": 4,
            "memory-perfect": 5, "memory-forgetful": 6}

u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


@dataclass
class MinResult:
    blocks: np.ndarray
    num_blocks: int
    refine_iters: int
    closure_iters: int = 0


@dataclass
class ProductOut:
    verdict: str
    explored: int
    levels: int
    counterexample: List[int] = field(default_factory=list)


def _dfa_args(delta, acc):
    delta = np.ascontiguousarray(delta, dtype=np.uint32)
    acc = np.ascontiguousarray(acc, dtype=np.uint8)
    k, n = delta.shape
    if acc.shape != (n,):
        raise ValueError("acc shape mismatch")
    return delta, acc, n, k


class _ORDfa(C.Structure):
    _fields_ = [("n", C.c_uint32), ("k", C.c_uint32), ("delta", C.c_void_p), ("acc", C.c_void_p),
                ("initial", C.c_int64)]


class _ORProduct(C.Structure):
    _fields_ = [("verdict", C.c_int32), ("levels", C.c_uint32), ("explored", C.c_uint64), ("cex_len", C.c_uint32)]


class COracle:
    """The C restatement (oracle/oracle.c)."""

    kind = "port"

    def __init__(self, path: Optional[str] = None):
        path = path or os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.or_gen_random.argtypes = [C.c_uint32, C.c_uint32, C.c_double, C.c_uint64, u32p, u8p]
        L.or_fib_word_len.restype = C.c_uint64
        L.or_fib_word_len.argtypes = [C.c_uint32]
        L.or_cycle_fib.restype = C.c_uint64
        L.or_cycle_fib.argtypes = [C.c_uint32]
        L.or_cycle_letters.restype = C.c_uint32
        L.or_cycle_letters.argtypes = [C.c_uint32]
        for fn in ("or_gen_fib", "or_gen_bitsplitter", "or_gen_bitsplitter_ext", "or_gen_cycle", "or_gen_chain"):
            getattr(L, fn).argtypes = [C.c_uint32, u32p, u8p]
        L.or_gen_memory.argtypes = [C.c_uint32, C.c_int, u32p, u8p]
        L.or_gen_synth.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, u32p, u8p]
        P = C.POINTER(_ORDfa)
        for fn in ("or_moore", "or_sort_pr", "or_naive_pr_fused"):
            getattr(L, fn).restype = C.c_uint32
            getattr(L, fn).argtypes = [P, u32p, C.POINTER(C.c_uint32)]
        L.or_naive_pr.restype = C.c_uint32
        L.or_naive_pr.argtypes = [P, C.c_int, C.c_uint64, u32p, C.POINTER(C.c_uint32)]
        L.or_trans_pr.restype = C.c_uint32
        L.or_trans_pr.argtypes = [P, C.c_int, C.c_uint64, u32p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.or_trans_minimize.restype = C.c_uint32
        L.or_trans_minimize.argtypes = [P, C.c_uint64, u32p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.c_void_p]
        L.or_build_transitive_alphabet.restype = C.c_uint32
        L.or_build_transitive_alphabet.argtypes = [P, u32p]
        L.or_floor_log2.restype = C.c_uint32
        L.or_floor_log2.argtypes = [C.c_uint32]
        L.or_explore_product.restype = C.c_int
        L.or_explore_product.argtypes = [P, P, C.c_int, C.c_void_p, C.c_uint64, u32p, C.c_uint32,
                                         C.POINTER(_ORProduct)]
        L.or_normalize.restype = C.c_uint32
        L.or_normalize.argtypes = [u32p, C.c_uint32, u32p]
        L.or_bfs_order.restype = C.c_uint32
        L.or_bfs_order.argtypes = [P, u32p]

    # -- generators ---------------------------------------------------------
    def gen_random(self, n: int, k: int, frac: float, seed: int):
        delta = np.empty((k, n), np.uint32)
        acc = np.empty(n, np.uint8)
        if self.lib.or_gen_random(n, k, frac, seed, delta, acc) != 0:
            raise ValueError("bad parameters")
        return delta, acc, 0

    def gen_synth(self, n: int, k: int, seed: int):
        delta = np.empty((k, n), np.uint32)
        acc = np.empty(n, np.uint8)
        self.lib.or_gen_synth(n, k, seed, delta, acc)
        return delta, acc, 0

    def gen_chain(self, n: int):
        delta = np.empty((1, n), np.uint32)
        acc = np.empty(n, np.uint8)
        self.lib.or_gen_chain(n, delta, acc)
        return delta, acc, 0

    def gen_family(self, name: str, p: int):
        L = self.lib
        if name == "fib":
            n, k, init = int(L.or_fib_word_len(p)), 1, 0
            fn = lambda d, a: L.or_gen_fib(p, d, a)
        elif name == "bitsplit":
            n, k, init = 1 << p, p - 1, -1
            fn = lambda d, a: L.or_gen_bitsplitter(p, d, a)
        elif name == "bitsplit-ext":
            n, k, init = 1 << (p + 1), 2 * p, 0
            fn = lambda d, a: L.or_gen_bitsplitter_ext(p, d, a)
        elif name == "cycle":
            n, k, init = int(L.or_cycle_fib(p)), int(L.or_cycle_letters(p)), 0
            fn = lambda d, a: L.or_gen_cycle(p, d, a)
        elif name in ("memory-perfect", "memory-forgetful"):
            n, k, init = 1 << p, 2, 0
            forget = 1 if name == "memory-forgetful" else 0
            fn = lambda d, a: L.or_gen_memory(p, forget, d, a)
        elif name == "chain":
            return self.gen_chain(p)
        else:
            raise ValueError(name)
        delta = np.empty((k, n), np.uint32)
        acc = np.empty(n, np.uint8)
        if fn(delta, acc) != 0:
            raise ValueError("bad parameters")
        return delta, acc, init

    # -- minimisers -----------------------------------------------------------
    @staticmethod
    def _mk(delta, acc, initial=-1):
        delta, acc, n, k = _dfa_args(delta, acc)
        d = _ORDfa(n, k, delta.ctypes.data, acc.ctypes.data, initial)
        return d, (delta, acc), n, k

    def minimize(self, algo: str, delta, acc, policy: int = 0, seed: int = 0,
                 max_pair_nodes: int = 1 << 16) -> MinResult:
        d, keep, n, k = self._mk(delta, acc)
        out = np.zeros(max(n, 1), np.uint32)
        it = C.c_uint32(0)
        cl = C.c_uint32(0)
        L = self.lib
        if algo == "moore":
            nb = L.or_moore(C.byref(d), out, C.byref(it))
        elif algo == "sort":
            nb = L.or_sort_pr(C.byref(d), out, C.byref(it))
        elif algo == "naive":
            nb = L.or_naive_pr(C.byref(d), policy, seed, out, C.byref(it))
        elif algo == "naive-fused":
            nb = L.or_naive_pr_fused(C.byref(d), out, C.byref(it))
        elif algo == "transpr":
            nb = L.or_trans_pr(C.byref(d), policy, seed, out, C.byref(it), C.byref(cl))
        elif algo == "trans":
            nb = L.or_trans_minimize(C.byref(d), max_pair_nodes, out, C.byref(it), C.byref(cl), None)
            if nb == 0xFFFFFFFF:
                raise MemoryError("pair-node budget")
        else:
            raise ValueError(algo)
        return MinResult(out[:n].copy(), int(nb), int(it.value), int(cl.value))

    def trans_apart(self, delta, acc):
        d, keep, n, k = self._mk(delta, acc)
        out = np.zeros(max(n, 1), np.uint32)
        ap = np.zeros(max(n * n, 1), np.uint8)
        it = C.c_uint32(0)
        cl = C.c_uint32(0)
        self.lib.or_trans_minimize(C.byref(d), 1 << 40, out, C.byref(it), C.byref(cl), ap.ctypes.data)
        return ap[: n * n].reshape(n, n)

    def transitive_alphabet(self, delta, acc):
        d, keep, n, k = self._mk(delta, acc)
        levels = int(self.lib.or_floor_log2(n)) + 1
        out = np.empty((k * levels, n), np.uint32)
        self.lib.or_build_transitive_alphabet(C.byref(d), out)
        return out

    def normalize(self, labels) -> Tuple[np.ndarray, int]:
        labels = np.ascontiguousarray(labels, np.uint32)
        out = np.empty_like(labels)
        nb = self.lib.or_normalize(labels, labels.size, out)
        return out, int(nb)

    def bfs_order(self, delta, acc, initial):
        d, keep, n, k = self._mk(delta, acc, initial)
        out = np.empty(max(n, 1), np.uint32)
        cnt = self.lib.or_bfs_order(C.byref(d), out)
        return out[:n], int(cnt)

    # -- product --------------------------------------------------------------
    def explore(self, mode: str, A, B, max_visited: int = 1 << 26, cex_cap: int = 1 << 16) -> ProductOut:
        da, keep_a, na, ka = self._mk(A[0], A[1], A[2])
        db, keep_b, nb_, kb = self._mk(B[0], B[1], B[2])
        cex = np.zeros(cex_cap, np.uint32)
        out = _ORProduct()
        rc = self.lib.or_explore_product(C.byref(da), C.byref(db), MODES[mode], None, max_visited, cex, cex_cap,
                                         C.byref(out))
        if rc == -1 or rc == -2:
            raise ValueError("invalid product arguments")
        if rc == -3:
            raise MemoryError("visited budget")
        return ProductOut(VERDICTS[out.verdict], int(out.explored), int(out.levels),
                          [int(x) for x in cex[: out.cex_len]])


class RefLib:
    """The reference library itself, compiled from /root/reference sources."""

    kind = "reference"

    def __init__(self, path: Optional[str] = None):
        path = path or os.path.join(HERE, "_ref", "libdfakit_ref.so")
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_generate.restype = C.c_int
        L.ref_generate.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_double, C.c_uint64, C.c_void_p, C.c_void_p,
                                   C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_int64)]
        L.ref_minimize.restype = C.c_int64
        L.ref_minimize.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_uint32, C.c_uint32, u32p, u8p, C.c_void_p,
                                   C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.ref_transitive_alphabet.restype = C.c_int
        L.ref_transitive_alphabet.argtypes = [C.c_uint32, C.c_uint32, u32p, u8p, C.c_void_p, C.POINTER(C.c_uint32)]
        L.ref_explore.restype = C.c_int
        L.ref_explore.argtypes = [C.c_int, C.c_uint32, C.c_uint32, u32p, u8p, C.c_int64, C.c_uint32, C.c_uint32, u32p,
                                  u8p, C.c_int64, C.c_uint64, C.POINTER(C.c_int32), C.POINTER(C.c_uint64),
                                  C.POINTER(C.c_uint32), u32p, C.c_uint32, C.POINTER(C.c_uint32)]

    def _gen(self, fam: int, p: int, p2: int = 0, frac: float = 0.0, seed: int = 0):
        n, k, init = C.c_uint32(), C.c_uint32(), C.c_int64()
        if self.lib.ref_generate(fam, p, p2, frac, seed, None, None, C.byref(n), C.byref(k), C.byref(init)) != 0:
            raise ValueError("bad parameters")
        delta = np.empty((k.value, n.value), np.uint32)
        acc = np.empty(n.value, np.uint8)
        self.lib.ref_generate(fam, p, p2, frac, seed, delta.ctypes.data, acc.ctypes.data, C.byref(n), C.byref(k),
                              C.byref(init))
        return delta, acc, int(init.value)

    def gen_random(self, n: int, k: int, frac: float, seed: int):
        return self._gen(0, n, k, frac, seed)

    def gen_family(self, name: str, p: int):
        return self._gen(FAMILIES[name], p)

    def minimize(self, algo: str, delta, acc, policy: int = 0, seed: int = 0, max_pair_nodes: int = 1 << 16,
                 want_blocks: bool = True) -> MinResult:
        delta, acc, n, k = _dfa_args(delta, acc)
        out = np.zeros(max(n, 1), np.uint32)
        it = C.c_uint32(0)
        cl = C.c_uint32(0)
        nb = self.lib.ref_minimize(ALGOS[algo], policy, seed, n, k, delta, acc,
                                   out.ctypes.data if want_blocks else None, C.byref(it), C.byref(cl))
        if nb == -1:
            raise MemoryError("reference resource budget")
        if nb < 0:
            raise RuntimeError("reference error")
        return MinResult(out[:n].copy(), int(nb), int(it.value), int(cl.value))

    def transitive_alphabet(self, delta, acc):
        delta, acc, n, k = _dfa_args(delta, acc)
        kk = C.c_uint32()
        self.lib.ref_transitive_alphabet(n, k, delta, acc, None, C.byref(kk))
        out = np.empty((kk.value, n), np.uint32)
        self.lib.ref_transitive_alphabet(n, k, delta, acc, out.ctypes.data, C.byref(kk))
        return out

    def explore(self, mode: str, A, B, max_visited: int = 1 << 26, cex_cap: int = 1 << 16) -> ProductOut:
        da, aa, na, ka = _dfa_args(A[0], A[1])
        db, ab, nb_, kb = _dfa_args(B[0], B[1])
        verdict, explored, levels, clen = C.c_int32(), C.c_uint64(), C.c_uint32(), C.c_uint32()
        cex = np.zeros(cex_cap, np.uint32)
        rc = self.lib.ref_explore(MODES[mode], na, ka, da, aa, A[2], nb_, kb, db, ab, B[2], max_visited,
                                  C.byref(verdict), C.byref(explored), C.byref(levels), cex, cex_cap, C.byref(clen))
        if rc == -1:
            raise ValueError("invalid product arguments")
        if rc == -3:
            raise MemoryError("visited budget")
        return ProductOut(VERDICTS[verdict.value], int(explored.value), int(levels.value),
                          [int(x) for x in cex[: clen.value]])
