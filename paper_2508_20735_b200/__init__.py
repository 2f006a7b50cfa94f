"""B200-native DFA minimisation and equivalence / inclusion checking.

Python mirror of the reference's library API (reference
include/dfakit/{dfa,minimize,equivalence}.hpp) over the C ABI of
libdfakit_b200.so.  Same names, same argument meaning, same error
behaviour (``ResourceError`` for budgets, ``ValueError`` where the reference
throws std::invalid_argument).  Every algorithm runs on the GPU; there is no
CPU fallback.

DFAs are numpy-backed: ``delta`` is uint32 of shape (k, n), letter-major
like the reference's ``delta[a][q]``; ``accepting`` is uint8 of shape (n,).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from ._native import (Context, DfakitError, NoDeviceError, ResourceError, CDfa, COptions, CProduct, CReport,
                      check, default_context, device_count, lib, EXPORTS, LIB_PATH)

__all__ = [
    "Dfa", "Partition", "RefinementReport", "TransResult", "ProductResult", "ElectionPolicy", "Algorithm",
    "ExploreMode", "Verdict", "ExploreOptions", "moore_minimize", "sort_pr", "naive_pr", "naive_pr_fused",
    "trans_pr", "trans_minimize", "build_transitive_alphabet", "minimize", "explore_product", "check_equiv",
    "check_inclusion", "check_equiv_uf", "Context", "default_context", "device_count", "ResourceError",
    "DfakitError", "NoDeviceError", "LIB_PATH", "EXPORTS", "K_DEFAULT_MAX_VISITED",
]

K_DEFAULT_MAX_VISITED = 1 << 26          # equivalence.hpp:26
K_DEFAULT_MAX_PAIR_NODES = 1 << 16       # minimize.hpp:38
K_DEFAULT_MAX_TRANSITIONS = 1 << 28      # minimize.hpp:41


class Algorithm(enum.IntEnum):           # minimize.hpp:9
    moore = 0
    trans = 1
    naive_pr = 2
    naive_pr_fused = 3
    sort_pr = 4
    trans_pr = 5


class ExploreMode(enum.IntEnum):         # equivalence.hpp:24
    equivalence = 0
    inclusion = 1
    full = 2


class Verdict(enum.IntEnum):             # equivalence.hpp:10
    equivalent = 0
    included = 1
    counterexample = 2


@dataclass(frozen=True)
class ElectionPolicy:                    # minimize.hpp:16-24
    kind: int = 0                        # 0 min_index, 1 arbitrary
    seed: int = 0

    @staticmethod
    def min_index() -> "ElectionPolicy":
        return ElectionPolicy(0, 0)

    @staticmethod
    def arbitrary(seed: int) -> "ElectionPolicy":
        return ElectionPolicy(1, seed)


@dataclass
class Dfa:
    """dfakit::Dfa (dfa.hpp:21-41)."""

    delta: np.ndarray
    accepting: np.ndarray
    initial: Optional[int] = None
    letter_names: Optional[List[str]] = None

    def __post_init__(self):
        self.delta = np.ascontiguousarray(self.delta, dtype=np.uint32)
        if self.delta.ndim != 2:
            raise ValueError("delta must have shape (alphabet_size, num_states)")
        self.accepting = np.ascontiguousarray(self.accepting, dtype=np.uint8)
        if self.accepting.shape != (self.delta.shape[1],):
            raise ValueError("accepting must have one entry per state")

    @property
    def num_states(self) -> int:
        return int(self.delta.shape[1])

    @property
    def alphabet_size(self) -> int:
        return int(self.delta.shape[0])

    def c_view(self) -> CDfa:
        init = -1 if self.initial is None else int(self.initial)
        return CDfa(self.num_states, self.alphabet_size, self.delta.ctypes.data, self.accepting.ctypes.data, init)


@dataclass
class Partition:
    """dfakit::Partition (dfa.hpp:46-60), canonical first-occurrence numbering."""

    block_of: np.ndarray
    num_blocks: int

    def __eq__(self, other) -> bool:
        return (isinstance(other, Partition) and self.num_blocks == other.num_blocks
                and np.array_equal(self.block_of, other.block_of))


@dataclass
class RefinementReport:
    """dfakit::RefinementReport (minimize.hpp:26-35) plus device statistics."""

    partition: Partition
    refining_iterations: int
    algorithm: Algorithm
    closure_iterations: int = 0
    passes: int = 0
    transitions_refined: int = 0
    states_sorted: int = 0
    hash_collisions: int = 0
    device_ms: float = 0.0


@dataclass
class TransResult:                       # minimize.hpp:48-51
    report: RefinementReport
    apart: np.ndarray


@dataclass
class ExploreOptions:                    # equivalence.hpp:28-34
    match_letters_by_name: bool = False
    max_visited: int = K_DEFAULT_MAX_VISITED


@dataclass
class ProductResult:                     # equivalence.hpp:12-22
    verdict: Verdict
    counterexample: List[int] = field(default_factory=list)
    explored_states: int = 0
    levels: int = 0
    device_ms: float = 0.0


def _ctx(ctx: Optional[Context]) -> Context:
    return ctx if ctx is not None else default_context()


def _report(rep: CReport, blocks: np.ndarray, algo: Algorithm) -> RefinementReport:
    return RefinementReport(Partition(blocks, int(rep.num_blocks)), int(rep.refining_iterations), algo,
                            int(rep.closure_iterations), int(rep.passes), int(rep.transitions_refined),
                            int(rep.states_sorted), int(rep.hash_collisions), float(rep.device_ms))


def minimize(dfa: Dfa, algo: Algorithm, policy: ElectionPolicy = ElectionPolicy.min_index(), *,
             max_transitions: int = K_DEFAULT_MAX_TRANSITIONS, max_pair_nodes: int = K_DEFAULT_MAX_PAIR_NODES,
             force_exact: bool = False, fingerprint_bits: int = 64, grouping: str = "auto",
             ctx: Optional[Context] = None) -> RefinementReport:
    """Generic entry (dfakit_minimize); the named functions below call it.

    sort_pr knobs (testing / comparison): force_exact never uses fingerprint
    keys, fingerprint_bits < 64 forces collisions, grouping="radix_sort"
    groups keys with the full LSD radix sort of the literal Alg. 4 instead of
    the counting-table / radix-bucket hashing default, grouping="staged"
    keeps every pass host-staged (no persistent small-m device loop)."""
    view = dfa.c_view()
    blocks = np.zeros(max(dfa.num_states, 1), np.uint32)
    codes = {"auto": 0, "radix_sort": 1, "staged": 2}
    if grouping not in codes:
        raise ValueError(f"grouping must be one of {sorted(codes)}, not {grouping!r}")
    opts = COptions(policy.kind, int(force_exact), policy.seed, max_transitions, max_pair_nodes, fingerprint_bits,
                    codes[grouping])
    rep = CReport()
    check(lib.dfakit_minimize(_ctx(ctx).handle, C.byref(view), int(algo), C.byref(opts), blocks.ctypes.data,
                              C.byref(rep)))
    return _report(rep, blocks[: dfa.num_states], Algorithm(algo))


def moore_minimize(dfa: Dfa, ctx: Optional[Context] = None) -> RefinementReport:
    """minimize.hpp:46 -- same partition and pass count as Moore refinement."""
    return minimize(dfa, Algorithm.moore, ctx=ctx)


def sort_pr(dfa: Dfa, ctx: Optional[Context] = None, **kw) -> RefinementReport:
    """minimize.hpp:72 -- sorting-based partition refinement (Alg. 4)."""
    return minimize(dfa, Algorithm.sort_pr, ctx=ctx, **kw)


def naive_pr(dfa: Dfa, policy: ElectionPolicy = ElectionPolicy.min_index(),
             ctx: Optional[Context] = None) -> RefinementReport:
    """minimize.hpp:62 -- leader-election refinement (Alg. 2)."""
    return minimize(dfa, Algorithm.naive_pr, policy, ctx=ctx)


def naive_pr_fused(dfa: Dfa, ctx: Optional[Context] = None) -> RefinementReport:
    """minimize.hpp:66 -- single-pass election + reassignment (Alg. 3)."""
    return minimize(dfa, Algorithm.naive_pr_fused, ctx=ctx)


def trans_pr(dfa: Dfa, policy: ElectionPolicy = ElectionPolicy.min_index(),
             max_transitions: int = K_DEFAULT_MAX_TRANSITIONS, ctx: Optional[Context] = None) -> RefinementReport:
    """minimize.hpp:82 -- naive_pr on the pointer-doubled alphabet (Alg. 5)."""
    return minimize(dfa, Algorithm.trans_pr, policy, max_transitions=max_transitions, ctx=ctx)


def trans_minimize(dfa: Dfa, max_pair_nodes: int = K_DEFAULT_MAX_PAIR_NODES,
                   ctx: Optional[Context] = None) -> TransResult:
    """minimize.hpp:55 -- pair-graph closure (Alg. 1), small n only."""
    view = dfa.c_view()
    n = dfa.num_states
    blocks = np.zeros(max(n, 1), np.uint32)
    apart = np.zeros(max(n * n, 1), np.uint8)
    rep = CReport()
    check(lib.dfakit_trans_minimize(_ctx(ctx).handle, C.byref(view), max_pair_nodes, blocks.ctypes.data,
                                    apart.ctypes.data, C.byref(rep)))
    return TransResult(_report(rep, blocks[:n], Algorithm.trans), apart[: n * n].reshape(n, n).astype(bool))


def build_transitive_alphabet(dfa: Dfa, max_transitions: int = K_DEFAULT_MAX_TRANSITIONS,
                              ctx: Optional[Context] = None) -> Dfa:
    """minimize.hpp:77 -- letters a^(2^i); names "<base>^1", "^2", "^4", ..."""
    view = dfa.c_view()
    kk = C.c_uint32()
    check(lib.dfakit_build_transitive_alphabet(_ctx(ctx).handle, C.byref(view), max_transitions, None,
                                               C.byref(kk)))
    out = np.empty((kk.value, dfa.num_states), np.uint32)
    check(lib.dfakit_build_transitive_alphabet(_ctx(ctx).handle, C.byref(view), max_transitions,
                                               out.ctypes.data, C.byref(kk)))
    k = dfa.alphabet_size
    levels = kk.value // k if k else 1
    names = []
    for a in range(k):
        base = dfa.letter_names[a] if dfa.letter_names else ("a" if k == 1 else f"a{a}")
        names += [f"{base}^{1 << i}" for i in range(levels)]
    return Dfa(out, dfa.accepting.copy(), dfa.initial, names)


def _letter_mapping(a: Dfa, b: Dfa, opts: ExploreOptions) -> Optional[np.ndarray]:
    """equivalence.cpp:87-123 -- identity, or by letter name."""
    if not opts.match_letters_by_name:
        if a.alphabet_size != b.alphabet_size:
            raise ValueError(f"alphabet size mismatch: {a.alphabet_size} vs {b.alphabet_size}")
        return None
    if a.letter_names is None or b.letter_names is None:
        raise ValueError("matching letters by name requires letter names on both inputs")
    if a.alphabet_size != b.alphabet_size:
        raise ValueError("letter name sets differ in size")
    of_b = {}
    for i, name in enumerate(b.letter_names):
        if name in of_b:
            raise ValueError(f"duplicate letter name '{name}'")
        of_b[name] = i
    used = set()
    out = np.empty(a.alphabet_size, np.uint32)
    for i, name in enumerate(a.letter_names):
        if name not in of_b:
            raise ValueError(f"letter '{name}' has no counterpart")
        if of_b[name] in used:
            raise ValueError(f"duplicate letter name '{name}'")
        used.add(of_b[name])
        out[i] = of_b[name]
    return out


def explore_product(a: Dfa, b: Dfa, mode: ExploreMode, opts: Optional[ExploreOptions] = None,
                    ctx: Optional[Context] = None) -> ProductResult:
    """equivalence.hpp:41 -- naive Hopcroft-Karp over the product (Alg. 6)."""
    opts = opts or ExploreOptions()
    if a.initial is None or b.initial is None:
        raise ValueError("product exploration requires initial states on both inputs")
    mapping = _letter_mapping(a, b, opts)
    va, vb = a.c_view(), b.c_view()
    cap = 1 << 16
    cex = np.zeros(cap, np.uint32)
    out = CProduct()
    check(lib.dfakit_explore_product(_ctx(ctx).handle, C.byref(va), C.byref(vb), int(mode),
                                     None if mapping is None else mapping.ctypes.data, opts.max_visited,
                                     cex.ctypes.data, cap, C.byref(out)))
    word = [int(x) for x in cex[: min(out.counterexample_len, cap)]]
    return ProductResult(Verdict(out.verdict), word, int(out.explored_states), int(out.levels), float(out.device_ms))


def check_equiv(a: Dfa, b: Dfa, opts: Optional[ExploreOptions] = None, ctx: Optional[Context] = None):
    """equivalence.hpp:45"""
    return explore_product(a, b, ExploreMode.equivalence, opts, ctx)


def check_inclusion(a: Dfa, b: Dfa, opts: Optional[ExploreOptions] = None, ctx: Optional[Context] = None):
    """equivalence.hpp:48"""
    return explore_product(a, b, ExploreMode.inclusion, opts, ctx)


def check_equiv_uf(a: Dfa, b: Dfa, ctx: Optional[Context] = None) -> ProductResult:
    """Hopcroft-Karp with a GPU union-find (paper §6 future work)."""
    if a.initial is None or b.initial is None:
        raise ValueError("equivalence checking requires initial states on both inputs")
    va, vb = a.c_view(), b.c_view()
    cap = 1 << 16
    cex = np.zeros(cap, np.uint32)
    out = CProduct()
    check(lib.dfakit_check_equiv_uf(_ctx(ctx).handle, C.byref(va), C.byref(vb), cex.ctypes.data, cap,
                                    C.byref(out)))
    word = [int(x) for x in cex[: min(out.counterexample_len, cap)]]
    return ProductResult(Verdict(out.verdict), word, int(out.explored_states), int(out.levels), float(out.device_ms))
