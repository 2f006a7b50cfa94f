"""ctypes binding of the C ABI in include/dfakit_b200.h.

The product has no Python or CPU implementation of any algorithm: if the
native library is missing this module raises at import time, and every call
on a machine without a CUDA device raises ``NoDeviceError``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libdfakit_b200.so")
# development only: DFAKIT_LIB_VARIANT=name loads lib/variants/libdfakit_b200_<name>.so
# (the same sources built with different compile-time tuning, `make variant`)
if os.environ.get("DFAKIT_LIB_VARIANT"):
    LIB_PATH = os.path.join(_HERE, "lib", "variants", f"libdfakit_b200_{os.environ['DFAKIT_LIB_VARIANT']}.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
        "the B200 library has no fallback implementation")

lib = C.CDLL(LIB_PATH)

DFAKIT_OK, E_INVALID, E_RESOURCE, E_CUDA, E_NODEVICE = 0, -1, -2, -3, -4


class DfakitError(RuntimeError):
    """A CUDA or internal failure inside libdfakit_b200."""


class ResourceError(DfakitError):
    """dfakit::ResourceError (reference include/dfakit/errors.hpp:21-24)."""


class NoDeviceError(DfakitError):
    """No CUDA device: the library refuses to run (there is no CPU path)."""


class CDfa(C.Structure):
    _fields_ = [("num_states", C.c_uint32), ("alphabet_size", C.c_uint32), ("delta", C.c_void_p),
                ("accepting", C.c_void_p), ("initial", C.c_int64)]


class CReport(C.Structure):
    _fields_ = [("num_blocks", C.c_uint32), ("refining_iterations", C.c_uint32), ("closure_iterations", C.c_uint32),
                ("algorithm", C.c_uint32), ("passes", C.c_uint64), ("transitions_refined", C.c_uint64),
                ("states_sorted", C.c_uint64), ("hash_collisions", C.c_uint32), ("reserved", C.c_uint32),
                ("device_ms", C.c_double)]


class CProduct(C.Structure):
    _fields_ = [("verdict", C.c_int32), ("levels", C.c_uint32), ("explored_states", C.c_uint64),
                ("counterexample_len", C.c_uint32), ("reserved", C.c_uint32), ("device_ms", C.c_double)]


class COptions(C.Structure):
    _fields_ = [("policy", C.c_uint32), ("force_exact", C.c_uint32), ("seed", C.c_uint64),
                ("max_transitions", C.c_uint64), ("max_pair_nodes", C.c_uint64), ("fingerprint_bits", C.c_uint32),
                ("grouping", C.c_uint32)]


class CPassPlan(C.Structure):
    _fields_ = [("strategy", C.c_uint32), ("field_bits", C.c_uint32), ("key_bits", C.c_uint32),
                ("keylab_bytes", C.c_uint32)]


_P = C.POINTER
_V = C.c_void_p
_sig = {
    "dfakit_abi_version": (C.c_int, []),
    "dfakit_last_error": (C.c_char_p, []),
    "dfakit_device_count": (C.c_int, []),
    "dfakit_ctx_create": (C.c_int, [C.c_int, _P(C.c_void_p)]),
    "dfakit_ctx_destroy": (None, [C.c_void_p]),
    "dfakit_ctx_stream": (C.c_void_p, [C.c_void_p]),
    "dfakit_ctx_kernel_launches": (C.c_uint64, [C.c_void_p]),
    "dfakit_profile_begin": (C.c_int, [C.c_void_p]),
    "dfakit_profile_end": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t]),
    "dfakit_minimize": (C.c_int, [C.c_void_p, _P(CDfa), C.c_int, _P(COptions), C.c_void_p, _P(CReport)]),
    "dfakit_moore_minimize": (C.c_int, [C.c_void_p, _P(CDfa), C.c_void_p, _P(CReport)]),
    "dfakit_sort_pr": (C.c_int, [C.c_void_p, _P(CDfa), C.c_void_p, _P(CReport)]),
    "dfakit_naive_pr": (C.c_int, [C.c_void_p, _P(CDfa), C.c_uint32, C.c_uint64, C.c_void_p, _P(CReport)]),
    "dfakit_naive_pr_fused": (C.c_int, [C.c_void_p, _P(CDfa), C.c_void_p, _P(CReport)]),
    "dfakit_trans_pr": (C.c_int, [C.c_void_p, _P(CDfa), C.c_uint32, C.c_uint64, C.c_uint64, C.c_void_p,
                                  _P(CReport)]),
    "dfakit_trans_minimize": (C.c_int, [C.c_void_p, _P(CDfa), C.c_uint64, C.c_void_p, C.c_void_p, _P(CReport)]),
    "dfakit_build_transitive_alphabet": (C.c_int, [C.c_void_p, _P(CDfa), C.c_uint64, C.c_void_p,
                                                   _P(C.c_uint32)]),
    "dfakit_minimize_device": (C.c_int, [C.c_void_p, _P(CDfa), C.c_int, _P(COptions), C.c_void_p, _P(CReport),
                                         C.c_void_p]),
    "dfakit_explore_product": (C.c_int, [C.c_void_p, _P(CDfa), _P(CDfa), C.c_int, C.c_void_p, C.c_uint64,
                                         C.c_void_p, C.c_uint32, _P(CProduct)]),
    "dfakit_check_equiv": (C.c_int, [C.c_void_p, _P(CDfa), _P(CDfa), C.c_uint64, C.c_void_p, C.c_uint32,
                                     _P(CProduct)]),
    "dfakit_check_inclusion": (C.c_int, [C.c_void_p, _P(CDfa), _P(CDfa), C.c_uint64, C.c_void_p, C.c_uint32,
                                         _P(CProduct)]),
    "dfakit_explore_product_device": (C.c_int, [C.c_void_p, _P(CDfa), _P(CDfa), C.c_int, C.c_void_p, C.c_uint64,
                                                C.c_void_p, C.c_uint32, _P(CProduct), C.c_void_p]),
    "dfakit_check_equiv_uf": (C.c_int, [C.c_void_p, _P(CDfa), _P(CDfa), C.c_void_p, C.c_uint32, _P(CProduct)]),
    "dfakit_check_equiv_uf_device": (C.c_int, [C.c_void_p, _P(CDfa), _P(CDfa), C.c_void_p, C.c_uint32,
                                               _P(CProduct), C.c_void_p]),
    "dfakit_gen_synth_device": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p,
                                          C.c_void_p]),
    "dfakit_gen_chain_device": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "dfakit_permute_states_device": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p,
                                               C.c_void_p, C.c_void_p, C.c_void_p, _P(C.c_uint32), C.c_void_p]),
    "dfakit_calibrate_gather": (C.c_int, [_V, C.c_uint64, C.c_uint32, C.c_uint64, _P(C.c_double)]),
    "dfakit_radix_sort_pairs_device": (C.c_int, [_V, _V, _V, _V, _V, C.c_uint64, C.c_uint32, _P(C.c_int32), _V]),
    "dfakit_comm_unique_id": (C.c_int, [_V]),
    "dfakit_comm_init": (C.c_int, [_V, _V, C.c_int, C.c_int, _P(C.c_void_p)]),
    "dfakit_comm_destroy": (None, [_V]),
    "dfakit_sort_pr_sharded": (C.c_int, [_V, _V, _P(CDfa), _V, _P(CReport), _P(C.c_uint64), _V]),
    "dfakit_sort_pr_sharded_host": (C.c_int, [_V, _V, _P(CDfa), _V, _P(CReport)]),
    "dfakit_local_hub_create": (C.c_int, [C.c_int, _P(C.c_void_p)]),
    "dfakit_local_hub_destroy": (None, [_V]),
    "dfakit_comm_init_local": (C.c_int, [_V, C.c_int, _P(C.c_void_p)]),
    # sharded sort_pr primitives (sharded.py)
    "dfakit_plan_pass": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                                   _P(CPassPlan)]),
    "dfakit_shard_init": (C.c_int, [_V, _P(CDfa), C.c_uint32, C.c_uint32, _V, _V, _P(C.c_uint32), _P(C.c_uint32),
                                    _P(C.c_uint64), _V]),
    "dfakit_shard_keylab": (C.c_int, [_V, _V, C.c_uint32, C.c_uint32, _P(CPassPlan), _V, _V]),
    "dfakit_shard_table_signature": (C.c_int, [_V, _P(CDfa), _V, _P(CPassPlan), _V, C.c_uint32, C.c_uint64, _V, _V,
                                               _V, _V]),
    "dfakit_shard_table_apply": (C.c_int, [_V, _P(CPassPlan), _V, C.c_uint32, _V, C.c_uint64, _V, _V, _V, _V, _V,
                                           _V, _V]),
    "dfakit_shard_partition": (C.c_int, [_V, _P(CDfa), _V, _P(CPassPlan), C.c_uint64, _V, C.c_uint32, C.c_uint64,
                                         C.c_uint32, _V, _V, _V]),
    "dfakit_shard_group": (C.c_int, [_V, _P(CDfa), _V, _P(CPassPlan), _V, C.c_uint64, _V, _V, _V]),
    "dfakit_shard_apply": (C.c_int, [_V, _V, _V, C.c_uint64, _V, _V, _V]),
    "dfakit_shard_compact": (C.c_int, [_V, _V, C.c_uint32, C.c_uint32, _V, _V, _V]),
    "dfakit_shard_canonical": (C.c_int, [_V, _V, C.c_uint32, _V, _P(C.c_uint32), _V]),
}
EXPORTS = tuple(_sig)
for _name, (_res, _args) in _sig.items():
    if os.environ.get("DFAKIT_LIB_VARIANT") and not hasattr(lib, _name):
        continue  # development variants may predate an export
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def check(status: int) -> None:
    if status == DFAKIT_OK:
        return
    msg = (lib.dfakit_last_error() or b"").decode(errors="replace")
    if status == E_INVALID:
        raise ValueError(msg)
    if status == E_RESOURCE:
        raise ResourceError(msg)
    if status == E_NODEVICE:
        raise NoDeviceError(msg)
    raise DfakitError(msg)


class Context:
    """One device, one CUDA stream, one stream-ordered memory pool."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib.dfakit_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    @property
    def stream(self) -> int:
        return lib.dfakit_ctx_stream(self.handle) or 0

    @property
    def kernel_launches(self) -> int:
        return int(lib.dfakit_ctx_kernel_launches(self.handle))

    def close(self) -> None:
        if self.handle:
            lib.dfakit_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass


_ctx_lock = threading.Lock()
_contexts: dict = {}


def default_context(device: int = 0) -> Context:
    with _ctx_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = Context(device)
            _contexts[device] = ctx
        return ctx


def device_count() -> int:
    return int(lib.dfakit_device_count())
