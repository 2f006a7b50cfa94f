"""The LSD radix sort behind sortPR's literal Alg. 4 grouping (reference
src/minimize.cpp:392 std::stable_sort), through its C ABI entry point,
against numpy's stable sort: keys AND values identical (stability), for
empty / single / ragged sizes, narrow and full 64-bit keys, heavy
duplication and tile-boundary sizes (3072-key tiles, look-back chains)."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def sort_pairs(dk, keys, vals, bits):
    from paper_2508_20735_b200 import _native as nat
    ctx = dk.default_context()
    m = len(keys)
    k0 = torch.from_numpy(keys.view(np.int64)).cuda() if m else torch.empty(1, dtype=torch.int64, device="cuda")
    v0 = torch.from_numpy(vals.view(np.int32)).cuda() if m else torch.empty(1, dtype=torch.int32, device="cuda")
    k1, v1 = torch.empty_like(k0), torch.empty_like(v0)
    flipped = C.c_int32(-1)
    torch.cuda.synchronize()
    nat.check(nat.lib.dfakit_radix_sort_pairs_device(ctx.handle, k0.data_ptr(), v0.data_ptr(), k1.data_ptr(),
                                                     v1.data_ptr(), m, bits, C.byref(flipped), None))
    torch.cuda.synchronize()
    ko, vo = (k1, v1) if flipped.value else (k0, v0)
    return ko[:m].cpu().numpy().view(np.uint64), vo[:m].cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("m,bits,dup", [(0, 64, 0), (1, 64, 0), (2, 8, 0), (3071, 11, 0), (3072, 16, 0),
                                        (3073, 20, 0), (100_000, 64, 0), (100_003, 37, 0), (1_000_000, 64, 0),
                                        (2_000_001, 24, 1), (1_000_000, 64, 2), (5_000_000, 32, 0)])
def test_radix_sort_pairs_matches_stable_sort(dk, m, bits, dup):
    rng = np.random.default_rng(m * 131 + bits)
    mask = np.uint64((1 << bits) - 1) if bits < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    keys = rng.integers(0, 1 << 63, size=m, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, size=m, dtype=np.uint64)
    if dup == 1:
        keys = rng.integers(0, 7, size=m).astype(np.uint64)  # a few huge runs
    elif dup == 2:
        keys = (rng.integers(0, 1000, size=m).astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15))
    keys &= mask
    # bits above key_bits must be ignored by the sort: set some
    noisy = keys | (np.uint64(0xF) << np.uint64(bits)) if bits <= 60 else keys
    vals = np.arange(m, dtype=np.uint32)
    order = np.argsort(keys, kind="stable")
    got_k, got_v = sort_pairs(dk, noisy.copy(), vals, bits)
    assert np.array_equal(got_v, vals[order])
    assert np.array_equal(got_k & mask, keys[order])
