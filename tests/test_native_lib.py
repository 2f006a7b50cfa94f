"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every entry point include/dfakit_b200.h declares, and refuses to compute
without a device (there is no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dfakit_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(dfakit_\w+)\s*\(", text, re.M)))


def test_header_declares_the_reference_entry_points():
    names = declared_functions()
    for must in ("dfakit_moore_minimize", "dfakit_sort_pr", "dfakit_naive_pr", "dfakit_naive_pr_fused",
                 "dfakit_trans_pr", "dfakit_trans_minimize", "dfakit_build_transitive_alphabet",
                 "dfakit_explore_product", "dfakit_check_equiv", "dfakit_check_inclusion",
                 "dfakit_check_equiv_uf"):
        assert must in names


def test_library_exports_every_declared_symbol(dk):
    lib = ctypes.CDLL(dk.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", dk.LIB_PATH], capture_output=True, text=True).stdout
    for n in declared_functions():
        assert re.search(rf"\bT {n}\b", out), n


def test_python_mirror_binds_every_export(dk):
    assert set(declared_functions()) == set(dk.EXPORTS)


def test_abi_version(dk):
    assert dk.lib.dfakit_abi_version() == 2


def test_library_carries_sm100a_code(dk):
    out = subprocess.run(["cuobjdump", "--list-elf", dk.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_means_no_compute(dk):
    if dk.device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(dk.NoDeviceError):
        dk.Context(0)
    d = dk.Dfa(np.zeros((1, 3), np.uint32), np.array([0, 1, 0], np.uint8), 0)
    with pytest.raises(dk.NoDeviceError):
        dk.sort_pr(d)


def test_dfa_validation_and_letter_mapping(dk):
    with pytest.raises(ValueError):
        dk.Dfa(np.zeros((1, 3), np.uint32), np.zeros(2, np.uint8))
    a = dk.Dfa(np.zeros((2, 1), np.uint32), np.zeros(1, np.uint8), 0, ["f", "t"])
    b = dk.Dfa(np.zeros((2, 1), np.uint32), np.zeros(1, np.uint8), 0, ["t", "f"])
    m = dk._letter_mapping(a, b, dk.ExploreOptions(match_letters_by_name=True))
    assert list(m) == [1, 0]
    c = dk.Dfa(np.zeros((2, 1), np.uint32), np.zeros(1, np.uint8), 0, ["f", "x"])
    with pytest.raises(ValueError):
        dk._letter_mapping(a, c, dk.ExploreOptions(match_letters_by_name=True))
    with pytest.raises(ValueError):
        dk._letter_mapping(a, dk.Dfa(np.zeros((3, 1), np.uint32), np.zeros(1, np.uint8), 0),
                           dk.ExploreOptions())


def test_pass_planner_host_only(dk):
    """dfakit_plan_pass needs no device: the key plan of the bench workload's
    passes (10M states, |Sigma| = 10) and of the small-key regimes."""
    from paper_2508_20735_b200.sharded import plan_pass, PLAN_TABLE, PLAN_PACKED, PLAN_FINGERPRINT
    p = plan_pass(10_000_000, 10, 2, 10_000_000)
    assert (p.strategy, p.field_bits, p.key_bits, p.keylab_bytes) == (PLAN_TABLE, 1, 11, 1)
    p = plan_pass(10_000_000, 10, 2000, 10_000_000)
    assert (p.strategy, p.key_bits, p.keylab_bytes) == (PLAN_FINGERPRINT, 64, 2)
    p = plan_pass(10_000_000, 10, 2000, 1000)           # small late pass: no O(n) relabel
    assert (p.strategy, p.keylab_bytes) == (PLAN_FINGERPRINT, 0)
    p = plan_pass(1000, 1, 10, 1000)                    # min-state labels pack into 20 bits
    assert (p.strategy, p.field_bits, p.keylab_bytes) == (PLAN_TABLE, 10, 0)
    p = plan_pass(5000, 3, 100, 5000)                   # 52-bit packed keys
    assert (p.strategy, p.key_bits) == (PLAN_PACKED, 52)
