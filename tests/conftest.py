"""Shared fixtures.  `-m gpu` tests need a CUDA device and call the product
through its C ABI; everything else runs on CPU (oracle vs golden fixtures,
host logic, library load/export checks, gloo multi-process tests)."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_vectors.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the product kernels")
    config.addinivalue_line("markers", "slow: full-size configuration checks")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    import pyoracle
    return pyoracle.COracle()


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref); skipped when it was not built."""
    import pyoracle
    path = os.path.join(ROOT, "oracle", "_ref", "libdfakit_ref.so")
    if not os.path.exists(path):
        try:
            pyoracle.build()
        except Exception:
            pass
    if not os.path.exists(path):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return pyoracle.RefLib(path)


@pytest.fixture(scope="session")
def dk():
    """The product package (loads libdfakit_b200.so; fails loudly if absent)."""
    import paper_2508_20735_b200 as pkg
    return pkg


def mkdfa(dk, triple):
    delta, acc, init = triple
    return dk.Dfa(delta, acc, None if init < 0 else init)


def digest(arr):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()[:32]
