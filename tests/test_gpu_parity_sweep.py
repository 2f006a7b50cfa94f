"""A seeded randomised parity sweep (tools/parity_sweep.py) as part of the
GPU suite: random automata with duplicated states and forced fingerprint
collisions through the production sortPR paths (speculative second pass,
lazy apply, record-free buckets, packed and sliced labels forced onto small
inputs), and product explorations (primary table, 64-slot hash table) --
every result equal to the oracle's."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_randomised_parity_sweep():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import parity_sweep
    msgs = []
    bad = parity_sweep.sweep(300, 2026, log=msgs.append)
    assert bad == 0, msgs[-20:]
