"""Test configuration.

-m "not gpu": oracle vs golden vectors and vs the reference, host logic,
              the C-ABI library loads and exports every declared symbol.
-m gpu      : parity of the sm_100a engine against the oracle (needs a B200).
"""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_traces():
    return dict(np.load(os.path.join(GOLDEN, "traces.npz")))


@pytest.fixture(scope="session")
def oracle():
    from oracle.ffi import Oracle, build
    build()
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.ffi import Ref, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref (the reference compiled from /root/reference) is not built here")
    return Ref()


@pytest.fixture(scope="session")
def se():
    """The product package; on a GPU box its context must come up (no fallback)."""
    import paper_2106_15319_b200 as pkg
    pkg.context(0)
    return pkg


def fromhex(lst):
    return np.array([float.fromhex(v) for v in lst], dtype=np.float64)


def sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def sort_trace(t):
    return np.sort(t, order=["task", "m", "k", "iter"])
