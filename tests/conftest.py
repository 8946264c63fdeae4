"""Shared fixtures.  `-m "not gpu"` runs here (no GPU); `-m gpu` on a B200.

The oracle (oracle/) is the checker only; product calls go through
paper_1403_7295_b200 -> include/paes_cuda.h -> libpaes_cuda.so.
"""
from __future__ import annotations

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: multi-GiB full-size parity (still run with -m gpu)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def digests():
    path = os.path.join(GOLDEN_DIR, "digests.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/digests.json not generated")
    with open(path) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def orc():
    import oracle

    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.ref_available():
        pytest.skip("oracle/_ref (reference compiled from its sources) not built")
    return oracle.RefLib()


@pytest.fixture(scope="session")
def lib():
    from paper_1403_7295_b200 import _native

    return _native.load(build_if_missing=True)


@pytest.fixture(scope="session")
def paes(lib):
    from paper_1403_7295_b200 import paes as P

    return P


@pytest.fixture(scope="session")
def gpu(paes):
    """Fails loudly (not skip) when a -m gpu test runs without a device."""
    n = paes.device_count()
    assert n > 0, "no CUDA device visible to libpaes_cuda.so"
    import torch

    assert torch.cuda.is_available()
    return 0
