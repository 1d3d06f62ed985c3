"""Shared test setup.

Markers: ``gpu`` tests need a CUDA device (run on the B200 box with
``pytest -m gpu``); everything else runs on CPU.  ``oracle/`` (the CPU
checker) and ``tests/golden`` (fixtures dumped from the reference) are put
on sys.path here — tests are the only importers of the oracle.
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build_library()
    return oracle


@pytest.fixture(scope="session")
def product():
    import paper_2408_07609_b200 as P
    return P


@pytest.fixture(scope="session")
def cuda_device():
    """The product's device; fails (does not skip) when no GPU is usable."""
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2408_07609_b200 import _native
    _native.lib()
    return 0
