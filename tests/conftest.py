"""Shared test setup.

* ``gpu`` marker: tests that need a B200 (the driver runs ``-m gpu`` on one).
* ``oracle`` fixture: the CPU checker (oracle/oracle.py, test infrastructure).
* ``ref`` fixture: the unmodified reference package built into oracle/_ref
  (skipped where it was not built).
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests", "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)

REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def ref():
    if not os.path.isdir(os.path.join(REF_DIR, "splatct")):
        pytest.skip("reference not built into oracle/_ref")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import splatct.raster  # noqa: F401
    import splatct
    return splatct
