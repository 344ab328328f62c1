import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# The reference package: the offline install under baseline/_ref (git-ignored, it travels
# to the GPU box with the snapshot), else its sources in the build container.
REFERENCE_PATHS = (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "reference: needs the reference package importable")


def reference_path():
    for p in REFERENCE_PATHS:
        if os.path.isdir(os.path.join(p, "moeplan")):
            return p
    return None


def reference_available() -> bool:
    return reference_path() is not None


@pytest.fixture(scope="session")
def moeplan():
    p = reference_path()
    if p is None:
        pytest.skip("reference package moeplan not installed (baseline/_ref) or present")
    if p not in sys.path:
        sys.path.insert(0, p)
    import moeplan as m
    return m
