"""The C-ABI library: loads, exports every symbol include/aurora_b200.h declares,
and the product path refuses to run without a GPU (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "aurora_b200.h")).read()
    return sorted(set(re.findall(r"^\s*int\s+(aurora_\w+)\s*\(", hdr, flags=re.M)))


def test_library_exports_header():
    from paper_2410_17043_b200 import _lib
    assert os.path.exists(_lib.LIB_PATH), "run `python __graft_entry__.py` first"
    so = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(so, s), s
    assert set(syms) == set(_lib.exported_symbols())
    L = _lib.load(require_cuda=False)
    assert L.aurora_version() >= 1
    assert L.aurora_raw_phase_cap(8) == 50 and L.aurora_phase_cap(8) == 106


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2410_17043_b200 as A
    from paper_2410_17043_b200._lib import AuroraLibraryError
    with pytest.raises(AuroraLibraryError):
        A.build_schedule(A.TrafficMatrix([[0, 1], [1, 0]]), A.ClusterSpec.uniform(2))
