"""ctypes binding of libaurora_b200.so (the C ABI declared in include/aurora_b200.h).

There is no fallback: if the library is missing or no CUDA device is visible,
every entry point raises. Build with ``python __graft_entry__.py`` (or
``make -C paper_2410_17043_b200/csrc``).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libaurora_b200.so")

AURORA_OK, AURORA_EINVAL, AURORA_EOVERFLOW, AURORA_ENOMATCH = 0, 1, 2, 3
AURORA_ECUDA, AURORA_EUNSUPPORTED, AURORA_ETIMEOUT = 10, 11, 12

_c_int, _c_i64, _vp = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p

# name -> argtypes (all pointers are passed as integers / void*)
_SIGNATURES = {
    "aurora_version": [],
    "aurora_raw_phase_cap": [_c_int],
    "aurora_phase_cap": [_c_int],
    "aurora_schedule_f64": [_vp, _vp, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "aurora_schedule_counts": [_vp, _vp, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int,
                               _c_int, _c_int, _vp],
    "aurora_route": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _c_int, _c_int,
                     _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "aurora_route_gate_floats": [_c_int, _c_int],
    "aurora_route_prepare_gate": [_vp, _c_int, _c_int, _vp, _vp],
    "aurora_route_tc_bytes": [_c_int, _c_int],
    "aurora_route_prepare_gate_tc": [_vp, _c_int, _c_int, _vp, _vp],
    "aurora_route_tc": [_vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _c_int, _c_int,
                        _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "aurora_pack": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                    _vp, _vp, _vp, _vp, _vp],
    "aurora_engine": [_c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_int,
                      _vp, _vp, _c_int, _vp, _vp, _c_int, _vp, _c_int, _c_int, _c_i64, _vp, _c_int, _vp, _vp, _vp,
                      _vp, ctypes.c_float, _vp],
    "aurora_engine_ctas": [_c_int, _c_int, _c_int, _c_int, _c_int, _c_int],
    "aurora_aggregate": [_vp, _c_i64, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int,
                         _c_int, _vp, _vp, _c_i64, _vp, _vp],
    "aurora_expert_ffn": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_i64, _c_int, _c_int, _vp, _vp, _c_int, _vp],
    "aurora_grouped_gemm": [_vp, _vp, _vp, _vp, _vp, _c_int, _c_i64, _c_int, _c_int, _c_int, _vp, _c_int, _vp],
    "aurora_expert_ffn_combine": [_vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_i64, _c_int, _c_int, _vp, _vp, _vp,
                                  _vp, _c_int, _c_int, _vp, _vp, _c_int, _vp, _vp, _c_int, _vp, _c_int, _vp],
    "aurora_exchange_counts": [_vp, _vp, _vp, _vp, _c_int, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_i64, _vp, _vp],
    "aurora_expert_hist": [_vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp],
    "aurora_pack_grouped": [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                            _vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp],
    "aurora_combine_wait": [_vp, _c_int, _c_int, _c_int, _c_int, _c_i64, _vp, _vp],
    "aurora_expert_ffn_packed": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_i64, _c_int, _c_int, _vp, _c_int, _vp,
                                 _c_int, _vp],
    "aurora_expert_sort": [_vp, _c_i64, _c_int, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp,
                           _vp, _c_int, _vp],
    "aurora_gather_rows": [_vp, _vp, _vp, _vp, _c_i64, _c_int, _vp],
    "aurora_expert_reduce": [_vp, _vp, _vp, _c_i64, _c_int, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _c_int, _vp],
    "aurora_expert_ffn_packed_scatter": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _c_int, _c_i64, _c_int, _c_int, _vp,
                                         _c_int, _vp, _vp, _vp, _vp, _c_int, _c_int, _vp, _c_i64, _c_int, _c_int,
                                         _vp, _vp, _c_int, _vp],
    "aurora_expert_reduce_combine": [_vp, _vp, _vp, _c_i64, _c_int, _vp, _c_int, _c_int, _c_int, _c_int, _vp,
                                     _vp, _vp, _vp, _vp, _c_int, _vp, _vp, _c_int, _c_int, _vp],
    "aurora_debug_schedule_cycles": [_vp, _c_int, _vp, _vp, _vp, _vp],
    "aurora_debug_set_schedule_profile": [_vp],
    "aurora_debug_set_schedule_variant": [_c_int],
    "aurora_debug_set_schedule_trace": [_vp],
    "aurora_debug_set_engine_trace": [_vp],
    "aurora_debug_set_gemm_trace": [_vp],
    "aurora_debug_set_early_rows": [_c_int],
    "aurora_ipc_handle_bytes": [],
    "aurora_ipc_get": [_vp, _vp, _vp],
    "aurora_ipc_open": [_vp, _c_i64, _vp],
    "aurora_ipc_close": [_vp],
}

_lib = None


class AuroraLibraryError(RuntimeError):
    """The CUDA library is missing or unusable; there is no CPU fallback."""


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def load(require_cuda: bool = True):
    """Load the library (cached). With ``require_cuda`` also insist on a GPU."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise AuroraLibraryError(
                f"{LIB_PATH} not built: run `python __graft_entry__.py` (nvcc, sm_100a). "
                "The Aurora B200 path has no CPU fallback.")
        L = ctypes.CDLL(LIB_PATH)
        for name, argtypes in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = argtypes
            fn.restype = ctypes.c_int
        _lib = L
    if require_cuda:
        import torch
        if not torch.cuda.is_available():
            raise AuroraLibraryError("no CUDA device visible: the Aurora B200 path runs on the GPU only")
    return _lib


def check(rc: int, what: str) -> None:
    if rc != AURORA_OK:
        raise AuroraLibraryError(f"{what} failed with code {rc}")


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
