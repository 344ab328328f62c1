"""moeplan/_b200.py -- the binding a maintainer adds on the reference side.

Binds the B200 scheduler (K2, ``aurora_schedule_f64`` in libaurora_b200.so,
declared in include/aurora_b200.h) behind the reference's ``ScheduleFn``
(``moeplan/sim.py:48``): ``build_schedule(d, cluster) -> CommSchedule`` with
the reference's own classes and errors (``moeplan/commsched.py:113-166``).
Only ctypes + the C ABI -- it does not import this repository's Python package.

    from moeplan import _b200
    moeplan.simulate_exclusive(profile, plan, cluster, schedule_fn=_b200.build_schedule)

Library location: ``$AURORA_B200_LIB``, else the repo's in-tree build.
"""
import ctypes
import math
import os

import numpy as np
import torch  # device buffers + the current stream

from moeplan.commsched import CommSchedule, DecompositionError, Phase

_HERE = os.path.dirname(os.path.abspath(__file__))
_PATH = os.environ.get("AURORA_B200_LIB",
                       os.path.join(os.path.dirname(_HERE), "paper_2410_17043_b200", "libaurora_b200.so"))
_lib = ctypes.CDLL(_PATH)
_vp, _i = ctypes.c_void_p, ctypes.c_int
_lib.aurora_schedule_f64.argtypes = [_vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.aurora_schedule_f64.restype = _i
_lib.aurora_raw_phase_cap.argtypes = [_i]
_lib.aurora_phase_cap.argtypes = [_i]

# return / status codes (include/aurora_b200.h)
_OK, _EINVAL, _EOVERFLOW, _ENOMATCH = 0, 1, 2, 3


def build_schedule(d, cluster) -> CommSchedule:
    """Contention-free schedule of ``d`` on ``cluster``, computed on the GPU;
    bit-identical to ``moeplan.commsched.build_schedule`` (commsched.py:291-324)."""
    n = d.n
    if cluster.n != n:
        raise ValueError(f"cluster has {cluster.n} GPUs, matrix has {n}")
    if n > 32:
        raise ValueError(f"the device scheduler supports n <= 32 GPUs, got {n}")
    dev = torch.device("cuda")
    D = torch.as_tensor(np.array(d.entries, dtype=np.float64), device=dev)  # a copy: inputs stay read-only
    B = torch.as_tensor(np.asarray(cluster.bandwidths, dtype=np.float64), device=dev)
    R, P = _lib.aurora_raw_phase_cap(n), _lib.aurora_phase_cap(n)
    raw_perm = torch.empty(max(R, 1) * n, dtype=torch.int32, device=dev)
    raw_dur = torch.empty(max(R, 1), dtype=torch.float64, device=dev)
    recv = torch.empty(P * n, dtype=torch.int32, device=dev)
    dur = torch.empty(P, dtype=torch.float64, device=dev)
    s = torch.zeros(3, dtype=torch.int32, device=dev)  # n_raw, n_phases, status
    bmax = torch.zeros(1, dtype=torch.float64, device=dev)
    rc = _lib.aurora_schedule_f64(D.data_ptr(), B.data_ptr(), n, raw_perm.data_ptr(), raw_dur.data_ptr(),
                                  s.data_ptr(), recv.data_ptr(), dur.data_ptr(), s[1:].data_ptr(),
                                  bmax.data_ptr(), s[2:].data_ptr(), torch.cuda.current_stream().cuda_stream)
    if rc != _OK:
        raise RuntimeError(f"aurora_schedule_f64 failed to launch ({rc})")
    _, n_ph, status = s.tolist()
    if status == _EINVAL:
        raise ValueError("time matrix entries must be non-negative")
    if status in (_EOVERFLOW, _ENOMATCH):
        raise DecompositionError("device decomposition failed")
    rows = recv[: n_ph * n].view(n_ph, n).tolist()
    phases = tuple(Phase(tuple((i, j) for i, j in enumerate(r) if j >= 0), float(t))
                   for r, t in zip(rows, dur[:n_ph].tolist()))
    return CommSchedule(n, phases, math.fsum(p.duration for p in phases))
