"""Aurora all-to-all scheduling, computed by the K2 CUDA kernel.

Drop-in for ``moeplan.commsched`` (reference ``pkg/src/moeplan/commsched.py``):
``build_schedule(d, cluster) -> CommSchedule`` has the reference's signature,
return type, exceptions and -- for every input the reference accepts with
n <= 32 -- bit-identical phases, durations and makespan. It is a valid
``ScheduleFn`` (reference ``sim.py:48``), e.g.::

    moeplan.simulate_exclusive(layer, plan, cluster, schedule_fn=build_schedule)

When handed the reference's own objects (anything whose type lives in the
``moeplan`` package) it returns the reference's ``CommSchedule``/``Phase``
classes and raises the reference's ``DecompositionError``, so the caller
cannot tell the difference except by speed.

The schedule itself is never computed on the host: the shim copies the
matrix to the GPU, runs ``aurora_schedule_f64`` and reads the tables back.
"""
from __future__ import annotations

import importlib
import math
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _lib
from .core import ClusterSpec, TrafficMatrix

__all__ = [
    "TIME_ATOL", "Phase", "CommSchedule", "DecompositionError", "ScheduleReport", "ScheduleFn",
    "bmax_homogeneous", "time_normalize_entries", "bmax_heterogeneous", "build_schedule",
    "decompose_raw", "validate_schedule", "schedule_tables",
]

TIME_ATOL = 1e-9  # commsched.py:40


@dataclass(frozen=True)
class Phase:
    """Concurrent transfers, distinct senders and receivers (commsched.py:113-123)."""

    transfers: tuple
    duration: float

    def senders(self) -> tuple:
        return tuple(s for s, _ in self.transfers)

    def receivers(self) -> tuple:
        return tuple(r for _, r in self.transfers)


@dataclass(frozen=True)
class CommSchedule:
    """Ordered contention-free phases (commsched.py:126-162)."""

    n: int
    phases: tuple
    makespan: float

    def per_pair_totals(self) -> np.ndarray:
        tot = np.zeros((self.n, self.n))
        for ph in self.phases:
            for s, r in ph.transfers:
                tot[s, r] += ph.duration
        return tot

    def completion_times(self) -> np.ndarray:
        finish = np.zeros(self.n)
        clock = 0.0
        for ph in self.phases:
            clock += ph.duration
            for s, r in ph.transfers:
                finish[s] = clock
                finish[r] = clock
        return finish

    def reversed(self) -> "CommSchedule":
        """Flip every transfer (the combine all-to-all); phases keep their order."""
        flipped = tuple(Phase(tuple(sorted((r, s) for s, r in ph.transfers)), ph.duration)
                        for ph in self.phases)
        return CommSchedule(self.n, flipped, self.makespan)


class DecompositionError(RuntimeError):
    """No perfect matching on the positive support / phase bound exceeded (commsched.py:165-166)."""


ScheduleFn = Callable[[TrafficMatrix, ClusterSpec], CommSchedule]


def bmax_homogeneous(d, bandwidth: float) -> float:
    """max(max row sum, max col sum) / B (commsched.py:169-178)."""
    if not bandwidth > 0:
        raise ValueError(f"bandwidth must be positive, got {bandwidth}")
    e = np.asarray(d.entries)
    return float(max(e.sum(axis=1).max(), e.sum(axis=0).max()) / bandwidth)


def time_normalize_entries(d, cluster) -> np.ndarray:
    """d_ij / min(B_i, B_j) (commsched.py:181-190), as a plain array."""
    if cluster.n != d.n:
        raise ValueError(f"cluster has {cluster.n} GPUs, matrix has {d.n}")
    b = np.asarray(cluster.bandwidths, dtype=float)
    t = np.asarray(d.entries, dtype=float) / np.minimum.outer(b, b)
    if np.isnan(t).any() or (t < 0).any():
        raise ValueError("time matrix entries must be non-negative")
    t = t.copy()
    np.fill_diagonal(t, 0.0)
    return t


def bmax_heterogeneous(t) -> float:
    """Largest per-GPU send or receive time (commsched.py:193-195)."""
    e = np.asarray(getattr(t, "entries", t), dtype=float)
    return float(max(e.sum(axis=1).max(), e.sum(axis=0).max()))


# ------------------------------------------------------------------ device --

def _reference_flavour(d):
    """If the caller passed moeplan objects, answer with moeplan classes."""
    mod = type(d).__module__ or ""
    if mod.split(".")[0] == "moeplan":
        return importlib.import_module("moeplan.commsched")
    return None


def schedule_tables(entries: np.ndarray, bandwidths: np.ndarray | None):
    """Run K2 on the GPU. Returns (status, raw_perm[R,n], raw_dur[R], phase_recv[P,n],
    phase_dur[P], b_max) as host numpy arrays."""
    import torch

    n = int(entries.shape[0])
    _check_n(n)
    L = _lib.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    # the reference's arrays are read-only (core.py:30-33): copy, never alias
    d = torch.tensor(np.array(entries, dtype=np.float64), device=dev)
    bw = None if bandwidths is None else torch.tensor(np.array(bandwidths, dtype=np.float64), device=dev)
    R, P = L.aurora_raw_phase_cap(n), L.aurora_phase_cap(n)
    i32 = dict(dtype=torch.int32, device=dev)
    f64 = dict(dtype=torch.float64, device=dev)
    raw_perm = torch.empty(max(R, 1) * n, **i32)
    raw_dur = torch.empty(max(R, 1), **f64)
    phase_recv = torch.empty(P * n, **i32)
    phase_dur = torch.empty(P, **f64)
    scal_i = torch.zeros(3, **i32)  # n_raw, n_phases, status
    bmax = torch.zeros(1, **f64)
    rc = L.aurora_schedule_f64(d.data_ptr(), None if bw is None else bw.data_ptr(), n,
                               raw_perm.data_ptr(), raw_dur.data_ptr(), scal_i[0:].data_ptr(),
                               phase_recv.data_ptr(), phase_dur.data_ptr(), scal_i[1:].data_ptr(),
                               bmax.data_ptr(), scal_i[2:].data_ptr(), _lib.stream_ptr())
    _lib.check(rc, "aurora_schedule_f64")
    n_raw, n_ph, status = (int(v) for v in scal_i.cpu())
    return (status,
            raw_perm[: n_raw * n].view(n_raw, n).cpu().numpy(), raw_dur[:n_raw].cpu().numpy(),
            phase_recv[: n_ph * n].view(n_ph, n).cpu().numpy(), phase_dur[:n_ph].cpu().numpy(),
            float(bmax.item()))


MAX_RANKS = 32  # K2 keeps one matrix row per lane of a warp (include/aurora_b200.h)


def _check_n(n: int) -> None:
    """The reference schedules any n; the device scheduler stops at a warp's
    32 lanes. Larger clusters are refused at the boundary (ValueError, the
    reference's class for inputs it cannot take) instead of falling back to a
    host scheduler -- see INTEGRATION.md."""
    if n > MAX_RANKS:
        raise ValueError(f"the device scheduler supports n <= {MAX_RANKS} GPUs, got {n}")


def _run(d, cluster):
    ref = _reference_flavour(d)
    if cluster.n != d.n:
        raise ValueError(f"cluster has {cluster.n} GPUs, matrix has {d.n}")
    _check_n(d.n)
    entries = np.asarray(d.entries, dtype=float)
    bw = np.asarray(cluster.bandwidths, dtype=float)
    status, raw_perm, raw_dur, phase_recv, phase_dur, b_max = schedule_tables(entries, bw)
    if status == _lib.AURORA_EINVAL:
        raise ValueError("time matrix entries must be non-negative / augmented matrix unbalanced")
    if status in (_lib.AURORA_EOVERFLOW, _lib.AURORA_ENOMATCH):
        err = ref.DecompositionError if ref else DecompositionError
        msg = ("decomposition exceeded the phase bound" if status == _lib.AURORA_EOVERFLOW
               else "no perfect matching on the positive support")
        raise err(msg)
    if status != _lib.AURORA_OK:
        raise _lib.AuroraLibraryError(f"scheduler status {status}")
    return ref, raw_perm, raw_dur, phase_recv, phase_dur, b_max


def build_schedule(d, cluster) -> CommSchedule:
    """Contention-free all-to-all schedule with makespan == b_max (commsched.py:291-324).

    Computed on the GPU by K2; bit-exact with the reference.
    """
    ref, _, _, phase_recv, phase_dur, _ = _run(d, cluster)
    PhaseT = ref.Phase if ref else Phase
    SchedT = ref.CommSchedule if ref else CommSchedule
    phases = tuple(
        PhaseT(tuple((i, int(j)) for i, j in enumerate(row) if j >= 0), float(dur))
        for row, dur in zip(phase_recv, phase_dur))
    return SchedT(d.n, phases, math.fsum(p.duration for p in phases))


def decompose_raw(d, cluster) -> list:
    """The raw permutation phases ``decompose(augment(time_normalize(d)))``
    returns (commsched.py:237-278), computed by the same kernel."""
    _, raw_perm, raw_dur, _, _, _ = _run(d, cluster)
    return [(tuple(int(v) for v in perm), float(dur)) for perm, dur in zip(raw_perm, raw_dur)]


@dataclass(frozen=True)
class ScheduleReport:
    """Violations found by validate_schedule (commsched.py:169-195)."""

    contention: tuple = ()
    conservation: tuple = ()
    optimality: tuple = ()

    @property
    def contention_ok(self) -> bool:
        return not self.contention

    @property
    def conservation_ok(self) -> bool:
        return not self.conservation

    @property
    def optimal(self) -> bool:
        return not self.optimality

    @property
    def ok(self) -> bool:
        return self.contention_ok and self.conservation_ok and self.optimal

    def issues(self) -> tuple:
        return self.contention + self.conservation + self.optimality


def validate_schedule(s, d, cluster, atol: float = TIME_ATOL) -> ScheduleReport:
    """Contention / conservation / optimality check (commsched.py:355-398)."""
    contention, conservation, optimality = [], [], []
    for k, ph in enumerate(s.phases):
        if ph.duration < 0:
            contention.append(f"phase {k}: negative duration {ph.duration}")
        snd = [a for a, _ in ph.transfers]
        rcv = [b for _, b in ph.transfers]
        if len(set(snd)) != len(snd):
            contention.append(f"phase {k}: a sender transmits to two receivers at once")
        if len(set(rcv)) != len(rcv):
            contention.append(f"phase {k}: a receiver accepts two senders at once")
        contention.extend(f"phase {k}: self-loop transfer {a}->{b}" for a, b in ph.transfers if a == b)
    t = time_normalize_entries(d, cluster)
    got = np.zeros((s.n, s.n))
    for ph in s.phases:
        for a, b in ph.transfers:
            got[a, b] += ph.duration
    for i, j in zip(*np.nonzero(np.abs(got - t) > atol)):
        conservation.append(f"pair ({i}, {j}): delivered {got[i, j]:.12g}, demanded {t[i, j]:.12g}")
    total = math.fsum(p.duration for p in s.phases)
    if abs(total - s.makespan) > atol:
        conservation.append(f"makespan {s.makespan:.12g} != sum of phase durations {total:.12g}")
    b_max = bmax_heterogeneous(t)
    if abs(s.makespan - b_max) > atol:
        optimality.append(f"makespan {s.makespan:.12g} != minimum time {b_max:.12g}")
    return ScheduleReport(tuple(contention), tuple(conservation), tuple(optimality))


# ---------------------------------------------------------------- wire format
def schedule_payload(s, d, cluster) -> dict:
    """One strategy's entry of ``moeplan schedule``'s JSON output
    (cli.py:75-100): makespan, phases as {duration, transfers}, and the
    validate_schedule verdicts (commsched.py:355-398)."""
    rep = validate_schedule(s, d, cluster)
    return {"makespan": s.makespan,
            "phases": [{"duration": p.duration, "transfers": [list(t) for t in p.transfers]} for p in s.phases],
            "contention_free": rep.contention_ok, "complete": rep.conservation_ok, "optimal": rep.optimal}


def schedule_from_payload(payload: dict, n: int) -> CommSchedule:
    """Inverse of :func:`schedule_payload`: a CommSchedule (e.g. one written by
    the reference CLI) the engine can execute through ``AuroraMoELayer.load_schedule``."""
    phases = tuple(Phase(tuple(sorted((int(a), int(b)) for a, b in ph["transfers"])), float(ph["duration"]))
                   for ph in payload["phases"])
    return CommSchedule(n, phases, float(payload["makespan"]))
