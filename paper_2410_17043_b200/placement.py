"""Aurora deployment: expert -> GPU assignment and cross-model colocation.

Mirrors ``moeplan.placement`` (reference ``pkg/src/moeplan/placement.py``)
on the host. Placement is decided once from calibration statistics
 and consumed by the layer as ``gpu_of_expert`` tables;
it is not on the per-batch path, so there is no kernel for it.

* ``assign_exclusive_hetero``  placement.py:46-60   (Theorem 3: sort loads vs compute)
* ``pair_case1``               placement.py:63-100  (Theorem 6: sort-based pairing)
* ``colocate_homogeneous``     placement.py:109-126 (Case I sort or bottleneck matching)
* ``colocate_heterogeneous``   placement.py:129-157 (two-stage heuristic)
* ``colocated_pair_cost``      sim.py:331-356       (stage-2 matching weight)
"""
from __future__ import annotations

import numpy as np

from .core import ClusterSpec, DeploymentPlan, LoadVector
from .matching import bottleneck_matching

__all__ = [
    "LOAD_ATOL", "CaseOnePreconditionError", "expert_loads", "assign_exclusive_hetero", "pair_case1",
    "colocate_homogeneous", "colocate_heterogeneous", "colocated_pair_cost",
]

LOAD_ATOL = 1e-9


class CaseOnePreconditionError(ValueError):
    """An expert's send and receive loads differ: Case I does not apply."""


def expert_loads(profile) -> np.ndarray:
    """Tokens each expert receives: column sums of the first all-to-all."""
    return profile.d_first.col_sums()


def assign_exclusive_hetero(loads, cluster: ClusterSpec) -> DeploymentPlan:
    """k-th most loaded expert -> k-th most capable GPU; stable (lowest index first) on ties."""
    v = np.asarray(loads, dtype=float)
    if v.ndim != 1 or v.shape[0] != cluster.n:
        raise ValueError(f"expected {cluster.n} expert loads, got shape {v.shape}")
    experts_by_load = np.argsort(-v, kind="stable")
    gpus_by_speed = np.argsort(-cluster.compute_scales, kind="stable")
    gpu_of = np.empty(cluster.n, dtype=int)
    gpu_of[experts_by_load] = gpus_by_speed
    return DeploymentPlan(tuple(int(g) for g in gpu_of))


def _symmetric_column(v, name: str) -> np.ndarray:
    if isinstance(v, LoadVector) or (hasattr(v, "send") and hasattr(v, "recv")):
        arr = np.column_stack([v.send, v.recv])
    else:
        arr = np.asarray(v, dtype=float)
    if arr.ndim == 2:
        if arr.shape[1] != 2:
            raise ValueError(f"{name} must have shape (n,) or (n, 2)")
        if (np.abs(arr[:, 0] - arr[:, 1]) > LOAD_ATOL).any():
            raise CaseOnePreconditionError(f"{name}: some expert sends and receives unequal amounts")
        return arr[:, 0]
    if arr.ndim != 1:
        raise ValueError(f"{name} must have shape (n,) or (n, 2)")
    return arr


def pair_case1(a, b):
    """Pair a ascending with b descending; returns (pairing, combined load h)."""
    av, bv = _symmetric_column(a, "a"), _symmetric_column(b, "b")
    if av.shape != bv.shape:
        raise ValueError(f"length mismatch: {av.shape} vs {bv.shape}")
    pairing = np.empty(av.shape[0], dtype=int)
    pairing[np.argsort(av, kind="stable")] = np.argsort(-bv, kind="stable")
    return tuple(int(p) for p in pairing), av + bv[pairing]


def colocate_homogeneous(profile_a, profile_b) -> DeploymentPlan:
    """Minimise the largest per-GPU combined send/receive volume (placement.py:109-126)."""
    if profile_a.n != profile_b.n:
        raise ValueError(f"models disagree on n: {profile_a.n} vs {profile_b.n}")
    la = LoadVector.from_traffic(profile_a.d_first)
    lb = LoadVector.from_traffic(profile_b.d_first)
    if la.symmetric(LOAD_ATOL) and lb.symmetric(LOAD_ATOL):
        pairing, _ = pair_case1(la.send, lb.send)
    else:
        weights = np.maximum(la.send[:, None] + lb.send[None, :], la.recv[:, None] + lb.recv[None, :])
        pairing = bottleneck_matching(weights).pairs
    return DeploymentPlan.from_pairing(pairing)


def colocated_pair_cost(profile_a, expert_a: int, profile_b, expert_b: int, gpu) -> float:
    """Compute plus token time of hosting one expert of each model on `gpu` (sim.py:331-356)."""
    ra = float(profile_a.d_first.col_sums()[expert_a])
    rb = float(profile_b.d_first.col_sums()[expert_b])
    sa = float(profile_a.d_first.row_sums()[expert_a])
    sb = float(profile_b.d_first.row_sums()[expert_b])
    work = (profile_a.gate_work + profile_a.agg_work + profile_a.ffn_base_work
            + profile_a.ffn_work_per_token * ra
            + profile_b.gate_work + profile_b.agg_work + profile_b.ffn_base_work
            + profile_b.ffn_work_per_token * rb)
    return work / gpu.compute_scale + (sa + ra + sb + rb) / gpu.bandwidth


def colocate_heterogeneous(profile_a, profile_b, cluster: ClusterSpec) -> DeploymentPlan:
    """Stage 1: homogeneous pairing; stage 2: bottleneck-match pairs to GPUs (placement.py:129-157)."""
    if cluster.n != profile_a.n:
        raise ValueError(f"cluster has {cluster.n} GPUs, models have {profile_a.n} experts")
    pairing = colocate_homogeneous(profile_a, profile_b).pairing
    n = cluster.n
    cost = np.array([[colocated_pair_cost(profile_a, p, profile_b, pairing[p], cluster.gpus[g])
                      for p in range(n)] for g in range(n)])
    pair_on_gpu = bottleneck_matching(cost).pairs
    gpu_a = np.empty(n, dtype=int)
    gpu_b = np.empty(n, dtype=int)
    for g, p in enumerate(pair_on_gpu):
        gpu_a[p] = g
        gpu_b[pairing[p]] = g
    return DeploymentPlan(tuple(int(v) for v in gpu_a), tuple(int(v) for v in gpu_b))
