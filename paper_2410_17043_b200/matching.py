"""Host-side bipartite matching for deployment planning.

Deployment (expert placement) is computed once per model from calibration
statistics, off the per-batch path, so it runs on the host.
These mirror ``moeplan.matching`` (reference ``pkg/src/moeplan/matching.py``)
with the same traversal order, hence the same matchings:

* ``hopcroft_karp``  matching.py:20-72  (full BFS layering, index-order DFS)
* ``bottleneck_matching``  matching.py:123-157  (binary search over distinct weights)

The per-batch schedule's matchings run on the GPU (csrc/schedule.cu).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

__all__ = ["hopcroft_karp", "bottleneck_matching", "Matching"]

_UNREACHED = -1


def hopcroft_karp(adjacency: Sequence[Sequence[int]], n_right: int | None = None):
    """(size, match_left) of a maximum matching; match_left[u] is None when unmatched."""
    n_left = len(adjacency)
    if n_right is None:
        n_right = 1 + max((v for row in adjacency for v in row), default=-1)
    mate_l = [None] * n_left
    mate_r = [None] * n_right
    layer = [0] * n_left

    def layering() -> bool:
        frontier = [u for u in range(n_left) if mate_l[u] is None]
        for u in range(n_left):
            layer[u] = 0 if mate_l[u] is None else _UNREACHED
        hit_free = False
        head = 0
        while head < len(frontier):
            u = frontier[head]
            head += 1
            for v in adjacency[u]:
                w = mate_r[v]
                if w is None:
                    hit_free = True
                elif layer[w] == _UNREACHED:
                    layer[w] = layer[u] + 1
                    frontier.append(w)
        return hit_free

    def augment_from(root: int) -> bool:
        # explicit stack of [vertex, next adjacency index, right vertex taken];
        # the acceptance test is evaluated when a candidate is reached, as in
        # the recursive formulation; on success the whole path is rematched
        path = [[root, 0, None]]
        while path:
            frame = path[-1]
            u, k = frame[0], frame[1]
            adj = adjacency[u]
            if k == len(adj):
                layer[u] = _UNREACHED
                path.pop()
                continue
            frame[1] = k + 1
            v = adj[k]
            w = mate_r[v]
            if w is None or layer[w] == layer[u] + 1:
                frame[2] = v
                if w is None:
                    for uu, _, vv in path:
                        mate_l[uu] = vv
                        mate_r[vv] = uu
                    return True
                path.append([w, 0, None])
        return False

    size = 0
    while layering():
        for u in range(n_left):
            if mate_l[u] is None and augment_from(u):
                size += 1
    return size, mate_l


@dataclass(frozen=True)
class Matching:
    """pairs[left] = right, and the largest selected weight (matching.py:115-120)."""

    pairs: tuple
    bottleneck_value: float


def bottleneck_matching(weights) -> Matching:
    """Perfect matching minimising the maximum selected weight (matching.py:123-157)."""
    w = np.asarray(weights, dtype=float)
    if w.ndim != 2 or w.shape[0] != w.shape[1] or w.shape[0] < 1:
        raise ValueError(f"weights must be a square matrix, got shape {w.shape}")
    if not np.isfinite(w).all():
        raise ValueError("weights must be finite")
    n = w.shape[0]
    levels = np.unique(w)

    def graph(th):
        return [list(np.flatnonzero(w[i] <= th)) for i in range(n)]

    lo, hi = 0, len(levels) - 1
    while lo < hi:
        mid = (lo + hi) // 2
        if hopcroft_karp(graph(levels[mid]), n_right=n)[0] == n:
            hi = mid
        else:
            lo = mid + 1
    _, mate = hopcroft_karp(graph(float(levels[lo])), n_right=n)
    pairs = tuple(int(v) for v in mate)
    return Matching(pairs, float(max(w[i, j] for i, j in enumerate(pairs))))
