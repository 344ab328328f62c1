"""Host mirror of csrc/apportion.cuh (bit-identical integer arithmetic): how a
process's copy CTAs are split among the ranks it drives. Used to build engine
tables on the host (baselines.to_engine_tables) with the same hand-over
thresholds K2 writes on the device."""
from __future__ import annotations

SPLIT_EVEN, SPLIT_VOLUME, SPLIT_BANDWIDTH = 0, 1, 2


def apportion(counts, n: int, n_local: int, ctot: int, mode: int, combine: bool, bw=None) -> list:
    C = [0] * n
    for g0 in range(0, n, n_local):
        m = n_local
        w = []
        for r in range(m):
            i = g0 + r
            v = 1
            if mode == SPLIT_VOLUME:
                v = sum(int(counts[q][i]) if combine else int(counts[i][q]) for q in range(n))
            elif mode == SPLIT_BANDWIDTH and bw is not None:
                v = int(float(bw[i]) * 1024.0 + 0.5)
            w.append(max(v, 0))
        W = sum(w)
        spare = ctot - m
        if W == 0 or spare <= 0:
            for r in range(m):
                C[g0 + r] = ctot // m + (1 if r < ctot % m else 0)
            continue
        rem = []
        given = 0
        for r in range(m):
            q = spare * w[r] // W
            rem.append(spare * w[r] - q * W)
            C[g0 + r] = 1 + q
            given += q
        for _ in range(spare - given):
            best = 0
            for r in range(1, m):
                if rem[r] > rem[best]:
                    best = r
            C[g0 + best] += 1
            rem[best] = -1
    return C
