"""Receiver-serialised baseline schedules (the paper's SJF / RCS comparison,
PAPER.md:747) as CommSchedules the B200 engine can execute.

Mirrors ``moeplan.baselines`` (reference ``pkg/src/moeplan/baselines.py``):

* ``schedule_fixed_order``  baselines.py:29-74  each sender walks its own destination
  order; a busy receiver makes later arrivals wait (earliest start, then
  earliest arrival, then lowest sender first)
* ``schedule_rcs``          baselines.py:91-99  random destination order per sender
* ``schedule_sjf``          baselines.py:102-109 smallest volume first

``to_engine_tables`` turns any CommSchedule with whole-token durations into the
engine's chunk tables, so Aurora's schedule, these baselines and the unpaced
mode run on the same copy engine. Host-side: these are
offline comparison plans, not the per-batch path.
"""
from __future__ import annotations

import math
from typing import Sequence

import numpy as np

from .commsched import CommSchedule, Phase, time_normalize_entries

__all__ = ["schedule_fixed_order", "schedule_rcs", "schedule_sjf", "to_engine_tables"]


def schedule_fixed_order(d, cluster, orders: Sequence[Sequence[int]]) -> CommSchedule:
    t = time_normalize_entries(d, cluster)
    n = t.shape[0]
    pending = []
    for i, order in enumerate(orders):
        listed = set(int(j) for j in order)
        if any(int(j) not in listed for j in np.flatnonzero(t[i] > 0)):
            raise ValueError(f"order for sender {i} misses destinations with demand")
        pending.append([(int(j), float(t[i, j])) for j in order if t[i, j] > 0])
    sender_free = [0.0] * n
    receiver_free = [0.0] * n
    busy = []  # (start, end, sender, receiver)
    left = sum(len(q) for q in pending)
    while left:
        pick = None
        for i in range(n):
            if not pending[i]:
                continue
            j, dur = pending[i][0]
            arrival = sender_free[i]
            key = (max(arrival, receiver_free[j]), arrival, i)
            if pick is None or key < pick[0]:
                pick = (key, i, j, dur)
        (start, _, _), i, j, dur = pick
        end = start + dur
        busy.append((start, end, i, j))
        sender_free[i] = receiver_free[j] = end
        pending[i].pop(0)
        left -= 1
    if not busy:
        return CommSchedule(n, (), 0.0)
    edges = sorted({x for s, e, _, _ in busy for x in (s, e)})
    phases = []
    for a, b in zip(edges, edges[1:]):
        if b - a <= 0:
            continue
        active = tuple(sorted((i, j) for s, e, i, j in busy if s <= a and e >= b))
        phases.append(Phase(active, b - a))
    return CommSchedule(n, tuple(phases), math.fsum(p.duration for p in phases))


def schedule_rcs(d, cluster, seed: int) -> CommSchedule:
    rng = np.random.default_rng(seed)
    orders = []
    for i in range(d.n):
        dests = list(np.nonzero(np.asarray(d.entries)[i] > 0)[0])
        rng.shuffle(dests)
        orders.append([int(j) for j in dests])
    return schedule_fixed_order(d, cluster, orders)


def schedule_sjf(d, cluster) -> CommSchedule:
    e = np.asarray(d.entries)
    orders = [[int(j) for j in sorted(np.nonzero(e[i] > 0)[0], key=lambda j: (e[i, j], j))] for i in range(d.n)]
    return schedule_fixed_order(d, cluster, orders)


def to_engine_tables(sched: CommSchedule, n: int, ctas_d=None, ctas_c=None):
    """CommSchedule (token-unit durations) -> (chunks[P,n,4], rchunks[P,n,4],
    n_in[n], n_out[n]) in the engine's format (include/aurora_b200.h): one entry
    per phase and sender {receiver, first token, count, run code}; a run is a
    stretch of consecutive phases of one pair, coded by its hand-over threshold
    (arrival signals of the earlier runs into the receiver; ctas_d / ctas_c =
    copy CTAs per rank, each signalling once per run, default 1) on its first
    entry and -1 on continuations."""
    cd = [1] * n if ctas_d is None else list(ctas_d)
    cc = [1] * n if ctas_c is None else list(ctas_c)
    P = max(1, len(sched.phases))
    ch = np.full((P, n, 4), 0, dtype=np.int32)
    ch[:, :, 0] = -1
    rch = ch.copy()
    issued = np.zeros((n, n), dtype=np.int64)
    cum = np.zeros((n, n))
    rcnt = np.zeros(n, dtype=np.int32)
    scnt = np.zeros(n, dtype=np.int32)
    prev = [-1] * n
    for k, ph in enumerate(sched.phases):
        cur = [-1] * n
        for i, j in ph.transfers:
            cum[i, j] += ph.duration
            start = int(issued[i, j])
            tok = int(round(cum[i, j])) - start
            issued[i, j] += tok
            cont = prev[i] == j
            r = s_ = -1
            if not cont:
                r, s_ = rcnt[j], scnt[i]
                rcnt[j] += cd[i]
                scnt[i] += cc[j]
            ch[k, i] = (j, start, tok, r)
            rch[k, j] = (i, start, tok, s_)
            cur[i] = j
        prev = cur
    return ch, rch, rcnt, scnt
