"""Two MoE models colocated on the same GPUs per Aurora's colocation plan (config C3).

Aurora pairs one expert of model a with one expert (slot) of model b on every
GPU so that the combined per-GPU send/receive volume is balanced
(``colocate_homogeneous``, reference placement.py:109-126; the combined matrix
is ``combine_colocated``, core.py:348-367). Model b here has twice as many
experts as there are GPUs, so its experts are first grouped into GPU "slots"
of two with the reference's same-model pairing (``colocate_same_model``,
baselines.py:126-137: most loaded with least loaded), and the slots are what
gets paired with model a -- the policy SURVEY.md §7 hard part 7 lays out.

Execution: each model runs its own :class:`~paper_2410_17043_b200.layer.AuroraMoELayer`
over the same ranks -- model a with one expert per rank, model b with its two
experts per rank as placed by the plan -- so the experts of both models that
share a GPU run as that GPU's tcgen05 grouped GEMMs.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .commsched import bmax_heterogeneous
from .core import DeploymentPlan, LayerProfile, TrafficMatrix, combine_colocated
from .placement import colocate_heterogeneous, colocate_homogeneous

__all__ = ["lina_slots", "ColocationPlan", "plan_colocation", "plan_colocation_hetero", "combined_bmax",
           "ColocatedLayers", "expert_work"]


def lina_slots(expert_loads) -> tuple:
    """Pair a model's most loaded expert with its least loaded one (baselines.py:126-137).

    Returns ``((e_hi, e_lo), ...)`` in slot order; ties resolve to the lower index
    (stable sort on -load)."""
    loads = np.asarray(expert_loads, dtype=float)
    E = loads.shape[0]
    if E % 2:
        raise ValueError(f"same-model pairing needs an even expert count, got {E}")
    order = np.argsort(-loads, kind="stable")
    return tuple((int(order[k]), int(order[E - 1 - k])) for k in range(E // 2))


def _profile(counts) -> LayerProfile:
    return LayerProfile(0.0, 0.0, 0.0, 0.0, TrafficMatrix(np.asarray(counts, dtype=float)))


@dataclass(frozen=True)
class ColocationPlan:
    plan: DeploymentPlan     # model a expert i on GPU assignment_a[i]; model-b slot s on assignment_b[s]
    slots: tuple             # model-b expert pairs, one slot per GPU
    gpu_of_a: tuple          # rank of every model-a expert
    gpu_of_b: tuple          # rank of every model-b expert

    @property
    def n(self) -> int:
        return self.plan.n


def plan_colocation(counts_a, slot_counts_b, slots) -> ColocationPlan:
    """``counts_a``: model a's GPU x GPU matrix with expert i on rank i;
    ``slot_counts_b``: model b's matrix with slot s on rank s (both from a
    calibration pass). Aurora's pairing (placement.py:109-126), model a on
    identity GPUs (DeploymentPlan.from_pairing, core.py:279-287)."""
    plan = colocate_homogeneous(_profile(counts_a), _profile(slot_counts_b))
    gpu_of_b = [0] * (2 * len(slots))
    for s, (e1, e2) in enumerate(slots):
        gpu_of_b[e1] = gpu_of_b[e2] = plan.assignment_b[s]
    return ColocationPlan(plan, tuple(slots), tuple(plan.assignment_a), tuple(gpu_of_b))


def expert_work(hidden: int, ffn: int, gemm_tflops: float = 1480.0, gate_agg_us: float = 13.4) -> dict:
    """LayerProfile work parameters (core.py:194-221) in the reference's time unit -- one
    token over one link direction, hidden x 2 B / 900 GB/s -- from measured device rates:
    an expert row costs 2 * 3 * hidden * ffn FLOPs at the expert GEMMs' measured rate
    (profiles/r02_bench_c2.json: 1.48 PFLOP/s), gate + aggregation ~13 us per rank
    (router + pack + aggregate of one rank's 2048 tokens)."""
    tau_us = hidden * 2 / 900e9 * 1e6
    row_us = 6.0 * hidden * ffn / (gemm_tflops * 1e12) * 1e6
    return {"gate_work": gate_agg_us / 2 / tau_us, "agg_work": gate_agg_us / 2 / tau_us,
            "ffn_work_per_token": row_us / tau_us, "ffn_base_work": 0.0}


def plan_colocation_hetero(counts_a, slot_counts_b, slots, cluster, work_a: dict, work_b: dict) -> ColocationPlan:
    """Aurora's heterogeneous colocation (placement.py:129-157): the homogeneous pairing,
    then pairs onto GPUs by bottleneck matching on colocated_pair_cost (sim.py:331-356),
    which weighs each pair's expert work by the GPU's compute_scale and its tokens by the
    GPU's bandwidth. ``work_*``: LayerProfile work fields of each model (expert_work)."""
    pa = LayerProfile(d_first=TrafficMatrix(np.asarray(counts_a, dtype=float)), **work_a)
    pb = LayerProfile(d_first=TrafficMatrix(np.asarray(slot_counts_b, dtype=float)), **work_b)
    plan = colocate_heterogeneous(pa, pb, cluster)
    gpu_of_b = [0] * (2 * len(slots))
    for s_, (e1, e2) in enumerate(slots):
        gpu_of_b[e1] = gpu_of_b[e2] = plan.assignment_b[s_]
    return ColocationPlan(plan, tuple(slots), tuple(plan.assignment_a), tuple(gpu_of_b))


def combined_bmax(counts_a, slot_counts_b, plan: DeploymentPlan) -> float:
    """b_max of both models' traffic under the plan (the colocated all-to-all bound,
    experiment.py:172-179)."""
    comb = combine_colocated(TrafficMatrix(np.asarray(counts_a, float)),
                             TrafficMatrix(np.asarray(slot_counts_b, float)), plan)
    return bmax_heterogeneous(comb.entries)


class ColocatedLayers:
    """Model a (one expert per rank) and model b (two experts per rank) on the
    same ranks, placed by a :class:`ColocationPlan`."""

    def __init__(self, cfg_a, cfg_b, cplan: ColocationPlan, *, interleave: Optional[bool] = None, **kw):
        import torch

        from .layer import AuroraMoELayer
        if cfg_a.ranks != cfg_b.ranks or cfg_b.experts != 2 * cfg_a.ranks or cfg_a.experts != cfg_a.ranks:
            raise ValueError("expects model a with one expert per rank and model b with two")
        self.cplan = cplan
        self.a = AuroraMoELayer(cfg_a, DeploymentPlan(cplan.gpu_of_a), **kw)
        self.b = AuroraMoELayer(cfg_b, None, gpu_of_expert=cplan.gpu_of_b, **kw)
        emulated = self.a.gemm_part is not None or self.b.gemm_part is not None
        if interleave is None:
            # not under the per-rank compute emulation (compute_scales): the two models' FFNs
            # would overlap on different SMs, handing every emulated GPU twice its CTA pairs
            interleave = os.environ.get("AURORA_C3_INTERLEAVE", "1") != "0" and not emulated
        elif interleave and emulated:
            raise ValueError("interleaving would break the per-rank compute emulation (compute_scales)")
        self.interleave = interleave
        self.side = torch.cuda.Stream(device=self.a.dev)
        self._ev = {k: torch.cuda.Event() for k in ("start", "n_a", "n_b", "b_done")}

    def forward(self, x_a, x_b, out_a=None, out_b=None):
        """One layer of each model. Serial (``interleave=False``): model a's whole
        layer, then model b's. Interleaved (default): the one-GPU form of the paper's
        Table 1 (the reference simulates it in
        sim.simulate_colocated, sim.py:192-257). Model b runs on a second stream:
        its gate G_b and its schedule (K2) beside model a's gate, K2 and dispatch
        N_a; its dispatch N_b right after N_a, so both all-to-alls form one dispatch
        window (the two copy engines never overlap: each waits on all of its own
        CTAs); then F_a, and F_b behind it with model a's aggregation A_a beside F_b.
        The combines C_a / C_b run inside the FFNs' last kernels (fused combine).
        Where one GPU differs from Table 1: N_b cannot hide under F_a here, because
        the dispatch is executed by SMs that the persistent GEMM holds."""
        import torch
        if not self.interleave:
            return self.a(x_a, out=out_a), self.b(x_b, out=out_b)
        for m in (self.a, self.b):
            if not m.combine_in_gemm or m.arrival_on or m.overlap:
                raise ValueError("interleaving needs the fused combine, no N1 and no AURORA_OVERLAP on both models")
        self.a._check_out(out_a, x_a)
        self.b._check_out(out_b, x_b)
        main = torch.cuda.current_stream(self.a.dev)
        ev = self._ev
        ev["start"].record(main)
        self.side.wait_event(ev["start"])
        self.a.front(x_a)                                       # G_a
        with torch.cuda.stream(self.side):
            self.b.front(x_b)                                   # G_b beside G_a
        self.a.send(dispatched=ev["n_a"])                       # K2_a + N_a
        with torch.cuda.stream(self.side):
            self.b.send(dispatch_after=ev["n_a"], dispatched=ev["n_b"])  # K2_b beside N_a, then N_b
        ya = self.a.finish(out_a, experts_after=ev["n_b"])     # F_a (+C_a), A_a
        with torch.cuda.stream(self.side):
            yb = self.b.finish(out_b)                           # F_b (+C_b), A_b
        ev["b_done"].record(self.side)
        main.wait_event(ev["b_done"])
        return ya, yb

    __call__ = forward

    def timeline(self, x_a, x_b) -> dict:
        """One traced forward of both models: ms from model a's start to each
        stage point of each model (the measured counterpart of the Table-1 spans)."""
        import torch
        pts = self.a.TRACE_POINTS
        self.a.trace = {k: torch.cuda.Event(enable_timing=True) for k in pts}
        self.b.trace = {k: torch.cuda.Event(enable_timing=True) for k in pts}
        try:
            self.forward(x_a, x_b)
            torch.cuda.synchronize(self.a.dev)
            t0 = self.a.trace["start"]
            return {name: {k: round(t0.elapsed_time(e), 4) for k, e in m.trace.items() if k in m._marked}
                    for name, m in (("a", self.a), ("b", self.b))}
        finally:
            self.a.trace = self.b.trace = None

    def check_status(self) -> None:
        self.a.check_status()
        self.b.check_status()
