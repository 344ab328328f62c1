"""Measured layers in the reference's experiment wire format.

``moeplan``'s experiment runner writes one CSV row per (scenario, strategy,
layer) with the columns of ``CSV_COLUMNS`` (reference experiment.py:26-39,
rows formatted by ``ResultRow.csv_values``, experiment.py:60-69, written by
``csv_text``, experiment.py:314-320). :func:`measured_rows` turns a
``bench.py`` line -- the device-measured dispatch / combine / layer times of
the Aurora schedule and of the SJF / RCS baselines executed by the same
engine -- into rows of that format, in the reference's time unit (one token
over one link direction at B = 1: hidden x 2 B / 900 GB/s), so measured
results sit in the same files as the reference's simulated ones.
"""
from __future__ import annotations

import csv
import io
from dataclasses import dataclass, field

__all__ = ["CSV_COLUMNS", "MeasuredRow", "csv_text", "measured_rows", "time_unit_us"]

CSV_COLUMNS = (
    "scenario", "strategy", "layer", "n", "noise_level", "seed", "comm_makespan_first",
    "comm_makespan_second", "inference_time", "utilization", "oracle_time", "oracle_ratio",
)


@dataclass(frozen=True)
class MeasuredRow:
    """One CSV row (the fields of the reference's ResultRow, experiment.py:45-58)."""

    scenario: str
    strategy: str
    layer: int
    n: int
    noise_level: float
    seed: int
    comm_makespan_first: float
    comm_makespan_second: float
    inference_time: float
    utilization: float
    oracle_time: float | None = None
    oracle_ratio: float | None = None
    timeline: dict = field(default_factory=dict)

    def csv_values(self) -> list:
        def fmt(v) -> str:
            if v is None:
                return ""
            if isinstance(v, float):
                return repr(v)
            return str(v)

        return [fmt(getattr(self, c)) for c in CSV_COLUMNS]


def csv_text(rows) -> str:
    """Same bytes as the reference's experiment.csv_text for the same rows."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(CSV_COLUMNS)
    for r in rows:
        w.writerow(r.csv_values())
    return buf.getvalue()


def time_unit_us(hidden: int, link_gbs: float = 900.0) -> float:
    """The reference's time unit for this layer: one token over one link direction."""
    return hidden * 2 / (link_gbs * 1e9) * 1e6


def measured_rows(line: dict) -> list:
    """Rows for a bench.py line: strategy ``aurora`` (the layer as run, dispatch and
    combine as timed by the staged pass) plus every baseline schedule the bench
    executed on the same engine (``all_to_all.baseline_schedules_on_engine``).
    Times in the reference's unit; ``utilization`` = the expert GEMMs' share of the
    step (the busy-compute fraction of sim.py's TimelineResult)."""
    cfg, a2a = line["config"], line["all_to_all"]
    tau = time_unit_us(cfg["hidden"])
    scenario = "exclusive-hetero" if "bandwidths" in cfg else "exclusive-homo"
    util = float(line.get("roofline", {}).get("gemm_share_of_step") or 0.0)
    step_us = line["ms_per_step"] * 1e3
    base = dict(scenario=scenario, layer=0, n=cfg["ranks"], noise_level=0.0, seed=cfg["seed"])
    rows = [MeasuredRow(strategy="aurora", comm_makespan_first=a2a["dispatch_us"] / tau,
                        comm_makespan_second=a2a["combine_us"] / tau, inference_time=step_us / tau,
                        utilization=util, **base)]
    for name, r in sorted(a2a.get("baseline_schedules_on_engine", {}).items()):
        # the baseline's layer = the measured Aurora step with its own all-to-all times swapped in
        t = step_us - a2a["dispatch_us"] - a2a["combine_us"] + r["dispatch_us"] + r["combine_us"]
        rows.append(MeasuredRow(strategy=name, comm_makespan_first=r["dispatch_us"] / tau,
                                comm_makespan_second=r["combine_us"] / tau, inference_time=t / tau,
                                utilization=util * step_us / t, **base))
    return rows
