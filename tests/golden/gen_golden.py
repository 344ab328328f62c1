"""Generate golden fixtures by running the REFERENCE itself (moeplan).

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_golden.py

Writes ``tests/golden/schedules.json.gz`` (build_schedule / decompose raw
permutations / phases / makespan / b_max / reversed) and
``tests/golden/placement.json.gz`` (placement and matching functions), plus
``tests/golden/spec_examples.json`` (the SPEC.md known answers). Floats are
stored with Python's repr (shortest round-trip), so the fixtures are
bit-exact. The reference is not available on the GPU box; the fixtures are
what travels.
"""
from __future__ import annotations

import gzip
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import moeplan  # noqa: E402
from moeplan import commsched, core, matching, placement  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def _sched_case(d, bw, tag):
    d = np.asarray(d, dtype=float)
    n = d.shape[0]
    cluster = core.ClusterSpec(tuple(core.GpuSpec(float(b)) for b in bw))
    tm = core.TrafficMatrix(d)
    case = {"tag": tag, "n": n, "d": tm.entries.tolist(), "bw": [float(b) for b in bw]}
    try:
        t = commsched.time_normalize(tm, cluster)
        b_max = commsched.bmax_heterogeneous(t)
        raw = commsched.decompose(commsched.augment(t)) if b_max > 0 else []
        s = commsched.build_schedule(tm, cluster)
    except Exception as exc:  # recorded, never expected on these inputs
        case["error"] = type(exc).__name__
        return case
    case["b_max"] = b_max
    case["raw"] = [[list(p), float(dur)] for p, dur in raw]
    case["phases"] = [[[list(tr) for tr in p.transfers], float(p.duration)] for p in s.phases]
    case["makespan"] = float(s.makespan)
    rev = s.reversed()
    case["reversed"] = [[[list(tr) for tr in p.transfers], float(p.duration)] for p in rev.phases]
    rep = commsched.validate_schedule(s, tm, cluster)
    case["valid"] = bool(rep.ok)
    case["completion_times"] = [float(v) for v in s.completion_times()]
    return case


def zipf_routing_counts(rng, n, tokens, k, skew):
    """Integer GPU x GPU counts from a synthetic Zipf router (E == n, identity
    placement): mirrors workload.py:49-52's popularity law on token counts."""
    ranks = rng.permutation(n)
    pop = 1.0 / (ranks + 1.0) ** skew
    pop = pop / pop.sum()
    counts = np.zeros((n, n))
    per = tokens // n
    for i in range(n):
        for _ in range(per):
            noisy = pop * rng.uniform(0.9, 1.1, size=n)
            e = rng.choice(n, size=min(k, n), replace=False, p=noisy / noisy.sum())
            for j in e:
                counts[i, j] += 1
    np.fill_diagonal(counts, 0)
    return counts


def gen_schedules():
    rng = np.random.default_rng(20241017)
    cases = []
    # Fig. 4
    cases.append(_sched_case([[0, 1, 1], [1, 0, 1], [0, 0, 0]], [1, 1, 1], "fig4"))
    cases.append(_sched_case([[0, 1, 1], [1, 0, 1], [0, 0, 0]], [1, 1, 0.5], "fig4_hetero"))
    cases.append(_sched_case([[0, 0, 5], [0, 0, 0], [0, 0, 0]], [1, 1, 1], "single_entry"))
    cases.append(_sched_case([[0, 4], [1, 0]], [1, 1], "n2"))
    cases.append(_sched_case([[0.0]], [1.0], "n1"))
    cases.append(_sched_case(np.zeros((4, 4)), [1] * 4, "zeros4"))
    # integer: Zipf MoE routing counts, small token counts per rank
    for n in (2, 3, 4, 5, 6, 8, 8, 8, 12, 16):
        for s in (0.0, 0.5, 1.0, 1.5, 2.0):
            for rep in range(3 if n <= 8 else 1):
                toks = int(rng.choice([64, 256, 1024])) * n
                c = zipf_routing_counts(rng, n, toks, 2, s)
                cases.append(_sched_case(c, [1.0] * n, f"zipf_n{n}_s{s}"))
    # integer: sparse / tied / tiny / structured
    for it in range(300):
        n = int(rng.choice([2, 3, 4, 5, 6, 7, 8, 9, 12, 16]))
        kind = it % 5
        if kind == 0:
            m = rng.integers(0, 10, size=(n, n)) * (rng.random((n, n)) < 0.3)
        elif kind == 1:
            m = np.full((n, n), int(rng.integers(1, 5)))
        elif kind == 2:
            m = rng.integers(0, 3, size=(n, n))
        elif kind == 3:
            m = rng.integers(0, 100000, size=(n, n))
        else:
            m = np.zeros((n, n))
            for _ in range(int(rng.integers(1, n + 1))):
                m[rng.integers(n), rng.integers(n)] = rng.integers(1, 50)
        cases.append(_sched_case(m.astype(float), [1.0] * n, f"int_kind{kind}"))
    # heterogeneous fp64: real-valued traffic, mixed bandwidths
    from moeplan.workload import SyntheticWorkloadSpec, generate_workload
    for it in range(200):
        n = int(rng.choice([2, 3, 4, 6, 8, 8, 12, 16]))
        sets = [[100.0, 80.0, 50.0, 40.0], [1.0, 0.8, 0.5, 0.4]]
        bw = rng.choice(sets[it % 2], size=n).tolist()
        if it % 3 == 0:
            m = rng.integers(0, 500, size=(n, n)).astype(float)
        else:
            spec = SyntheticWorkloadSpec(n=n, skew=float(rng.choice([0.0, 1.0, 2.0])),
                                         total_tokens=float(rng.choice([1000.0, 4096.0, 12345.6])),
                                         seed=int(rng.integers(1 << 30)))
            m = np.asarray(generate_workload(spec).layers[0].d_first.entries)
        cases.append(_sched_case(m, bw, "hetero"))
    # homogeneous but non-unit bandwidth (B = 900e9 / 8192 bytes per token)
    for it in range(20):
        n = 8
        c = zipf_routing_counts(rng, n, 1024 * n, 2, 1.0)
        cases.append(_sched_case(c, [900e9 / 8192] * n, "homo_bw"))
    return cases


def gen_placement():
    rng = np.random.default_rng(7)
    out = {"assign_exclusive_hetero": [], "pair_case1": [], "bottleneck_matching": [],
           "colocate_homogeneous": [], "colocate_heterogeneous": [], "hopcroft_karp": [],
           "deploy_to_gpus": [], "combine_colocated": [], "expert_loads": []}
    from moeplan.workload import SyntheticWorkloadSpec, generate_workload
    for it in range(40):
        n = int(rng.choice([2, 3, 4, 6, 8]))
        scales = rng.choice([1.0, 0.8, 0.5, 0.4], size=n)
        cluster = core.ClusterSpec(tuple(core.GpuSpec(float(s) * 100, float(s)) for s in scales))
        loads = rng.integers(0, 6, size=n).astype(float) if it % 2 else rng.random(n) * 100
        plan = placement.assign_exclusive_hetero(loads, cluster)
        out["assign_exclusive_hetero"].append({"loads": loads.tolist(), "scales": scales.tolist(),
                                               "bw": (scales * 100).tolist(),
                                               "assignment": list(plan.assignment_a)})
        a = rng.integers(0, 10, size=n).astype(float)
        b = rng.integers(0, 10, size=n).astype(float)
        pairing, h = placement.pair_case1(a, b)
        out["pair_case1"].append({"a": a.tolist(), "b": b.tolist(), "pairing": list(pairing), "h": h.tolist()})
        w = rng.integers(0, 6, size=(n, n)).astype(float) if it % 2 else rng.random((n, n))
        m = matching.bottleneck_matching(w)
        out["bottleneck_matching"].append({"w": w.tolist(), "pairs": list(m.pairs), "value": m.bottleneck_value})
        adj = [sorted(set(int(v) for v in rng.choice(n, size=int(rng.integers(0, n + 1))))) for _ in range(n)]
        size, ml = matching.hopcroft_karp(adj, n_right=n)
        out["hopcroft_karp"].append({"adj": adj, "size": size, "match_left": [(-1 if v is None else int(v)) for v in ml]})
        specs = [SyntheticWorkloadSpec(n=n, skew=float(rng.choice([0.0, 1.0, 2.0])), total_tokens=1000.0,
                                       seed=int(rng.integers(1 << 30))) for _ in range(2)]
        la, lb = (generate_workload(s).layers[0] for s in specs)
        if it % 4 == 0:  # symmetric loads -> Case I sort path (placement.py:122-123)
            sym = lambda L: core.LayerProfile(L.gate_work, L.agg_work, L.ffn_work_per_token, L.ffn_base_work,
                                              core.TrafficMatrix((L.d_first.entries + L.d_first.entries.T)))
            la, lb = sym(la), sym(lb)
        pl = placement.colocate_homogeneous(la, lb)
        prof = lambda L: {"gate_work": L.gate_work, "agg_work": L.agg_work,
                          "ffn_work_per_token": L.ffn_work_per_token, "ffn_base_work": L.ffn_base_work,
                          "d": L.d_first.entries.tolist()}
        out["colocate_homogeneous"].append({"a": prof(la), "b": prof(lb), "assignment_a": list(pl.assignment_a),
                                            "assignment_b": list(pl.assignment_b), "pairing": list(pl.pairing)})
        ph = placement.colocate_heterogeneous(la, lb, cluster)
        out["colocate_heterogeneous"].append({"a": prof(la), "b": prof(lb), "scales": scales.tolist(),
                                              "bw": (scales * 100).tolist(),
                                              "assignment_a": list(ph.assignment_a),
                                              "assignment_b": list(ph.assignment_b)})
        out["expert_loads"].append({"d": la.d_first.entries.tolist(), "loads": placement.expert_loads(la).tolist()})
        perm = [int(v) for v in rng.permutation(n)]
        dep = core.deploy_to_gpus(la.d_first, perm)
        out["deploy_to_gpus"].append({"d": la.d_first.entries.tolist(), "assignment": perm, "out": dep.entries.tolist()})
        comb = core.combine_colocated(la.d_first, lb.d_first, pl)
        out["combine_colocated"].append({"a": la.d_first.entries.tolist(), "b": lb.d_first.entries.tolist(),
                                         "assignment_a": list(pl.assignment_a), "assignment_b": list(pl.assignment_b),
                                         "out": comb.entries.tolist()})
    return out


def spec_examples():
    """SPEC.md known answers, evaluated by the reference."""
    ex = {}
    fig4 = core.TrafficMatrix([[0, 1, 1], [1, 0, 1], [0, 0, 0]])
    c3 = core.ClusterSpec.uniform(3)
    s = commsched.build_schedule(fig4, c3)
    ex["fig4_rows"] = fig4.row_sums().tolist()
    ex["fig4_cols"] = fig4.col_sums().tolist()
    ex["fig4_bmax"] = commsched.bmax_homogeneous(fig4, 1.0)
    a = commsched.augment(commsched.time_normalize(fig4, c3))
    ex["fig4_x"] = a.x.tolist()
    ex["fig4_dprime"] = a.d_prime.tolist()
    ex["fig4_phases"] = [[[list(t) for t in p.transfers], p.duration] for p in s.phases]
    ex["fig4_makespan"] = s.makespan
    ex["fig4_naive_makespan"] = moeplan.schedule_fixed_order(fig4, c3, [[1, 2], [0, 2], []]).makespan
    ex["bmax_homogeneous_0_4_1_0_B2"] = commsched.bmax_homogeneous(core.TrafficMatrix([[0, 4], [1, 0]]), 2.0)
    ch = core.ClusterSpec((core.GpuSpec(1.0), core.GpuSpec(1.0), core.GpuSpec(0.5)))
    ex["fig4_hetero_t"] = commsched.time_normalize(fig4, ch).entries.tolist()
    ex["fig4_hetero_bmax"] = commsched.bmax_heterogeneous(commsched.time_normalize(fig4, ch))
    ex["reverse_0_2_3_0"] = core.reverse_all_to_all(core.TrafficMatrix([[0, 2], [3, 0]])).entries.tolist()
    pl = placement.assign_exclusive_hetero([9, 4, 1], core.ClusterSpec(
        (core.GpuSpec(1, 1), core.GpuSpec(2, 2), core.GpuSpec(4, 4))))
    ex["assign_9_4_1"] = list(pl.assignment_a)
    ex["pair_case1_135_246_hmax"] = float(max(placement.pair_case1([1, 3, 5], [2, 4, 6])[1]))
    ex["bottleneck_5454"] = matching.bottleneck_matching([[5, 4], [5, 4]]).bottleneck_value
    ex["single_entry_phases"] = [[[list(t) for t in p.transfers], p.duration] for p in
                                 commsched.build_schedule(core.TrafficMatrix([[0, 0, 5], [0, 0, 0], [0, 0, 0]]),
                                                          c3).phases]
    swapped = core.DeploymentPlan.from_pairing([1, 0])
    ex["combine_swapped"] = core.combine_colocated(core.TrafficMatrix([[0, 1], [0, 0]]),
                                                   core.TrafficMatrix([[0, 0], [2, 0]]), swapped).entries.tolist()
    return ex


def main():
    sched = gen_schedules()
    with gzip.open(os.path.join(HERE, "schedules.json.gz"), "wt") as f:
        json.dump({"generator": "moeplan " + moeplan.__version__ + ", numpy " + np.__version__, "cases": sched}, f)
    with gzip.open(os.path.join(HERE, "placement.json.gz"), "wt") as f:
        json.dump(gen_placement(), f)
    with open(os.path.join(HERE, "spec_examples.json"), "w") as f:
        json.dump(spec_examples(), f, indent=1)
    print(f"{len(sched)} schedule cases; errors: {sum('error' in c for c in sched)}")


if __name__ == "__main__":
    main()
