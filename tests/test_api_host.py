"""Host side of the drop-in: boundary types, placement, reversal and the
validator, checked against the reference's golden outputs."""
import numpy as np
import pytest

import paper_2410_17043_b200 as A
from golden_io import placement_cases, schedule_cases, spec_examples


def test_traffic_matrix_validation_mirrors_reference():
    with pytest.raises(ValueError):
        A.TrafficMatrix([[0, 1]])
    with pytest.raises(ValueError):
        A.TrafficMatrix([[0, np.nan], [0, 0]])
    with pytest.raises(ValueError, match=r"negative entry at \(0, 1\)"):
        A.TrafficMatrix([[0, -1], [0, 0]])
    m = A.TrafficMatrix([[5, 2], [3, 7]])
    assert m.entries.tolist() == [[0, 2], [3, 0]]
    assert not m.entries.flags.writeable
    src = np.array([[0.0, 1.0], [2.0, 0.0]])
    m = A.TrafficMatrix(src)
    src[0, 1] = 9
    assert m.entries[0, 1] == 1.0  # never aliases caller memory
    assert A.reverse_all_to_all(A.TrafficMatrix([[0, 2], [3, 0]])).entries.tolist() == \
        spec_examples()["reverse_0_2_3_0"]


def test_cluster_and_plan_validation():
    with pytest.raises(ValueError):
        A.GpuSpec(0.0)
    with pytest.raises(ValueError):
        A.ClusterSpec((A.GpuSpec(1.0, 2.0), A.GpuSpec(2.0, 1.0)))
    with pytest.raises(ValueError):
        A.ClusterSpec(())
    with pytest.raises(ValueError):
        A.DeploymentPlan((0, 0))
    p = A.DeploymentPlan.from_pairing([1, 0])
    assert p.assignment_b == (1, 0) and p.pairing == (1, 0)
    comb = A.combine_colocated(A.TrafficMatrix([[0, 1], [0, 0]]), A.TrafficMatrix([[0, 0], [2, 0]]), p)
    assert comb.entries.tolist() == spec_examples()["combine_swapped"]


def test_placement_matches_reference_goldens():
    g = placement_cases()
    for c in g["assign_exclusive_hetero"]:
        cl = A.ClusterSpec(tuple(A.GpuSpec(b, s) for b, s in zip(c["bw"], c["scales"])))
        assert list(A.assign_exclusive_hetero(c["loads"], cl).assignment_a) == c["assignment"]
    for c in g["pair_case1"]:
        pairing, h = A.pair_case1(c["a"], c["b"])
        assert list(pairing) == c["pairing"] and h.tolist() == c["h"]
    for c in g["bottleneck_matching"]:
        m = A.bottleneck_matching(c["w"])
        assert list(m.pairs) == c["pairs"] and m.bottleneck_value == c["value"]
    for c in g["hopcroft_karp"]:
        size, ml = A.hopcroft_karp(c["adj"], n_right=len(c["adj"]))
        assert size == c["size"] and [(-1 if v is None else v) for v in ml] == c["match_left"]

    def prof(p):
        return A.LayerProfile(p["gate_work"], p["agg_work"], p["ffn_work_per_token"], p["ffn_base_work"],
                              A.TrafficMatrix(p["d"]))

    for c in g["colocate_homogeneous"]:
        pl = A.colocate_homogeneous(prof(c["a"]), prof(c["b"]))
        assert list(pl.assignment_a) == c["assignment_a"] and list(pl.assignment_b) == c["assignment_b"]
        assert list(pl.pairing) == c["pairing"]
    for c in g["colocate_heterogeneous"]:
        cl = A.ClusterSpec(tuple(A.GpuSpec(b, s) for b, s in zip(c["bw"], c["scales"])))
        pl = A.colocate_heterogeneous(prof(c["a"]), prof(c["b"]), cl)
        assert list(pl.assignment_a) == c["assignment_a"] and list(pl.assignment_b) == c["assignment_b"]
    for c in g["deploy_to_gpus"]:
        assert A.deploy_to_gpus(A.TrafficMatrix(c["d"]), c["assignment"]).entries.tolist() == c["out"]
    for c in g["combine_colocated"]:
        pl = A.DeploymentPlan(tuple(c["assignment_a"]), tuple(c["assignment_b"]))
        out = A.combine_colocated(A.TrafficMatrix(c["a"]), A.TrafficMatrix(c["b"]), pl)
        assert out.entries.tolist() == c["out"]
    for c in g["expert_loads"]:
        lp = A.LayerProfile(0, 0, 0, 0, A.TrafficMatrix(c["d"]))
        assert A.expert_loads(lp).tolist() == c["loads"]


def test_spec_placement_examples():
    ex = spec_examples()
    cl = A.ClusterSpec((A.GpuSpec(1, 1), A.GpuSpec(2, 2), A.GpuSpec(4, 4)))
    assert list(A.assign_exclusive_hetero([9, 4, 1], cl).assignment_a) == ex["assign_9_4_1"]
    assert float(max(A.pair_case1([1, 3, 5], [2, 4, 6])[1])) == ex["pair_case1_135_246_hmax"]
    assert A.bottleneck_matching([[5, 4], [5, 4]]).bottleneck_value == ex["bottleneck_5454"]
    with pytest.raises(A.CaseOnePreconditionError):
        A.pair_case1(np.array([[1, 2]]), np.array([[1, 1]]))


def test_reversed_and_validator_on_golden_schedules():
    for c in schedule_cases()[:200]:
        phases = tuple(A.Phase(tuple(tuple(t) for t in tr), d) for tr, d in c["phases"])
        s = A.CommSchedule(c["n"], phases, c["makespan"])
        rev = s.reversed()
        assert [[[list(t) for t in p.transfers], p.duration] for p in rev.phases] == c["reversed"]
        assert s.completion_times().tolist() == c["completion_times"]
        cl = A.ClusterSpec(tuple(A.GpuSpec(b) for b in c["bw"]))
        assert A.validate_schedule(s, A.TrafficMatrix(c["d"]), cl).ok == c["valid"]
    # a contended schedule is reported
    bad = A.CommSchedule(3, (A.Phase(((0, 2), (1, 2)), 1.0),), 1.0)
    rep = A.validate_schedule(bad, A.TrafficMatrix([[0, 0, 1], [0, 0, 1], [0, 0, 0]]), A.ClusterSpec.uniform(3))
    assert not rep.contention_ok and not rep.optimal


def test_lina_slots_spec_example():
    """SPEC.md:444 (baselines.py:126-137): loads [8, 6, 2, 1] -> pairs (8,1), (6,2)."""
    from paper_2410_17043_b200.colocation import lina_slots
    assert lina_slots([8, 6, 2, 1]) == ((0, 3), (1, 2))
    assert lina_slots([1, 1, 1, 1]) == ((0, 3), (1, 2))
    with pytest.raises(ValueError):
        lina_slots([1, 2, 3])


@pytest.mark.reference
def test_lina_slots_vs_reference(moeplan):
    from paper_2410_17043_b200.colocation import lina_slots
    rng = np.random.default_rng(3)
    for _ in range(50):
        n = int(rng.choice([2, 4, 6, 8, 16]))
        d = rng.integers(0, 20, size=(n, n)).astype(float)
        prof = moeplan.LayerProfile(0, 0, 0, 0, moeplan.TrafficMatrix(d))
        ref = moeplan.colocate_same_model(prof)
        assert lina_slots(moeplan.TrafficMatrix(d).col_sums()) == ref


def test_baseline_schedules_fig4_and_tables():
    from paper_2410_17043_b200 import baselines as B
    fig4 = A.TrafficMatrix([[0, 1, 1], [1, 0, 1], [0, 0, 0]])
    c3 = A.ClusterSpec.uniform(3)
    naive = B.schedule_fixed_order(fig4, c3, [[1, 2], [0, 2], []])
    assert naive.makespan == spec_examples()["fig4_naive_makespan"] == 3.0
    assert A.validate_schedule(naive, fig4, c3).contention_ok
    ch, rch, n_in, n_out = B.to_engine_tables(naive, 3)
    tot = np.zeros((3, 3))
    for row in ch:
        for i, (j, first, cnt, seq) in enumerate(row):
            if j >= 0:
                tot[i, j] += cnt
    assert tot.tolist() == fig4.entries.tolist()
    assert n_in.sum() == n_out.sum()


@pytest.mark.reference
def test_baseline_schedules_vs_reference(moeplan):
    from paper_2410_17043_b200 import baselines as B
    rng = np.random.default_rng(11)
    for it in range(60):
        n = int(rng.choice([2, 3, 4, 6, 8]))
        d = (rng.integers(0, 30, size=(n, n)) * (rng.random((n, n)) < 0.7)).astype(float)
        cl_ref = moeplan.ClusterSpec.uniform(n)
        tm_ref = moeplan.TrafficMatrix(d)
        cl, tm = A.ClusterSpec.uniform(n), A.TrafficMatrix(d)
        for ref, got in ((moeplan.schedule_sjf(tm_ref, cl_ref), B.schedule_sjf(tm, cl)),
                         (moeplan.schedule_rcs(tm_ref, cl_ref, it), B.schedule_rcs(tm, cl, it))):
            assert [(p.transfers, p.duration) for p in ref.phases] == [(p.transfers, p.duration) for p in got.phases]
            assert ref.makespan == got.makespan


def test_schedule_wire_format_matches_reference_cli():
    """schedule_payload produces the reference CLI's JSON entry (cli.py:75-100)
    and round-trips through schedule_from_payload (oracle-built schedule, so
    no GPU is needed)."""
    import json
    import numpy as np
    from oracle.oracle import build_schedule_oracle
    import paper_2410_17043_b200 as A
    from paper_2410_17043_b200.commsched import CommSchedule, Phase, schedule_from_payload, schedule_payload
    rng = np.random.default_rng(5)
    d = rng.integers(0, 400, size=(6, 6)).astype(float)
    np.fill_diagonal(d, 0)
    o = build_schedule_oracle(d)
    phases = tuple(Phase(tuple(t), dur) for t, dur in o["phases"])
    s = CommSchedule(6, phases, sum(p.duration for p in phases))
    cl = A.ClusterSpec.uniform(6)
    pay = schedule_payload(s, A.TrafficMatrix(d), cl)
    assert pay["contention_free"] and pay["complete"] and pay["optimal"]
    back = schedule_from_payload(json.loads(json.dumps(pay)), 6)
    assert [(p.transfers, p.duration) for p in back.phases] == [(p.transfers, p.duration) for p in s.phases]
    try:
        import sys
        sys.path.insert(0, "/root/reference/pkg/src")
        from moeplan import commsched as RC
        from moeplan.core import ClusterSpec as RCl, TrafficMatrix as RT
    except Exception:
        return
    ref = RC.build_schedule(RT(d), RCl.uniform(6))
    rep = RC.validate_schedule(ref, RT(d), RCl.uniform(6))
    ref_pay = {"makespan": ref.makespan,
               "phases": [{"duration": p.duration, "transfers": [list(t) for t in p.transfers]} for p in ref.phases],
               "contention_free": rep.contention_ok, "complete": rep.conservation_ok, "optimal": rep.optimal}
    assert json.dumps(pay) == json.dumps(ref_pay)


def test_reference_error_classes_host(moeplan, monkeypatch):
    """Errors map to the reference's classes with the device result faked (no
    GPU): a cluster / matrix size mismatch is ValueError (commsched.py:181-190),
    a device status of phase overflow or no perfect matching is moeplan's own
    DecompositionError (commsched.py:165-166, 260-272) when the caller passed
    moeplan objects, and this package's DecompositionError otherwise."""
    import numpy as np
    import pytest
    import paper_2410_17043_b200 as A
    from paper_2410_17043_b200 import _lib, commsched as C
    tm = moeplan.TrafficMatrix(np.ones((4, 4)))
    with pytest.raises(ValueError):
        A.build_schedule(tm, moeplan.ClusterSpec.uniform(3))
    empty = (np.zeros((0, 4), np.int32), np.zeros(0), np.zeros((0, 4), np.int32), np.zeros(0), 3.0)
    for status in (_lib.AURORA_EOVERFLOW, _lib.AURORA_ENOMATCH):
        monkeypatch.setattr(C, "schedule_tables", lambda e, b, s=status: (s,) + empty)
        with pytest.raises(moeplan.commsched.DecompositionError):
            A.build_schedule(tm, moeplan.ClusterSpec.uniform(4))
        with pytest.raises(A.DecompositionError):
            A.build_schedule(A.TrafficMatrix(np.ones((4, 4))), A.ClusterSpec.uniform(4))
    monkeypatch.setattr(C, "schedule_tables", lambda e, b: (_lib.AURORA_EINVAL,) + empty)
    with pytest.raises(ValueError):
        A.build_schedule(tm, moeplan.ClusterSpec.uniform(4))
    monkeypatch.undo()
    with pytest.raises(ValueError, match="n <= 32"):  # beyond the device scheduler: a clear error, no fallback
        A.build_schedule(A.TrafficMatrix(np.ones((33, 33))), A.ClusterSpec.uniform(33))


def test_measured_rows_in_reference_csv_format(moeplan):
    """report.csv_text writes the reference's experiment CSV (experiment.py:26-39,
    314-320) byte for byte: the same rows built as moeplan.experiment.ResultRow
    and passed to its own csv_text give identical text; measured_rows reads a
    committed bench line."""
    import json
    import os
    import moeplan.experiment as mexp
    from paper_2410_17043_b200 import report
    assert report.CSV_COLUMNS == mexp.CSV_COLUMNS
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    line = json.loads(open(os.path.join(root, "profiles", "r02_bench_c2.json")).read().strip().splitlines()[-1])
    rows = report.measured_rows(line)
    assert [r.strategy for r in rows][0] == "aurora" and len(rows) >= 1
    ref_rows = [mexp.ResultRow(**{c: getattr(r, c) for c in report.CSV_COLUMNS}) for r in rows]
    assert report.csv_text(rows) == mexp.csv_text(ref_rows)


def test_colocation_hetero_plan_matches_reference(moeplan):
    """plan_colocation_hetero builds LayerProfiles with the measured-rate work model and
    places pairs by colocate_heterogeneous: the same DeploymentPlan as the reference's own
    colocate_heterogeneous (placement.py:129-157) on the same profiles and cluster."""
    import numpy as np
    from paper_2410_17043_b200.colocation import expert_work, plan_colocation_hetero
    from paper_2410_17043_b200 import ClusterSpec, GpuSpec
    rng = np.random.default_rng(11)
    bws = (1.0, 1.0, 0.8, 0.8, 0.5, 0.5, 0.4, 0.4)
    for it in range(20):
        ca = rng.integers(0, 3000, (8, 8)).astype(float)
        cb = rng.integers(0, 1500, (8, 8)).astype(float)
        wa, wb = expert_work(4096, 14336), expert_work(4096, 7168)
        slots = [(2 * i, 2 * i + 1) for i in range(8)]
        cp = plan_colocation_hetero(ca, cb, slots, ClusterSpec(tuple(GpuSpec(b, b) for b in bws)), wa, wb)
        ref = moeplan.colocate_heterogeneous(
            moeplan.LayerProfile(d_first=moeplan.TrafficMatrix(ca), **wa),
            moeplan.LayerProfile(d_first=moeplan.TrafficMatrix(cb), **wb),
            moeplan.ClusterSpec(tuple(moeplan.GpuSpec(b, b) for b in bws)))
        assert tuple(cp.plan.assignment_a) == tuple(ref.assignment_a)
        assert tuple(cp.plan.assignment_b) == tuple(ref.assignment_b)
        assert sorted(cp.gpu_of_b) == [g for g in range(8) for _ in range(2)]


def test_cluster_partition_host():
    """The emulated-compute split of the GEMM's CTA pairs: proportional (largest
    remainder), at least one pair per rank, covering every pair exactly once."""
    import pytest
    from paper_2410_17043_b200.layer import AuroraMoELayer
    part = AuroraMoELayer.cluster_partition([1.0, 1.0, 0.8, 0.8, 0.5, 0.5, 0.4, 0.4], 74)
    sizes = [b - a for a, b in zip(part, part[1:])]
    assert part[0] == 0 and part[-1] == 74 and min(sizes) >= 1
    assert sizes == sorted(sizes, reverse=True) and sizes[0] > sizes[-1]
    assert AuroraMoELayer.cluster_partition([1e-6, 1.0], 2) == [0, 1, 2]
    with pytest.raises(ValueError):
        AuroraMoELayer.cluster_partition([1.0] * 9, 8)
