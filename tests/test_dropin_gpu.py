"""The drop-in through the reference's own objects: ``moeplan`` (installed
under baseline/_ref) calls the device scheduler K2 as its ``ScheduleFn``
(reference sim.py:48) or with its module-level ``build_schedule`` rebound,
and cannot tell the difference: same classes, same phases, same timelines,
same experiment rows, same exceptions."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2410_17043_b200 as A
    return A


def _moe_counts(rng, n, skew):
    """Integer MoE routing counts (Zipf popularity, workload.py:49-52)."""
    pop = 1.0 / (rng.permutation(n) + 1.0) ** skew
    d = np.round(np.outer(rng.uniform(1500, 2500, n), pop / pop.sum()) * rng.uniform(0.9, 1.1, (n, n)))
    np.fill_diagonal(d, 0)
    return d


def _same(s_ref, s_dev, moeplan):
    assert type(s_dev) is moeplan.commsched.CommSchedule
    assert all(type(p) is moeplan.commsched.Phase for p in s_dev.phases)
    assert s_dev.n == s_ref.n
    assert [(p.transfers, p.duration) for p in s_dev.phases] == [(p.transfers, p.duration) for p in s_ref.phases]
    assert s_dev.makespan == s_ref.makespan


def test_build_schedule_returns_reference_objects(A, moeplan):
    """build_schedule(moeplan.TrafficMatrix, moeplan.ClusterSpec) returns
    moeplan.commsched.CommSchedule / Phase, phase for phase equal to
    moeplan.build_schedule (commsched.py:291-324) -- homogeneous integer,
    heterogeneous fp64 and real-valued matrices, n = 2..16."""
    rng = np.random.default_rng(0)
    for case in range(60):
        n = int(rng.choice([2, 3, 4, 8, 8, 8, 16]))
        d = _moe_counts(rng, n, rng.uniform(0, 2)) if case % 3 else rng.random((n, n)) * 1000
        if case % 4 == 0:
            bw = rng.choice([100.0, 80.0, 50.0, 40.0], n)
            cl = moeplan.ClusterSpec(tuple(moeplan.GpuSpec(float(b)) for b in bw))
        else:
            cl = moeplan.ClusterSpec.uniform(n)
        tm = moeplan.TrafficMatrix(d)
        ref = moeplan.build_schedule(tm, cl)
        dev = A.build_schedule(tm, cl)
        _same(ref, dev, moeplan)
        assert moeplan.validate_schedule(dev, tm, cl).ok
        # the combine schedule (CommSchedule.reversed, commsched.py:153-162) on the returned object
        assert [(p.transfers, p.duration) for p in dev.reversed().phases] == \
               [(p.transfers, p.duration) for p in ref.reversed().phases]


def test_simulate_exclusive_with_device_schedule_fn(A, moeplan):
    """simulate_exclusive(profile, plan, cluster, schedule_fn=A.build_schedule)
    (sim.py:130-154) gives the same timeline as the reference's own scheduler,
    for homogeneous and heterogeneous clusters and non-identity plans."""
    for seed in range(6):
        n = 8
        spec = moeplan.SyntheticWorkloadSpec(n=n, skew=0.4 * seed, total_tokens=16384.0, seed=seed)
        prof = moeplan.generate_workload(spec).layers[0]
        if seed % 2:
            cl = moeplan.ClusterSpec(tuple(moeplan.GpuSpec(b, b) for b in (1.0, 1.0, 0.8, 0.8, 0.5, 0.5, 0.4, 0.4)))
            plan = moeplan.assign_exclusive_hetero(moeplan.expert_loads(prof), cl)
        else:
            cl = moeplan.ClusterSpec.uniform(n)
            plan = moeplan.DeploymentPlan.identity(n)
        ref = moeplan.simulate_exclusive(prof, plan, cl)
        dev = moeplan.simulate_exclusive(prof, plan, cl, schedule_fn=A.build_schedule)
        assert dev.inference_time == ref.inference_time
        assert dev.spans == ref.spans
        assert np.array_equal(dev.per_gpu_utilization, ref.per_gpu_utilization)


def test_experiment_with_build_schedule_rebound(A, moeplan, monkeypatch):
    """Full replacement: rebind the module-level build_schedule names the
    reference imports (sim.py:23, experiment.py:19, cli.py:19) to the device
    scheduler and run the reference's own experiment driver
    (experiment.run_experiment, experiment.py:293-311): identical result rows."""
    import moeplan.cli as mcli
    import moeplan.experiment as mexp
    cfg_kw = dict(strategies=("aurora", "sjf"), seed=3)
    prof = moeplan.generate_workload(moeplan.SyntheticWorkloadSpec(n=8, skew=1.2, total_tokens=4096.0,
                                                                   layer_count=3, seed=3))
    configs = [
        moeplan.ExperimentConfig("exclusive-homo", moeplan.ClusterSpec.uniform(8), (prof,), **cfg_kw),
        moeplan.ExperimentConfig("exclusive-hetero",
                                 moeplan.ClusterSpec(tuple(moeplan.GpuSpec(b, b) for b in
                                                           (1.0, 1.0, 0.8, 0.8, 0.5, 0.5, 0.4, 0.4))),
                                 (prof,), **cfg_kw),
    ]
    ref_rows = [mexp.run_experiment(c) for c in configs]
    calls = []

    def device_schedule(d, cluster):
        calls.append(d.n)
        return A.build_schedule(d, cluster)

    for mod in (moeplan.commsched, moeplan.sim, mexp, mcli):
        if hasattr(mod, "build_schedule"):
            monkeypatch.setattr(mod, "build_schedule", device_schedule)
    dev_rows = [mexp.run_experiment(c) for c in configs]
    assert calls, "the device scheduler was not called"
    for (r_rows, r_err), (d_rows, d_err) in zip(ref_rows, dev_rows):
        assert r_err == d_err == []
        assert [r.csv_values() for r in r_rows] == [r.csv_values() for r in d_rows]
        assert [r.timeline for r in r_rows] == [r.timeline for r in d_rows]


def test_layer_traffic_through_reference_scheduler(A, moeplan):
    """The matrix a real layer forward built on the device (K1) handed to the
    reference: moeplan.build_schedule on it equals the schedule K2 computed
    inside the layer (in-layer int32 path), and the layer's DeploymentPlan
    relabelling matches deploy_to_gpus (core.py:337-345) on destinations."""
    import torch
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg = MoEConfig(hidden=512, ffn=256, experts=8, top_k=2, tokens=4096, ranks=8, skew=1.5, seed=2)
    layer = AuroraMoELayer(cfg, A.DeploymentPlan((5, 2, 7, 0, 1, 3, 6, 4)))
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    layer(x)
    torch.cuda.synchronize()
    layer.check_status()
    counts = layer.counts.cpu().numpy().astype(float)
    ref = moeplan.build_schedule(moeplan.TrafficMatrix(counts), moeplan.ClusterSpec.uniform(8))
    got = layer.schedule_objects()
    assert [(p.transfers, p.duration) for p in got.phases] == [(p.transfers, p.duration) for p in ref.phases]
    assert got.makespan == ref.makespan
    # destinations relabelled by the plan: column e of the expert-space matrix lands on rank plan[e]
    from oracle.oracle import pack_oracle
    idx = layer.topk_idx.cpu().numpy()
    by_expert, _, _ = pack_oracle(idx, list(range(8)), 8)
    if cfg.top_k == 2:  # distinct experts per token, one expert per rank: no dedupe differences
        moved = np.zeros_like(by_expert)
        for e, g in enumerate(layer.plan.assignment_a):
            moved[:, g] = by_expert[:, e]
        assert np.array_equal(moved, layer.counts.cpu().numpy())
