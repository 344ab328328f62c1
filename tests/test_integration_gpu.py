"""The reference-side binding exactly as INTEGRATION.md ships it
(integration/moeplan_b200.py: ctypes + the C ABI, no import of this repo's
package): bit-identical schedules and the reference simulator's timelines."""
import importlib.util
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def binding(moeplan):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    spec = importlib.util.spec_from_file_location("moeplan_b200", os.path.join(ROOT, "integration", "moeplan_b200.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_binding_schedule_and_timelines(binding, moeplan):
    rng = np.random.default_rng(3)
    for case in range(40):
        n = int(rng.choice([2, 4, 8, 8, 16]))
        pop = 1.0 / (rng.permutation(n) + 1.0) ** rng.uniform(0, 2)
        d = np.round(np.outer(rng.uniform(500, 2500, n), pop / pop.sum()) * rng.uniform(0.9, 1.1, (n, n)))
        if case % 3 == 0:
            d = rng.random((n, n)) * 1000
        cl = (moeplan.ClusterSpec(tuple(moeplan.GpuSpec(float(b), float(b)) for b in rng.choice([1.0, .8, .5, .4], n)))
              if case % 4 == 0 else moeplan.ClusterSpec.uniform(n))
        tm = moeplan.TrafficMatrix(d)
        ref = moeplan.build_schedule(tm, cl)
        got = binding.build_schedule(tm, cl)
        assert type(got) is moeplan.commsched.CommSchedule
        assert [(p.transfers, p.duration) for p in got.phases] == [(p.transfers, p.duration) for p in ref.phases]
        assert got.makespan == ref.makespan
        prof = moeplan.LayerProfile(1.0, 1.0, 0.3, 0.0, tm)
        plan = moeplan.DeploymentPlan.identity(n)
        a = moeplan.simulate_exclusive(prof, plan, cl)
        b = moeplan.simulate_exclusive(prof, plan, cl, schedule_fn=binding.build_schedule)
        assert a.inference_time == b.inference_time and a.spans == b.spans
    with pytest.raises(ValueError):
        binding.build_schedule(moeplan.TrafficMatrix(np.ones((4, 4))), moeplan.ClusterSpec.uniform(3))
