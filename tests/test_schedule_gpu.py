"""K2 on the GPU vs the reference (golden fixtures) and vs the oracle (fuzz)."""
import math

import numpy as np
import pytest

from golden_io import as_lists, schedule_cases, spec_examples

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2410_17043_b200 as A
    return A


def _cluster(A, bw):
    return A.ClusterSpec(tuple(A.GpuSpec(float(b)) for b in bw))


def test_device_schedule_bit_exact_on_reference_goldens(A):
    cases = schedule_cases()
    for c in cases:
        tm, cl = A.TrafficMatrix(c["d"]), _cluster(A, c["bw"])
        s = A.build_schedule(tm, cl)
        got = [[[list(t) for t in p.transfers], p.duration] for p in s.phases]
        assert got == c["phases"], c["tag"]
        assert s.makespan == c["makespan"], c["tag"]
        if c["raw"]:
            raw = A.decompose_raw(tm, cl)
            assert [[list(p), d] for p, d in raw] == c["raw"], c["tag"]
        rev = s.reversed()
        assert [[[list(t) for t in p.transfers], p.duration] for p in rev.phases] == c["reversed"]
        assert A.validate_schedule(s, tm, cl).ok


def test_device_schedule_fig4(A):
    ex = spec_examples()
    s = A.build_schedule(A.TrafficMatrix([[0, 1, 1], [1, 0, 1], [0, 0, 0]]), A.ClusterSpec.uniform(3))
    assert [[[list(t) for t in p.transfers], p.duration] for p in s.phases] == ex["fig4_phases"]
    assert s.makespan == 2.0
    empty = A.build_schedule(A.TrafficMatrix([[0.0]]), A.ClusterSpec.uniform(1))
    assert empty.phases == () and empty.makespan == 0.0


def _fuzz_matrix(rng, n, kind):
    if kind == 0:  # MoE-like integer counts
        pop = 1.0 / (rng.permutation(n) + 1.0) ** rng.uniform(0, 2)
        return np.round(np.outer(rng.uniform(200, 2000, n), pop / pop.sum()) * rng.uniform(0.9, 1.1, (n, n)))
    if kind == 1:  # sparse small ints with ties
        return rng.integers(0, 4, (n, n)) * (rng.random((n, n)) < 0.4)
    if kind == 2:  # real-valued
        return rng.random((n, n)) * 1000
    return rng.integers(0, 1 << 20, (n, n)).astype(float)


def test_device_schedule_fuzz_vs_oracle(A):
    from oracle.oracle import build_schedule_oracle
    rng = np.random.default_rng(2024)
    for it in range(400):
        n = int(rng.choice([2, 3, 4, 5, 7, 8, 8, 8, 11, 16, 24, 32]))
        kind = it % 4
        m = _fuzz_matrix(rng, n, kind).astype(float)
        bw = rng.choice([100.0, 80.0, 50.0, 40.0], size=n) if it % 5 == 0 else np.ones(n)
        tm, cl = A.TrafficMatrix(m), _cluster(A, bw)
        o = build_schedule_oracle(tm.entries, bw)
        s = A.build_schedule(tm, cl)
        assert [(p.transfers, p.duration) for p in s.phases] == o["phases"], (n, kind)
        assert s.makespan == o["makespan"]
        assert math.isclose(s.makespan, o["b_max"], rel_tol=1e-12, abs_tol=1e-9)


def test_device_schedule_errors(A):
    with pytest.raises(ValueError):
        A.build_schedule(A.TrafficMatrix(np.ones((33, 33))), A.ClusterSpec.uniform(33))
    with pytest.raises(ValueError):
        A.build_schedule(A.TrafficMatrix(np.ones((3, 3))), A.ClusterSpec.uniform(2))
