"""The CPU oracle, pinned against the reference's own outputs (golden fixtures)
and, where the reference is importable, against it live."""
import numpy as np
import pytest

from golden_io import as_lists, schedule_cases, spec_examples
from oracle.oracle import build_schedule_oracle, numpy_row_sums, pack_oracle, router_oracle


@pytest.fixture(scope="module")
def cases():
    return schedule_cases()


def test_oracle_matches_reference_goldens(cases):
    assert len(cases) > 600
    for c in cases:
        o = build_schedule_oracle(c["d"], c["bw"])
        assert [[list(p), d] for p, d in o["raw"]] == c["raw"], c["tag"]
        assert as_lists(o["phases"]) == c["phases"], c["tag"]
        assert o["makespan"] == c["makespan"] and o["b_max"] == c["b_max"], c["tag"]


def test_oracle_spec_fig4():
    ex = spec_examples()
    o = build_schedule_oracle([[0, 1, 1], [1, 0, 1], [0, 0, 0]])
    assert as_lists(o["phases"]) == ex["fig4_phases"]
    assert o["makespan"] == ex["fig4_makespan"] == 2.0
    assert o["raw"] == [((1, 2, 0), 1.0), ((2, 0, 1), 1.0)]
    o = build_schedule_oracle([[0, 0, 5], [0, 0, 0], [0, 0, 0]])
    assert as_lists(o["phases"]) == ex["single_entry_phases"]
    h = build_schedule_oracle([[0, 1, 1], [1, 0, 1], [0, 0, 0]], [1, 1, 0.5])
    assert h["b_max"] == ex["fig4_hetero_bmax"] == 4.0
    assert h["t"].tolist() == ex["fig4_hetero_t"]


def test_numpy_summation_order_restated():
    rng = np.random.default_rng(1)
    for n in range(1, 40):
        m = rng.random((n, n)) * 10 ** rng.uniform(-3, 3, size=(n, n))
        assert numpy_row_sums(m).tolist() == m.sum(axis=1).tolist()


@pytest.mark.reference
def test_oracle_vs_reference_live_fuzz(moeplan):
    from moeplan import ClusterSpec, GpuSpec, TrafficMatrix, build_schedule
    from moeplan.commsched import augment, decompose, time_normalize
    rng = np.random.default_rng(99)
    for it in range(150):
        n = int(rng.integers(1, 11))
        hetero = it % 3 == 0
        m = rng.integers(0, 40, size=(n, n)).astype(float) * (rng.random((n, n)) < rng.uniform(0.2, 1))
        if hetero:
            m = m * rng.random((n, n)) * 3
        bw = rng.choice([1.0, 0.8, 0.5, 0.4], size=n) if hetero else np.ones(n)
        cl = ClusterSpec(tuple(GpuSpec(float(b)) for b in bw))
        tm = TrafficMatrix(m)
        ref = build_schedule(tm, cl)
        o = build_schedule_oracle(tm.entries, bw)
        assert o["phases"] == [(p.transfers, p.duration) for p in ref.phases]
        assert o["makespan"] == ref.makespan
        if ref.phases:
            raw = decompose(augment(time_normalize(tm, cl)))
            assert o["raw"] == [(tuple(p), d) for p, d in raw]


def test_router_oracle_semantics():
    rng = np.random.default_rng(3)
    T, H, E, k = 37, 512, 8, 2
    import torch
    x = torch.randn(T, H).to(torch.bfloat16)
    w = (torch.randn(E, H) / H ** 0.5).to(torch.bfloat16)
    bias = rng.standard_normal(E).astype(np.float32)
    from oracle.oracle import bf16_bits
    logits, idx, wts = router_oracle(bf16_bits(x), bf16_bits(w), bias, k)
    ref = x.double() @ w.double().T + torch.from_numpy(bias).double()
    assert np.allclose(logits, ref.numpy(), atol=1e-4)
    for t in range(T):
        order = sorted(range(E), key=lambda e: (-logits[t, e], e))
        assert list(idx[t]) == order[:k]
    assert np.allclose(wts.sum(1), 1.0, atol=1e-6)
    # exact ties -> lowest index
    lt = np.zeros((1, E), dtype=np.float32)
    from oracle.oracle import lib
    out_i = np.zeros((1, 3), dtype=np.int32)
    out_w = np.zeros((1, 3), dtype=np.float32)
    lib().oracle_router_topk(lt.ctypes.data, 1, E, 3, out_i.ctypes.data, out_w.ctypes.data)
    assert out_i.tolist() == [[0, 1, 2]]


def test_pack_oracle_small():
    topk = np.array([[0, 1], [1, 0], [2, 3], [3, 3 - 1], [0, 2], [1, 1 + 2]], dtype=np.int32)
    counts, lists, pos = pack_oracle(topk, [0, 0, 1, 1], 2)  # 4 experts on 2 GPUs, 3 tokens per rank
    # rank 0 has tokens 0,1,2; token 0 -> experts 0,1 both on GPU 0 (dedupe)
    assert counts.tolist() == [[2, 1], [2, 3]]
    assert lists[0][0] == [0, 1] and lists[0][1] == [2]
    assert lists[1][0] == [4, 5] and lists[1][1] == [3, 4, 5]
    assert pos[0].tolist() == [0, 0] and pos[4].tolist() == [0, 1] and pos[5].tolist() == [1, 2]


def test_bf16_emulation_helpers():
    """bf16_round is torch's round-to-nearest-even; aggregate_oracle follows
    the device order (one expert per rank: fp32 slot sum; several: per-rank
    bf16 pre-reduction first)."""
    import torch
    from oracle.oracle import aggregate_oracle, bf16_round, row_errors
    rng = np.random.default_rng(0)
    a = (rng.standard_normal(1 << 16) * np.exp(rng.uniform(-20, 20, 1 << 16))).astype(np.float32)
    assert np.array_equal(bf16_round(a), torch.from_numpy(a).bfloat16().float().numpy())
    y = bf16_round(rng.standard_normal((3, 4, 8)).astype(np.float32))
    w = rng.random((3, 4)).astype(np.float32)
    idx = np.array([[0, 1, 2, 3], [3, 2, 1, 0], [0, 2, 4, 6]])
    one = aggregate_oracle(y, idx, w)
    assert np.array_equal(one, bf16_round(sum(w[:, s:s + 1] * y[:, s] for s in range(4))))
    gpu_of = [0, 0, 1, 1, 2, 2, 3, 3]  # two experts per rank
    two = aggregate_oracle(y, idx, w, gpu_of)
    t = 0  # experts 0,1 -> rank 0; 2,3 -> rank 1
    exp0 = bf16_round(bf16_round(w[t, 0] * y[t, 0] + w[t, 1] * y[t, 1]) + bf16_round(w[t, 2] * y[t, 2] + w[t, 3] * y[t, 3]))
    assert np.array_equal(two[0], exp0)
    rel, glob = row_errors(two, two)
    assert rel.max() == 0 and glob == 0
