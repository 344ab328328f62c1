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


def _expected_chunks(phases, counts, n, cd=None, cc=None):
    """Host restatement of the engine tables: one entry per phase and sender
    (receiver, first, count, run code); a run = consecutive phases of one pair,
    coded r (index among the receiver's runs) first, -1-r on continuations."""
    cd = cd or [1] * n
    cc = cc or [1] * n
    P = len(phases)
    ch = [[(-1, 0, 0, 0)] * n for _ in range(P)]
    rch = [[(-1, 0, 0, 0)] * n for _ in range(P)]
    issued = np.zeros((n, n), dtype=np.int64)
    rcnt = [0] * n
    scnt = [0] * n
    prev = [-1] * n
    for k, (transfers, dur) in enumerate(phases):
        tok = int(round(dur))
        cur = [-1] * n
        for i, j in transfers:
            start = int(issued[i, j])
            issued[i, j] += tok
            cont = prev[i] == j
            r = s = -1
            if not cont:
                r, s = rcnt[j], scnt[i]
                rcnt[j] += cd[i]
                scnt[i] += cc[j]
            ch[k][i] = (j, start, tok, r)
            rch[k][j] = (i, start, tok, s)
            cur[i] = j
        prev = cur
    return ch, rch, rcnt, scnt


def test_counts_path_int_domain_and_chunk_tables(A):
    """aurora_schedule_counts (int32 counts, uniform cluster: the int32 fast
    path) vs the oracle, plus its chunk tables vs a host restatement."""
    import torch
    from oracle.oracle import build_schedule_oracle
    from paper_2410_17043_b200 import _lib
    L = _lib.load()
    rng = np.random.default_rng(77)
    for it in range(200):
        n = int(rng.choice([2, 3, 4, 6, 8, 8, 8, 12, 16]))
        c = _fuzz_matrix(rng, n, it % 2).astype(np.int32)
        dev = torch.device("cuda")
        counts = torch.tensor(c, dtype=torch.int32, device=dev)
        P = L.aurora_phase_cap(n)
        i32 = dict(dtype=torch.int32, device=dev)
        pr = torch.empty(P, n, **i32)
        pd = torch.empty(P, dtype=torch.float64, device=dev)
        si = torch.zeros(2, **i32)
        chunks = torch.empty(P, n, 4, **i32)
        rchunks = torch.empty(P, n, 4, **i32)
        n_in = torch.empty(n, **i32)
        n_out = torch.empty(n, **i32)
        prog = torch.zeros(1, **i32)
        # thresholds in runs, or in signals of apportioned copy CTAs (one process driving all ranks,
        # or n_local-rank groups), checked against the host mirror of the apportioning
        from paper_2410_17043_b200.apportion import apportion
        mode = it % 4
        if mode == 0:
            split_args, cd, cc = (0, 0, 0, 0), None, None
        else:
            nl = n if mode != 3 or n % 2 else n // 2
            tot = nl * (3 + it % 5)
            sp = (1, 0, 1)[mode - 1]
            split_args = (nl, tot, tot + nl, sp)
            cd = apportion(c, n, nl, tot, sp, False)
            cc = apportion(c, n, nl, tot + nl, sp, True)
        rc = L.aurora_schedule_counts(counts.data_ptr(), None, n, pr.data_ptr(), pd.data_ptr(), si.data_ptr(),
                                      chunks.data_ptr(), rchunks.data_ptr(), n_in.data_ptr(), n_out.data_ptr(),
                                      si[1:].data_ptr(), prog.data_ptr(), *split_args, _lib.stream_ptr())
        assert rc == 0
        torch.cuda.synchronize()
        nph, status = si.tolist()
        assert status == 0
        d = c.astype(float)
        np.fill_diagonal(d, 0)
        o = build_schedule_oracle(d)
        got = [(tuple((i, int(j)) for i, j in enumerate(row) if j >= 0), float(t))
               for row, t in zip(pr[:nph].tolist(), pd[:nph].tolist())]
        assert got == o["phases"], (n, it)
        ch, rch, rcnt, sseq = _expected_chunks(o["phases"], d, n, cd, cc)
        assert [[tuple(x) for x in row] for row in chunks[:nph].tolist()] == ch
        assert [[tuple(x) for x in row] for row in rchunks[:nph].tolist()] == rch
        assert n_in.tolist() == rcnt and n_out.tolist() == sseq
        assert int(prog.item()) == nph | (1 << 20)


def test_heterogeneous_chunk_rounding_fuzz(A):
    """The fp64 heterogeneous path in the layer (aurora_schedule_counts with
    bandwidths): fractional phase durations become whole-token chunks by
    cumulative rounding; a pair whose rounded total missed its count would need
    a fix-up after the engine may have consumed the entry (AURORA_EINVAL). Over
    1500 MoE-like and adversarial matrices with the paper's bandwidth ratios
     and random ones, the status is always OK, the schedule is
    bit-exact with the oracle, and every pair's chunks sum to its count."""
    import torch
    from oracle.oracle import build_schedule_oracle
    from paper_2410_17043_b200 import _lib
    L = _lib.load()
    rng = np.random.default_rng(2024)
    dev = torch.device("cuda")
    i32 = dict(dtype=torch.int32, device=dev)
    fails = 0
    for it in range(1500):
        n = int(rng.choice([2, 4, 8, 8, 8, 16]))
        if it % 3 == 0:
            bw = np.asarray([(1.0, 0.8, 0.5, 0.4)[q % 4] for q in range(n)])[rng.permutation(n)]
        elif it % 3 == 1:
            bw = rng.choice([100.0, 80.0, 50.0, 40.0], n)
        else:
            bw = rng.uniform(0.05, 3.0, n)
        c = _fuzz_matrix(rng, n, it % 2 if it % 7 else 3).astype(np.int64)
        c = np.minimum(c, (1 << 20)).astype(np.int32)
        counts = torch.tensor(c, device=dev)
        bwt = torch.tensor(bw, dtype=torch.float64, device=dev)
        P = L.aurora_phase_cap(n)
        pr = torch.empty(P, n, **i32)
        pd = torch.empty(P, dtype=torch.float64, device=dev)
        si = torch.zeros(2, **i32)
        chunks = torch.empty(P, n, 4, **i32)
        rchunks = torch.empty(P, n, 4, **i32)
        n_in, n_out, prog = torch.empty(n, **i32), torch.empty(n, **i32), torch.zeros(1, **i32)
        rc = L.aurora_schedule_counts(counts.data_ptr(), bwt.data_ptr(), n, pr.data_ptr(), pd.data_ptr(),
                                      si.data_ptr(), chunks.data_ptr(), rchunks.data_ptr(), n_in.data_ptr(),
                                      n_out.data_ptr(), si[1:].data_ptr(), prog.data_ptr(), 0, 0, 0, 0,
                                      _lib.stream_ptr())
        assert rc == 0
        torch.cuda.synchronize()
        nph, status = si.tolist()
        if status != 0:
            fails += 1
            continue
        d = c.astype(float)
        np.fill_diagonal(d, 0)
        o = build_schedule_oracle(d, bw)
        got = [(tuple((i, int(j)) for i, j in enumerate(row) if j >= 0), float(t))
               for row, t in zip(pr[:nph].tolist(), pd[:nph].tolist())]
        assert got == o["phases"], (n, it)
        tot = np.zeros((n, n))
        for row in chunks[:nph].cpu().numpy():
            for i, (j, first, cnt, _) in enumerate(row):
                if j >= 0:
                    tot[i, j] += cnt
        assert np.array_equal(tot, d), it
    assert fails == 0, f"{fails} of 1500 heterogeneous schedules needed a chunk fix-up (EINVAL)"


def test_int8_decomposition_variants_vs_oracle(A):
    """Every K2 variant of the in-layer n <= 8 integer path gives the oracle's
    schedule, and all give the same engine chunk tables, on 600 MoE-like /
    sparse-with-ties / wide-range count matrices (aurora_debug_set_schedule_variant:
    0 = cell-lane decomposition + cell-lane strip (default), 1 = per-step masks
    with FastMatch8b, 2 = cell-lane decomposition + row-lane strip, 3 = row-lane
    incremental decomposition + row-lane strip)."""
    import torch
    from oracle.oracle import build_schedule_oracle
    from paper_2410_17043_b200 import _lib
    L = _lib.load()
    rng = np.random.default_rng(4242)
    dev = torch.device("cuda")
    i32 = dict(dtype=torch.int32, device=dev)
    try:
        for it in range(600):
            n = int(rng.integers(1, 9))
            kind = it % 3
            if kind == 2:
                c = rng.integers(0, 1 << 24, (n, n)) * (rng.random((n, n)) < 0.7)
            else:
                c = _fuzz_matrix(rng, n, kind)
            c = c.astype(np.int32)
            d = c.astype(float)
            np.fill_diagonal(d, 0)
            o = build_schedule_oracle(d)["phases"]
            counts = torch.tensor(c, **i32)
            P = L.aurora_phase_cap(n)
            tables = None
            for variant in (0, 1, 2, 3):
                assert L.aurora_debug_set_schedule_variant(variant) == 0
                pr = torch.empty(P, n, **i32)
                pd = torch.empty(P, dtype=torch.float64, device=dev)
                si = torch.zeros(2, **i32)
                ch = torch.empty(P, n, 4, **i32)
                rch = torch.empty(P, n, 4, **i32)
                nin = torch.empty(n, **i32)
                nout = torch.empty(n, **i32)
                assert L.aurora_schedule_counts(counts.data_ptr(), None, n, pr.data_ptr(), pd.data_ptr(),
                                                si.data_ptr(), ch.data_ptr(), rch.data_ptr(), nin.data_ptr(),
                                                nout.data_ptr(), si[1:].data_ptr(), None, 0, 0, 0, 0,
                                                _lib.stream_ptr()) == 0
                torch.cuda.synchronize()
                nph, status = si.tolist()
                assert status == 0
                got = [(tuple((i, int(j)) for i, j in enumerate(row) if j >= 0), float(t))
                       for row, t in zip(pr[:nph].tolist(), pd[:nph].tolist())]
                assert got == o, (it, n, variant)
                t = [v[:nph].cpu() if v.dim() > 1 else v.cpu() for v in (ch, rch, nin, nout)]
                if tables is None:
                    tables = t
                assert all(torch.equal(a, b) for a, b in zip(t, tables)), (it, n, variant)
    finally:
        L.aurora_debug_set_schedule_variant(0)
