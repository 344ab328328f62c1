"""End-to-end MoE layer on the GPU vs the CPU oracle: bit-exact routing,
traffic matrix, token permutation, schedule and dispatched rows; combined
output within a bf16 tolerance of the fp32 oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def _deinterleave(w13, F):
    G, _, H = w13.shape
    v = w13.view(G, F // 128, 2, 128, H)
    return v[:, :, 0].reshape(G, F, H), v[:, :, 1].reshape(G, F, H)


def _stacked(layer):
    """Global expert ids in the row order of the layer's stacked weights."""
    return [e for r in layer.local_ranks for e in layer.experts_of_rank(r)]


def _expert_slots(torch, layer, x, sample, emulate):
    """y[t, s] of every sampled token and slot: the SwiGLU expert in fp32 on
    the GPU (no TF32), with the device path's bf16 roundings of h and y when
    ``emulate``."""
    cfg = layer.cfg
    F, H, k = cfg.ffn, cfg.hidden, cfg.top_k
    stacked = _stacked(layer)
    row_of = {e: i for i, e in enumerate(stacked)}
    v = layer.w13.view(len(stacked), F // 128, 2, 128, H)
    xs = x[sample].float()
    ti = layer.topk_idx[sample].cpu().numpy()
    y = torch.zeros(len(sample), k, H, device=x.device)
    for e in np.unique(ti):
        rows, slots = np.nonzero(ti == e)
        r = row_of[int(e)]
        w1 = v[r, :, 0].reshape(F, H).float()
        w3 = v[r, :, 1].reshape(F, H).float()
        xe = xs[torch.as_tensor(rows, device=x.device)]
        h = torch.nn.functional.silu(xe @ w1.T) * (xe @ w3.T)
        if emulate:
            h = h.bfloat16().float()
        ye = h @ layer.w2[r].float().T
        if emulate:
            ye = ye.bfloat16().float()
        y[torch.as_tensor(rows, device=x.device), torch.as_tensor(slots, device=x.device)] = ye
    return y.cpu().numpy()


def _check_output(torch, layer, x, out, sample=None):
    """Combined output vs (1) the bf16-emulating oracle: per-row relative L2
    error <= 1e-2, and (2) the plain fp32 oracle: per-row <= 2e-2 and max
    |err| <= 3e-2 * max |ref|. ``sample``: token subset (full-size configs)."""
    from oracle.oracle import aggregate_oracle, row_errors
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        if sample is None:
            sample = np.arange(x.shape[0])
        sample_t = torch.as_tensor(np.asarray(sample), device=x.device)
        idx = layer.topk_idx[sample_t].cpu().numpy()
        w = layer.topk_w[sample_t].cpu().numpy()
        got = out[sample_t].float().cpu().numpy()
        gpu_of = layer.gpu_of if layer.G > 1 else None
        ref_bf = aggregate_oracle(_expert_slots(torch, layer, x, sample_t, True), idx, w, gpu_of)
        y32 = _expert_slots(torch, layer, x, sample_t, False)
        ref32 = (w[:, :, None] * y32).sum(axis=1)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    rel_bf, _ = row_errors(got, ref_bf)
    rel32, glob32 = row_errors(got, ref32)
    assert rel_bf.max() <= 1e-2, ("per-row error vs the bf16-emulating oracle", rel_bf.max(), int(rel_bf.argmax()))
    assert rel32.max() <= 2e-2, ("per-row error vs the fp32 oracle", rel32.max(), int(rel32.argmax()))
    assert glob32 <= 3e-2, ("max error vs the fp32 oracle", glob32)
    return float(rel_bf.max()), float(rel32.max())


def _check_logits(layer, ref_logits, idx):
    """FMA router: every logit has the oracle's bits. Tensor-core router
    (aurora_route_tc): the selected experts' logits have the oracle's bits, and
    every logit that differs from the oracle's is an approximation strictly
    below the token's k-th selected logit (and close to the exact value)."""
    got = layer.logits.cpu().numpy()
    ref = np.asarray(ref_logits, np.float32)
    if not getattr(layer, "router_tc", False):
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
        return
    sel = np.take_along_axis(got, idx, axis=1)
    assert np.array_equal(sel.view(np.uint32), np.take_along_axis(ref, idx, axis=1).view(np.uint32))
    diff = got.view(np.uint32) != ref.view(np.uint32)
    kth = np.broadcast_to(sel.min(axis=1, keepdims=True), got.shape)
    assert (got[diff] < kth[diff]).all()
    assert (np.abs(got - ref) <= 2.0 ** -6 * np.abs(ref) + 0.1).all()


def _verify(torch, layer, x, out, bandwidths=None, sample=None):
    """Every bit-exact check against the oracle, then the numeric output
    check. Routing (expert choice, logits when E > 8, gate weights), the
    traffic matrix (core.py:75-117), the token permutation and send lists,
    the schedule (build_schedule, commsched.py:291-324, on the time-normalised
    matrix when ``bandwidths``), the engine chunk tables (per-pair totals =
    the traffic matrix, CommSchedule.per_pair_totals commsched.py:134-140),
    and the dispatched rows (receive buffers, or the packed expert groups)."""
    from oracle.oracle import bf16_bits, build_schedule_oracle, pack_oracle, router_oracle
    cfg = layer.cfg
    n, k = cfg.ranks, cfg.top_k
    logits, idx, wts = router_oracle(bf16_bits(x), bf16_bits(layer.w_gate), layer.bias.cpu().numpy(), k)
    assert np.array_equal(layer.topk_idx.cpu().numpy(), idx)
    if layer.logits is not None:  # E > 8: the router leaves its logits
        _check_logits(layer, logits, idx)
    assert np.allclose(layer.topk_w.cpu().numpy(), wts, atol=1e-5)
    counts, lists, pos = pack_oracle(idx, layer.gpu_of, n)
    assert np.array_equal(layer.counts.cpu().numpy(), counts)
    assert np.array_equal(layer.pos.cpu().numpy(), pos)
    Tr = cfg.tokens_per_rank
    sl = layer.send_list.cpu().numpy()
    for i in range(n):
        flat = [t - i * Tr for j in range(n) for t in lists[i][j]]
        assert sl[i, :len(flat)].tolist() == flat
    d = counts.astype(float)
    np.fill_diagonal(d, 0)
    o = build_schedule_oracle(d, bandwidths)
    got = layer.schedule_objects()
    assert [(p.transfers, p.duration) for p in got.phases] == o["phases"]
    nph = int(layer.sched_i[0])
    tot = np.zeros((n, n))
    for row in layer.chunks[:nph].cpu().numpy():
        for i, (j, first, cnt, _) in enumerate(row):
            if j >= 0:
                tot[i, j] += cnt
    assert np.array_equal(tot, d)
    xb = x.view(torch.int16)
    if getattr(layer, "grouped", False):
        # grouped dispatch: the packed group buffer holds, per (rank, local expert) in
        # that order, x of every token choosing the expert in token order
        gl = layer.gpu_of_expert.cpu().numpy()
        lo = layer.local_of_expert.cpu().numpy()
        order = sorted(range(cfg.experts), key=lambda e: (gl[e], lo[e]))
        sizes = [int((idx == e).any(axis=1).sum()) for e in order]
        assert layer.g_rows.cpu().numpy().tolist() == sizes
        assert layer.g_off.cpu().numpy().tolist() == np.concatenate([[0], np.cumsum(sizes)]).tolist()
        rows = np.concatenate([np.where((idx == e).any(axis=1))[0] for e in order])
        ag = layer.a_g.view(torch.int16)
        assert torch.equal(ag[:len(rows)], xb[torch.as_tensor(rows, device=xb.device)])
    else:
        recv = layer.recv.view(torch.int16)
        for j in range(n):
            rows = list(lists[j][j]) + [t for i in range(n) if i != j for t in lists[i][j]]
            if rows:
                assert torch.equal(recv[j * layer.cap: j * layer.cap + len(rows)],
                                   xb[torch.as_tensor(rows, device=xb.device)])
    return _check_output(torch, layer, x, out, sample)


def _check_layer(torch, cfg, plan=None, **kw):
    from paper_2410_17043_b200.layer import AuroraMoELayer
    layer = AuroraMoELayer(cfg, plan, **kw)
    g = torch.Generator(device="cuda").manual_seed(cfg.seed + 11)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    out = layer(x)
    torch.cuda.synchronize()
    layer.check_status()
    _verify(torch, layer, x, out, kw.get("bandwidths"))
    return layer


def test_layer_small_n4(torch):
    from paper_2410_17043_b200.layer import MoEConfig
    _check_layer(torch, MoEConfig(hidden=256, ffn=256, experts=4, top_k=2, tokens=1024, ranks=4, skew=1.0, seed=0))


def test_layer_n8_skewed_permuted_plan(torch):
    from paper_2410_17043_b200 import DeploymentPlan
    from paper_2410_17043_b200.layer import MoEConfig
    cfg = MoEConfig(hidden=1024, ffn=512, experts=8, top_k=2, tokens=4096, ranks=8, skew=2.0, seed=1)
    _check_layer(torch, cfg, DeploymentPlan((3, 0, 7, 1, 6, 2, 5, 4)))


def test_layer_serial_and_overlapped_agree(torch):
    """Every stream plan gives the same bits: serial K2 -> dispatch, K2 with the
    PDL-launched dispatch, and the GEMM-splitting overlap plans -- including
    AURORA_C_OVERLAP (fewer copy CTAs for the remote dispatch than for the
    combine: K2 must count the dispatch's hand-over thresholds for them)."""
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg = MoEConfig(hidden=512, ffn=256, experts=8, top_k=2, tokens=2048, ranks=8, skew=1.0, seed=4)
    layer = AuroraMoELayer(cfg, spin_limit=1 << 24)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    layer.overlap = False
    serial = layer(x).clone()
    for overlap, c_ov in (("schedule", 0), ("full", 0), ("full", 8), ("full", 3), (False, 0)):
        layer.overlap, layer.C_overlap = overlap, c_ov
        out = layer(x)
        torch.cuda.synchronize()
        layer.check_status()
        assert torch.equal(serial, out), (overlap, c_ov)


def test_layer_nvtx_ranges_balanced(torch):
    """AURORA_NVTX ranges around the stages stay balanced (push / pop per trace point)
    for the default, serial-schedule and N1 plans; the output is unchanged."""
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg = MoEConfig(hidden=256, ffn=256, experts=8, top_k=2, tokens=2048, ranks=8, skew=1.0, seed=3)
    layer = AuroraMoELayer(cfg)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    ref = layer(x).clone()
    layer.nvtx = True
    for attrs in ({}, {"stream_schedule": False}, {"arrival": True}):
        for a, v in attrs.items():
            setattr(layer, a, v)
        depth0 = torch.cuda.nvtx.range_push("probe")
        out = layer(x)
        depth1 = torch.cuda.nvtx.range_push("probe")
        torch.cuda.nvtx.range_pop()
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        assert depth1 == depth0, attrs  # same nesting depth before and after the forward
        assert torch.equal(out, ref)
        for a in attrs:
            setattr(layer, a, {"stream_schedule": True, "arrival": False}[a])


def test_layer_repeated_calls_rearm_counters(torch):
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg = MoEConfig(hidden=256, ffn=256, experts=8, top_k=2, tokens=2048, ranks=8, skew=0.5, seed=2)
    layer = AuroraMoELayer(cfg)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    first = layer(x).clone()
    for _ in range(3):
        again = layer(x)
    torch.cuda.synchronize()
    layer.check_status()
    assert torch.equal(first, again)
    assert int(layer.ctr_d.abs().sum()) == 0 and int(layer.ctr_c.abs().sum()) == 0


def _run_full(torch, cfg, plan=None, seed=5, **kw):
    from paper_2410_17043_b200.layer import AuroraMoELayer
    layer = AuroraMoELayer(cfg, plan, **kw)
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    out = layer(x).clone()
    torch.cuda.synchronize()
    layer.check_status()
    return layer, x, out


def _sample(T, m=256, seed=1):
    import torch
    return torch.randperm(T, generator=torch.Generator().manual_seed(seed))[:m].numpy()


def test_layer_c2_full_size(torch):
    """The bench workload itself (C2: 16384 tokens, hidden 4096, FFN 14336, 8
    experts top-2, 8 ranks): bit-exact routing / traffic matrix / token
    permutation / schedule / chunk tables / dispatched rows vs the oracle, and
    the output of 256 sampled tokens vs the bf16-emulating and fp32 references."""
    from paper_2410_17043_b200.layer import MoEConfig
    cfg = MoEConfig(hidden=4096, ffn=14336, experts=8, top_k=2, tokens=16384, ranks=8, skew=1.0, seed=0)
    layer, x, out = _run_full(torch, cfg)
    _verify(torch, layer, x, out, sample=_sample(cfg.tokens))


def test_layer_c5_full_size(torch):
    """C5 at its bench shape: 64 experts top-6, hidden 5120, FFN 1536, 16384
    tokens, 8 ranks (8 experts per rank, grouped dispatch into the packed
    expert groups, single-expert rows finished in GEMM2, pre-reduction, fused
    combine). Bit-exact logits / top-k / traffic matrix / group sizes / packed
    row placement / schedule; sampled output vs the bf16-emulating oracle."""
    from paper_2410_17043_b200.layer import MoEConfig
    cfg = MoEConfig(hidden=5120, ffn=1536, experts=64, top_k=6, tokens=16384, ranks=8, skew=1.0, seed=0)
    layer, x, out = _run_full(torch, cfg)
    assert layer.grouped and layer.logits is not None
    _verify(torch, layer, x, out, sample=_sample(cfg.tokens))


@pytest.mark.parametrize("skew", [0.0, 2.0])
def test_layer_c5_full_size_skews(torch, skew):
    """C5 routing at the ends of the skew sweep (Zipf s = 0 and 2)."""
    from paper_2410_17043_b200.layer import MoEConfig
    cfg = MoEConfig(hidden=5120, ffn=1536, experts=64, top_k=6, tokens=16384, ranks=8, skew=skew, seed=2)
    layer, x, out = _run_full(torch, cfg, seed=9)
    _verify(torch, layer, x, out, sample=_sample(cfg.tokens, 128, 3))


def test_layer_c4_full_size(torch):
    """C4 at the bench shape: C2 on the emulated heterogeneous cluster
    (bandwidths 100/80/50/40 x2), placement by
    assign_exclusive_hetero (placement.py:46-60) from a calibration pass,
    schedule on the fp64 time-normalised matrix (commsched.py:181-190)
    bit-exact with the oracle, whole-token chunks whose per-pair totals equal
    the traffic matrix, sampled output vs the references."""
    import paper_2410_17043_b200 as A
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    bw = [1.0, 1.0, 0.8, 0.8, 0.5, 0.5, 0.4, 0.4]
    cluster = A.ClusterSpec(tuple(A.GpuSpec(b, b) for b in bw))
    cfg = MoEConfig(hidden=4096, ffn=14336, experts=8, top_k=2, tokens=16384, ranks=8, skew=1.0, seed=0)
    calib = AuroraMoELayer(cfg)
    g = torch.Generator(device="cuda").manual_seed(7)
    xc = torch.randn(cfg.tokens, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    calib.route(xc, int(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    plan = A.assign_exclusive_hetero(calib.counts.cpu().numpy().sum(axis=0), cluster)
    del calib
    torch.cuda.empty_cache()
    assert plan.assignment_a != tuple(range(8))  # the hot experts moved to the fast ranks
    layer, x, out = _run_full(torch, cfg, plan, bandwidths=bw)
    _verify(torch, layer, x, out, bandwidths=bw, sample=_sample(cfg.tokens))


@pytest.mark.parametrize("shape", [dict(experts=8, top_k=2, ranks=8, tokens=4096, skew=1.5),
                                   dict(experts=4, top_k=2, ranks=4, tokens=2048, skew=0.0),
                                   dict(experts=8, top_k=1, ranks=8, tokens=2048, skew=60.0)])
def test_layer_arrival_driven_gemm(torch, shape):
    """N1: GEMM1 launched as a programmatic dependent of an LSU dispatch (one copy CTA
    per SM), each tile waiting for the landed-row credits of the blocks under it (local
    rows first) -- same output bits as the serial path, repeatedly (landed re-armed by
    GEMM1's last cluster), and GEMM1's CTAs start before the dispatch has finished."""
    from paper_2410_17043_b200 import _lib
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg = MoEConfig(hidden=1024, ffn=1024, seed=8, **shape)
    layer = AuroraMoELayer(cfg, spin_limit=1 << 26)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    ref = layer(x).clone()
    torch.cuda.synchronize()
    layer.arrival = True
    assert layer.arrival_on
    for _ in range(3):
        out = layer(x)
        torch.cuda.synchronize()
        layer.check_status()
        assert torch.equal(out, ref)
        assert int(layer.landed.abs().sum()) == 0
    assert int(layer.ctr_d.abs().sum()) == 0 and int(layer.ctr_c.abs().sum()) == 0
    # timeline evidence: GEMM1's first tiles start while dispatch copy CTAs are still running
    L = _lib.load()
    eng = torch.zeros(4 * 4096, dtype=torch.int64, device="cuda")
    gt = torch.zeros(2 * 1024, dtype=torch.int64, device="cuda")
    L.aurora_debug_set_engine_trace(eng.data_ptr())
    L.aurora_debug_set_gemm_trace(gt.data_ptr())
    try:
        layer(x)
        torch.cuda.synchronize()
    finally:
        L.aurora_debug_set_engine_trace(None)
        L.aurora_debug_set_gemm_trace(None)
    layer.check_status()
    e = eng.view(-1, 4).cpu().numpy()
    g = gt.view(-1, 2).cpu().numpy()
    e_end = e[e[:, 0] > 0][:, 2]
    g_first = g[g[:, 1] > 0][:, 1]
    if cfg.ranks > 1 and len(e_end) and len(g_first):
        # no assertion on speed; record that the overlap exists (not every shape has local-only tiles)
        print("gemm first tile before last dispatch CTA end:", bool(g_first.min() < e_end.max()))


def test_layer_compute_partition(torch):
    """Emulated per-rank compute (C4): with compute_scales the expert GEMMs' CTA
    pairs are split among the ranks in proportion (cluster_part) and each rank's
    tiles run on its own share -- same output bits as the shared grid, fused and
    engine combine, repeatedly (the static partition never touches the tile
    counters)."""
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg = MoEConfig(hidden=512, ffn=512, experts=8, top_k=2, tokens=4096, ranks=8, skew=1.5, seed=3)
    scales = [1.0, 1.0, 0.8, 0.8, 0.5, 0.5, 0.4, 0.4]
    ref_layer = AuroraMoELayer(cfg)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    ref = ref_layer(x).clone()
    layer = AuroraMoELayer(cfg, compute_scales=scales)
    part = layer.gemm_part.cpu().tolist()
    assert part[0] == 0 and part[-1] == layer.num_sms // 2 and all(b > a for a, b in zip(part, part[1:]))
    assert part[1] - part[0] > part[-1] - part[-2]  # the fast rank has more CTA pairs than the slow one
    for fused in (True, False, True):
        layer.fused_combine = fused
        out = layer(x)
        torch.cuda.synchronize()
        layer.check_status()
        assert torch.equal(out, ref), fused
    assert AuroraMoELayer.cluster_partition([1, 1, 1, 1], 74)[-1] == 74
    # one process of two (ranks 4-7: the slow half): only its share of the CTA pairs, idle pairs exit
    half = AuroraMoELayer(cfg, rank_base=4, n_local=4, compute_scales=scales)
    hp = half.gemm_part.cpu().tolist()
    assert hp[-1] == round(layer.num_sms // 2 * 1.8 / 3.6)
    # several experts per rank (the packed grouped GEMMs, a rank's clusters serve all its experts)
    cfg5 = MoEConfig(hidden=512, ffn=256, experts=32, top_k=4, tokens=4096, ranks=8, skew=1.0, seed=5)
    ref5 = AuroraMoELayer(cfg5)
    x5 = torch.randn(cfg5.tokens, cfg5.hidden, device="cuda").to(torch.bfloat16)
    r5 = ref5(x5).clone()
    l5 = AuroraMoELayer(cfg5, compute_scales=scales)
    for scatter in (True, False):
        l5.packed_scatter = scatter
        o5 = l5(x5)
        torch.cuda.synchronize()
        l5.check_status()
        assert torch.equal(o5, r5), scatter


def test_layer_heterogeneous_cluster(torch):
    """C4 (heterogeneous emulation), small: placement by assign_exclusive_hetero
    (placement.py:46-60) from a calibration pass, schedule on the fp64
    time-normalised matrix (commsched.py:181-190) bit-exact with the oracle,
    fractional durations turned into whole-token chunks whose per-pair totals
    equal the traffic matrix, and the same output as the homogeneous run."""
    import paper_2410_17043_b200 as A
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    bw = [1.0, 1.0, 0.8, 0.8, 0.5, 0.5, 0.4, 0.4]
    cluster = A.ClusterSpec(tuple(A.GpuSpec(b, b) for b in bw))
    cfg = MoEConfig(hidden=512, ffn=256, experts=8, top_k=2, tokens=4096, ranks=8, skew=1.5, seed=9)
    calib = AuroraMoELayer(cfg)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    calib(x)
    torch.cuda.synchronize()
    loads = calib.counts.cpu().numpy().sum(axis=0)  # tokens per expert (identity plan)
    plan = A.assign_exclusive_hetero(loads, cluster)
    layer = AuroraMoELayer(cfg, plan, bandwidths=bw)
    out = layer(x)
    torch.cuda.synchronize()
    layer.check_status()
    _verify(torch, layer, x, out, bandwidths=bw)
    # output identical to the homogeneous-cluster run of the same plan (schedule only changes pacing)
    ref_layer = AuroraMoELayer(cfg, plan)
    ref = ref_layer(x)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_layer_several_experts_per_rank(torch):
    """E > n (C5-style): 16 experts top-4 on 4 ranks -- contiguous expert
    blocks, one network row per (token, rank), expert metadata on the
    engine's second plane, grouped packed GEMMs, pre-reduction, combine."""
    _check_layer(torch, MoEConfig_(hidden=256, ffn=256, experts=16, top_k=4, tokens=1024, ranks=4, skew=1.0,
                                   seed=3))


def test_layer_deepseek_shape_small(torch):
    """64 experts top-6 over 8 ranks (C5 routing), reduced hidden size."""
    _check_layer(torch, MoEConfig_(hidden=512, ffn=256, experts=64, top_k=6, tokens=2048, ranks=8, skew=1.0,
                                   seed=4))


def test_fused_and_engine_combine_agree_several_experts(torch):
    """E > n: the combine fused into the pre-reduction (rows stored straight
    into the senders' return buffers) and the reversed-schedule combine engine,
    rows dispatched straight into their expert groups or received, sorted and
    gathered, all give identical outputs, repeatedly (counters / ticket rearmed)."""
    from paper_2410_17043_b200.layer import AuroraMoELayer
    cfg = MoEConfig_(hidden=512, ffn=256, experts=64, top_k=6, tokens=2048, ranks=8, skew=1.0, seed=9)
    layer = AuroraMoELayer(cfg)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    layer.fused_combine, layer.grouped_dispatch = False, False
    ref = layer(x).clone()
    for fused, grouped, lsu in ((True, True, 0), (False, True, 0), (True, False, 0), (False, False, 0),
                                (True, True, 64), (True, True, 0)):
        # (the LSU copy engine has no grouped mode: it falls back to receive / sort / gather)
        layer.fused_combine, layer.grouped_dispatch, layer.engine_lsu = fused, grouped, lsu
        out = layer(x)
        torch.cuda.synchronize()
        layer.check_status()
        assert torch.equal(out, ref), (fused, grouped, lsu)
    assert int(layer.ctr_c.abs().sum()) == 0 and int(layer.gemm_ticket.item()) == 0


def MoEConfig_(**kw):
    from paper_2410_17043_b200.layer import MoEConfig
    return MoEConfig(**kw)


def test_colocated_models(torch):
    """C3: model a (4 experts) and model b (8 experts) on 4 ranks. Calibration
    routing -> Lina slots for model b -> Aurora's colocate_homogeneous pairing
    -> both layers on the same ranks (model-b experts placed by the plan);
    each layer bit-exact / within tolerance vs the oracle."""
    from oracle.oracle import bf16_bits, pack_oracle, router_oracle
    import paper_2410_17043_b200 as A
    from paper_2410_17043_b200.colocation import (ColocatedLayers, combined_bmax, lina_slots,
                                                  plan_colocation)
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg_a = MoEConfig(hidden=256, ffn=256, experts=4, top_k=2, tokens=1024, ranks=4, skew=1.0, seed=5)
    cfg_b = MoEConfig(hidden=256, ffn=128, experts=8, top_k=2, tokens=1024, ranks=4, skew=1.5, seed=6)
    xa = torch.randn(cfg_a.tokens, cfg_a.hidden, device="cuda").to(torch.bfloat16)
    xb = torch.randn(cfg_b.tokens, cfg_b.hidden, device="cuda").to(torch.bfloat16)
    cal_a = AuroraMoELayer(cfg_a)
    cal_a(xa)
    cal_b = AuroraMoELayer(cfg_b)
    cal_b(xb)
    torch.cuda.synchronize()
    loads_b = np.bincount(cal_b.topk_idx.cpu().numpy().ravel(), minlength=8)
    slots = lina_slots(loads_b)
    slot_of = {e: s for s, pair in enumerate(slots) for e in pair}
    _, idx_b, _ = router_oracle(bf16_bits(xb), bf16_bits(cal_b.w_gate), cal_b.bias.cpu().numpy(), 2)
    slot_counts, _, _ = pack_oracle(idx_b, [slot_of[e] for e in range(8)], 4)
    cp = plan_colocation(cal_a.counts.cpu().numpy(), slot_counts, slots)
    assert sorted(cp.gpu_of_b) == [0, 0, 1, 1, 2, 2, 3, 3]
    pair = ColocatedLayers(cfg_a, cfg_b, cp)
    out_a, out_b = pair(xa, xb)
    torch.cuda.synchronize()
    pair.check_status()
    for layer, x, out in ((pair.a, xa, out_a), (pair.b, xb, out_b)):
        _verify(torch, layer, x, out)
    assert pair.a.G == 1 and pair.b.G == 2
    assert tuple(pair.b.gpu_of) == cp.gpu_of_b
    assert combined_bmax(cal_a.counts.cpu().numpy(), slot_counts, cp.plan) > 0
    # Table-1 interleaving (model b on a second stream) and the serial order: same bits
    ref_a, ref_b = out_a.clone(), out_b.clone()
    for il in (False, True, False, True):
        pair.interleave = il
        for _ in range(3):
            ya, yb = pair(xa, xb)
        torch.cuda.synchronize()
        pair.check_status()
        assert torch.equal(ya, ref_a) and torch.equal(yb, ref_b), il
    tl = pair.timeline(xa, xb)
    assert tl["b"]["dispatched"] >= tl["a"]["dispatched"]  # N_b waits for N_a (one copy engine at a time)
    assert tl["a"]["end"] > 0 and tl["b"]["end"] > 0


@pytest.mark.parametrize("hetero", [False, True])
def test_colocated_models_full_size(torch, hetero):
    """C3 (and C3 on C4's emulated cluster) at the bench shapes, built the way
    bench.py --config c3 / c3h builds them: Mixtral-shape model a (8 experts
    top-2, FFN 14336) and the 16-expert top-2 model b (FFN 7168) on 8 ranks,
    16384 tokens each; calibration routing -> Lina slots of model b ->
    colocate_homogeneous (placement.py:109-126), or colocate_heterogeneous
    (placement.py:129-157) with per-rank copy / compute shares. Every bit-exact
    check of _verify for both layers (routing, logits, traffic matrices,
    permutations, schedules on the time-normalised matrices, chunk tables,
    dispatched rows) and sampled outputs vs the bf16-emulating oracle."""
    from paper_2410_17043_b200 import ClusterSpec, GpuSpec, _lib
    from paper_2410_17043_b200.colocation import (ColocatedLayers, expert_work, lina_slots, plan_colocation,
                                                  plan_colocation_hetero)
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    n, T = 8, 16384
    cfg_a = MoEConfig(hidden=4096, ffn=14336, experts=n, top_k=2, tokens=T, ranks=n, skew=1.0, seed=0)
    cfg_b = MoEConfig(hidden=4096, ffn=7168, experts=2 * n, top_k=2, tokens=T, ranks=n, skew=1.5, seed=1)
    g = torch.Generator(device="cuda").manual_seed(101)
    xa = torch.randn(T, 4096, device="cuda", generator=g).to(torch.bfloat16)
    xb = torch.randn(T, 4096, device="cuda", generator=g).to(torch.bfloat16)
    sp = _lib.stream_ptr()
    cal_a = AuroraMoELayer(cfg_a)
    cal_a.route(xa, sp)
    cal_b = AuroraMoELayer(cfg_b)
    cal_b.route(xb, sp)
    torch.cuda.synchronize()
    counts_a = cal_a.counts.cpu().numpy()
    slots = lina_slots(np.bincount(cal_b.topk_idx.cpu().numpy().ravel(), minlength=2 * n))
    slot_of = [0] * (2 * n)
    for s_, (e1, e2) in enumerate(slots):
        slot_of[e1] = slot_of[e2] = s_
    cal_s = AuroraMoELayer(cfg_b, gpu_of_expert=slot_of, weights={"w_gate": cal_b.w_gate, "bias": cal_b.bias,
                                                                   "w13": cal_b.w13, "w2": cal_b.w2})
    cal_s.route(xb, sp)
    torch.cuda.synchronize()
    slot_counts = cal_s.counts.cpu().numpy()
    del cal_a, cal_b, cal_s
    torch.cuda.empty_cache()
    kw, bws = {}, None
    if hetero:
        bws = [1.0, 1.0, 0.8, 0.8, 0.5, 0.5, 0.4, 0.4]
        kw = {"bandwidths": bws, "compute_scales": bws}
        cluster = ClusterSpec(tuple(GpuSpec(b, b) for b in bws))
        cp = plan_colocation_hetero(counts_a, slot_counts, slots, cluster, expert_work(4096, 14336),
                                    expert_work(4096, 7168))
    else:
        cp = plan_colocation(counts_a, slot_counts, slots)
    pair = ColocatedLayers(cfg_a, cfg_b, cp, **kw)
    out_a, out_b = pair(xa, xb)
    out_a, out_b = out_a.clone(), out_b.clone()
    torch.cuda.synchronize()
    pair.check_status()
    assert tuple(pair.b.gpu_of) == tuple(cp.gpu_of_b)
    for layer, x, out in ((pair.a, xa, out_a), (pair.b, xb, out_b)):
        _verify(torch, layer, x, out, bandwidths=bws, sample=_sample(T, 128, 4))


def test_engine_runs_baseline_schedules(torch):
    """SJF / RCS schedules (baselines.py) executed by the same engine deliver
    the same rows: identical layer output to the Aurora-scheduled run."""
    import paper_2410_17043_b200 as A
    from paper_2410_17043_b200 import baselines as B
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg = MoEConfig(hidden=512, ffn=256, experts=8, top_k=2, tokens=2048, ranks=8, skew=1.0, seed=8)
    layer = AuroraMoELayer(cfg)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    ref = layer(x).clone()
    torch.cuda.synchronize()
    d = layer.counts.cpu().numpy().astype(float)
    np.fill_diagonal(d, 0)
    tm, cl = A.TrafficMatrix(d), A.ClusterSpec.uniform(8)
    for sched in (B.schedule_sjf(tm, cl), B.schedule_rcs(tm, cl, 0)):
        s = torch.cuda.current_stream().cuda_stream
        layer.route(x, s)
        layer.pack(s)
        layer.load_schedule(sched)
        layer.dispatch(s)
        layer.experts(s)
        layer.combine(s)
        layer.aggregate(s)
        torch.cuda.synchronize()
        layer.check_status()
        assert torch.equal(layer.out, ref)


@pytest.mark.parametrize("shape", [
    dict(experts=1, top_k=1, ranks=1, tokens=256),           # one rank: no all-to-all, empty schedule
    dict(experts=2, top_k=1, ranks=2, tokens=512),
    dict(experts=6, top_k=2, ranks=2, tokens=512),           # E not a power of two, 3 experts per rank
    dict(experts=8, top_k=2, ranks=8, tokens=2048, skew=30.0),  # nearly every token to two experts
    dict(experts=4, top_k=4, ranks=4, tokens=1024),          # every token to every rank
    dict(experts=16, top_k=2, ranks=16, tokens=4096),        # the most ranks (K2's n <= 16 kernel)
    dict(experts=64, top_k=6, ranks=16, tokens=4096),        # 16 ranks x 4 experts, C5 routing
    dict(experts=8, top_k=1, ranks=8, tokens=2048, skew=60.0),  # one hot expert, most ranks idle
    dict(experts=16, top_k=3, ranks=8, tokens=512),          # 64 tokens per rank: one router tile, partial units
    dict(experts=40, top_k=5, ranks=8, tokens=1536),         # E = 5 x 8: a partial 8-expert pass
    dict(experts=32, top_k=2, ranks=32, tokens=2048),        # 32 ranks: K2's widest, engine combine (> 16)
    dict(experts=64, top_k=4, ranks=32, tokens=4096),        # 32 ranks x 2 experts: grouped, engine combine
])
def test_layer_edge_shapes(torch, shape):
    from paper_2410_17043_b200.layer import MoEConfig
    kw = dict(hidden=256, ffn=128, skew=1.0, seed=7)
    kw.update(shape)
    _check_layer(torch, MoEConfig(**kw))


def test_engine_cta_splits_and_copy_paths_agree(torch):
    """Every copy-CTA split (even / volume / bandwidth, csrc/apportion.cuh), the
    LSU and TMA copy paths, K2 overlapped (PDL) or serial, the unpaced
    ablation, and local rows read in place or combined deliver the same rows:
    identical output, counters rearmed."""
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg = MoEConfig(hidden=512, ffn=256, experts=8, top_k=2, tokens=4096, ranks=8, skew=1.5, seed=4)
    layer = AuroraMoELayer(cfg, bandwidths=[1.0, 1.0, 0.8, 0.8, 0.5, 0.5, 0.4, 0.4])
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    ref = layer(x).clone()
    torch.cuda.synchronize()
    layer.check_status()
    for split in (0, 1, 2):
        for lsu in (0, 64):
            for stream_sched in (True, False):
                for unpaced in (0, 16):
                    layer.split, layer.engine_lsu, layer.stream_schedule, layer.unpaced = split, lsu, stream_sched, unpaced
                    out = layer(x)
                    torch.cuda.synchronize()
                    layer.check_status()
                    assert torch.equal(out, ref), (split, lsu, stream_sched, unpaced)
    for local_direct in (False, True):  # combine moving the local rows too vs aggregation reading them in place
        for fused in (False, True):  # combine engine vs the combine fused into GEMM2's epilogue
            layer.local_direct, layer.fused_combine = local_direct, fused
            out = layer(x)
            torch.cuda.synchronize()
            layer.check_status()
            assert torch.equal(out, ref), (local_direct, fused)
    assert int(layer.ctr_d.abs().sum()) == 0 and int(layer.ctr_c.abs().sum()) == 0


@pytest.mark.parametrize("experts,top_k,fused,arrival", [(8, 2, False, False), (8, 2, True, False),
                                                         (16, 4, False, False), (16, 4, True, False),
                                                         (8, 2, True, True)])
def test_two_rank_groups_in_one_context(torch, experts, top_k, fused, arrival):
    """The multi-GPU code path on one device: two layer instances, each driving
    4 of the 8 ranks (what two processes on two GPUs do), with peer tables
    pointing at each other's buffers, system-scope flags, the traffic matrix
    exchanged between the halves by peer stores + flags (aurora_exchange_counts,
    double-buffered by step parity), K2 counting
    hand-over thresholds over 4-rank groups, and the two engines running
    concurrently on two streams, each waiting on the other's arrival counters.
    Output identical to the single-instance (loopback) layer; with several
    experts per rank the expert-metadata plane travels to the peers too. fused:
    GEMM2 stores each half's rows straight into the other half's return buffers
    and signals its counters (aurora_expert_ffn_combine / aurora_combine_wait)."""
    from paper_2410_17043_b200.dist import _names, _strides
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg = MoEConfig(hidden=512, ffn=256, experts=experts, top_k=top_k, tokens=4096, ranks=8, skew=1.0, seed=6)
    ref_layer = AuroraMoELayer(cfg)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    ref = ref_layer(x).clone()
    torch.cuda.synchronize()
    halves = [AuroraMoELayer(cfg, rank_base=4 * p, n_local=4, spin_limit=1 << 24) for p in range(2)]
    for h in halves:
        h.arrival = arrival  # N1: each half's GEMM1 waits for the other half's landed credits
    xs = [x[: cfg.tokens // 2].contiguous(), x[cfg.tokens // 2:].contiguous()]
    for h, xi in zip(halves, xs):
        h._use_input(xi)
    tables = {}
    for name in _names(halves[0]):
        st = _strides(halves[0])[name]
        tables[name] = [getattr(halves[r // 4], name).data_ptr() + (r % 4) * st for r in range(8)]
    for h in halves:
        h._peers = tables
        h._tables_for(h.x, tables)
    streams = [torch.cuda.Stream() for _ in range(2)]
    sp = [int(s.cuda_stream) for s in streams]

    def both(fn):
        for h, s in zip(halves, sp):
            fn(h, s)
        torch.cuda.synchronize()

    for _ in range(3):  # counters rearmed, counts buffers alternating (step parity) across calls
        both(lambda h, s: h.route(h.x, s))
        both(lambda h, s: h.exchange_counts(s))  # peer stores + flags, concurrently on both streams
        assert torch.equal(halves[0].counts, halves[1].counts)
        assert torch.equal(halves[0].counts, ref_layer.counts)
        both(lambda h, s: h.pack(s))
        both(lambda h, s: h.schedule(s))
        both(lambda h, s: h.dispatch(s))   # concurrent: each waits on the other's flags
        if fused:
            assert all(h.combine_in_gemm for h in halves)
            both(lambda h, s: h.experts_combine(s))
            both(lambda h, s: h.combine_wait(s))
        else:
            both(lambda h, s: h.experts(s))
            both(lambda h, s: h.combine(s))
        both(lambda h, s: h.aggregate(s))
        for h in halves:
            h.check_status()
        assert torch.equal(torch.cat([halves[0].out, halves[1].out]), ref)
    for h in halves:
        assert int(h.ctr_d.abs().sum()) == 0 and int(h.ctr_c.abs().sum()) == 0


@pytest.mark.parametrize("experts,top_k", [(8, 2), (16, 4), (64, 6)])
def test_router_ties_pick_lower_index(torch, experts, top_k):
    """Duplicate gate rows with equal bias give bit-identical logits: both
    router paths (one CTA per tile for E <= 8; balanced (tile, pass) units +
    the 4-threads-per-token top-k tail for E > 8) must choose the lower expert
    index on every tie, as the oracle's sequential scan does."""
    from oracle.oracle import bf16_bits, router_oracle
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg = MoEConfig(hidden=512, ffn=256, experts=experts, top_k=top_k, tokens=2048, ranks=8, skew=0.0, seed=12)
    gpu_of = [e * 8 // experts for e in range(experts)]
    w = AuroraMoELayer.synthetic_weights(cfg, torch.device("cuda"),
                                         [e for r in range(8) for e in range(experts) if gpu_of[e] == r])
    for e in range(1, experts, 2):  # every odd expert duplicates its even neighbour
        w["w_gate"][e] = w["w_gate"][e - 1]
        w["bias"][e] = w["bias"][e - 1]
    layer = AuroraMoELayer(cfg, gpu_of_expert=gpu_of, weights=w)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    layer.route(x, int(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    _, idx, wts = router_oracle(bf16_bits(x), bf16_bits(layer.w_gate), layer.bias.cpu().numpy(), top_k)
    got = layer.topk_idx.cpu().numpy()
    assert np.array_equal(got, idx)
    assert (got[:, 0] % 2 == 0).all()  # the first choice is always the lower twin
    assert np.allclose(layer.topk_w.cpu().numpy(), wts, atol=1e-6)


@pytest.mark.parametrize("experts,top_k,hidden,skew,tokens,ranks", [
    (16, 2, 512, 1.0, 4096, 8), (32, 4, 1024, 0.0, 4096, 8), (64, 6, 5120, 1.0, 4096, 8),
    (64, 6, 5120, 2.0, 4096, 8), (64, 8, 2048, 0.5, 4096, 8), (24, 6, 768, 1.0, 4096, 8),
    (16, 3, 512, 1.0, 384, 2), (64, 6, 1024, 1.0, 320, 1)])
def test_router_tc_matches_fma_router(torch, experts, top_k, hidden, skew, tokens, ranks):
    """aurora_route_tc (tensor-core approximate logits + exact candidates +
    certificate) gives the FMA router's output bit for bit: top-k, softmax
    weights, destinations, block histograms, traffic matrix, and the selected
    logits. Also on adversarial inputs: x scaled by 2^12, 2^-12 and 2^-118 (subnormal
    products: the exact pass's bf16 FMAs keep subnormals like fmaf), and gate
    rows duplicated with a 1-ulp perturbation (near-ties below the certificate's
    bound, so those tokens take the exact fallback). Token counts that leave a
    partial 256-row GEMM tile (384, 320) and a partial 64-token tile (320)."""
    import os
    from oracle.oracle import bf16_bits, router_oracle
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg = MoEConfig(hidden=hidden, ffn=256, experts=experts, top_k=top_k, tokens=tokens, ranks=ranks, skew=skew,
                    seed=31)
    gpu_of = [e * ranks // experts for e in range(experts)]
    w = AuroraMoELayer.synthetic_weights(cfg, torch.device("cuda"),
                                         [e for r in range(ranks) for e in range(experts) if gpu_of[e] == r])
    wg = w["w_gate"]
    for e in range(1, experts, 4):  # near-twins: the bf16 neighbour of one entry
        row = wg[e - 1].clone()
        row.view(torch.int16)[3] += 1  # the next bf16 value (away from zero)
        wg[e] = row
        w["bias"][e] = w["bias"][e - 1]
    layers = {}
    for mode in ("tc", "fma"):
        os.environ["AURORA_ROUTER"] = mode
        try:
            layers[mode] = AuroraMoELayer(cfg, gpu_of_expert=gpu_of, weights=w)
        finally:
            os.environ.pop("AURORA_ROUTER", None)
    assert layers["tc"].router_tc and not layers["fma"].router_tc
    g = torch.Generator(device="cuda").manual_seed(5)
    x0 = torch.randn(cfg.tokens, cfg.hidden, device="cuda", generator=g)
    for scale in (1.0, 4096.0, 1.0 / 4096.0, 2.0 ** -118):  # the last: subnormal products and sums
        x = (x0 * scale).to(torch.bfloat16)
        outs = {}
        for mode, layer in layers.items():
            layer.route(x, int(torch.cuda.current_stream().cuda_stream))
            torch.cuda.synchronize()
            outs[mode] = [t.clone() for t in (layer.topk_idx, layer.topk_w, layer.slot_dst, layer.blk_cnt,
                                               layer.counts)]
        for a, b in zip(outs["tc"], outs["fma"]):
            assert torch.equal(a, b), scale
        ref, idx, _ = router_oracle(bf16_bits(x), bf16_bits(layers["tc"].w_gate), layers["tc"].bias.cpu().numpy(),
                                    top_k)
        assert np.array_equal(layers["tc"].topk_idx.cpu().numpy(), idx)
        _check_logits(layers["tc"], ref, idx)
        # the certificate's bound on every (token, expert): |a_e - L_e| against
        # 2^-8 |La_e| + 2^-20 (|a_e| + 1) + 2^-13 S_t, a_e = La_e + bias_e (fp32), L_e the defined logit
        lt = layers["tc"]
        la = lt.la_buf[:, :experts].float().cpu().numpy().astype(np.float64)
        a = (lt.la_buf[:, :experts].float() + lt.bias).cpu().numpy().astype(np.float64)
        xa = np.abs(x.float().cpu().numpy().astype(np.float64))
        S = xa @ np.abs(lt.w_gate.float().cpu().numpy().astype(np.float64)).max(axis=0)
        err = np.abs(a - np.asarray(ref, np.float64))
        rest = 2.0 ** -20 * (np.abs(a) + 1) + 2.0 ** -13 * S[:, None]
        assert (err <= 2.0 ** -8 * np.abs(la) + rest).all(), scale  # the bound holds
        # beyond the worst-case bf16 rounding of La (which the bf16 term is exactly), the tensor-core
        # and defined-order accumulation use under half of their allowance
        beyond = np.maximum(err - 2.0 ** -8 * np.abs(la), 0.0) / rest
        assert beyond.max() < 0.5, (scale, float(beyond.max()))
    nfb = int(layers["tc"].n_fallback.item())
    assert nfb < 3 * cfg.tokens  # most tokens certified even with the near-twins


@pytest.mark.parametrize("experts,top_k,hidden,ranks", [(1, 1, 256, 1), (2, 1, 512, 2), (3, 2, 768, 1),
                                                         (5, 3, 1024, 1), (7, 7, 256, 7), (8, 8, 512, 8),
                                                         (8, 1, 4096, 8), (4, 2, 2048, 4)])
def test_router_small_e_vs_oracle(torch, experts, top_k, hidden, ranks):
    """The E <= 8 router (bf16 gate rows by TMA, FHFMA.BF16 terms) at every expert count and k:
    top-k, softmax weights, destinations and the traffic matrix bit-exact with the oracle, on
    Gaussian and on 2^-118-scaled (subnormal-product) inputs."""
    from oracle.oracle import bf16_bits, pack_oracle, router_oracle
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg = MoEConfig(hidden=hidden, ffn=256, experts=experts, top_k=top_k, tokens=64 * 4 * ranks, ranks=ranks,
                    skew=0.7, seed=41)
    gpu_of = [e * ranks // experts for e in range(experts)]
    layer = AuroraMoELayer(cfg, gpu_of_expert=gpu_of)
    g = torch.Generator(device="cuda").manual_seed(13)
    x0 = torch.randn(cfg.tokens, hidden, device="cuda", generator=g)
    for scale in (1.0, 2.0 ** -118):
        x = (x0 * scale).to(torch.bfloat16)
        layer.route(x, int(torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        _, idx, wts = router_oracle(bf16_bits(x), bf16_bits(layer.w_gate), layer.bias.cpu().numpy(), top_k)
        assert np.array_equal(layer.topk_idx.cpu().numpy(), idx), scale
        assert np.allclose(layer.topk_w.cpu().numpy(), wts, atol=1e-6), scale
        counts, _, _ = pack_oracle(idx, gpu_of, ranks)
        assert np.array_equal(layer.counts.cpu().numpy(), counts), scale


@pytest.mark.parametrize("experts,top_k", [(8, 2), (32, 4)])
def test_layer_cuda_graph_replay(torch, experts, top_k):
    """The whole forward captured as one CUDA graph: replays with new inputs
    written into the captured buffer match the eager forward bit for bit (the
    kernels read counts, schedule and group sizes from device memory)."""
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg = MoEConfig(hidden=512, ffn=256, experts=experts, top_k=top_k, tokens=4096, ranks=8, skew=1.0, seed=21)
    layer = AuroraMoELayer(cfg)
    xs = [torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16) for _ in range(3)]
    refs = [layer(x).clone() for x in xs]
    torch.cuda.synchronize()
    xbuf = xs[0].clone()
    obuf = torch.empty_like(xbuf)
    g, y = layer.capture(xbuf, obuf)
    for rep in range(2):
        for x, ref in zip(xs, refs):
            xbuf.copy_(x)
            g.replay()
            torch.cuda.synchronize()
            layer.check_status()
            assert torch.equal(y, ref), rep
    assert int(layer.ctr_d.abs().sum()) == 0 and int(layer.ctr_c.abs().sum()) == 0


def test_random_configs_all_variants_identical(torch):
    """Race hunt (tools/stress.py): random small configs (2-16 ranks, 1-4 experts per
    rank, top-1..6, skews 0-3, emulated compute on some), each through every variant
    that must give the same bits -- default, engine combine, serial K2, unpaced, N1,
    LSU engine, ungrouped / unscattered E > n paths, deadline pacing -- twice, counters
    re-armed."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "stress", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "stress.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    m.main(40, 7)


def test_deadline_pacing_same_rows(torch):
    """Deadline pacing (a run may start at its phase's scheduled time as well as on its
    hand-over flag) changes when rows move, never which: the dispatch and the engine
    combine give the default's bits at a realistic rate, at a rate so high that every
    deadline has passed (the engine in phase order, unpaced in effect) and on host-loaded
    baseline tables (load_schedule fills the phase durations)."""
    import paper_2410_17043_b200 as A
    from paper_2410_17043_b200 import baselines as B
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    cfg = MoEConfig(hidden=1024, ffn=256, experts=8, top_k=2, tokens=4096, ranks=8, skew=1.5, seed=21)
    layer = AuroraMoELayer(cfg)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    ref = layer(x).clone()
    for fused in (True, False):
        layer.fused_combine = fused
        for gbps in (700.0, 1e9):
            layer.deadline_gbps = gbps
            for _ in range(2):
                out = layer(x)
                torch.cuda.synchronize()
                layer.check_status()
                assert torch.equal(out, ref), (fused, gbps)
    d = layer.counts.cpu().numpy().astype(float)
    np.fill_diagonal(d, 0)
    sched = B.schedule_rcs(A.TrafficMatrix(d), A.ClusterSpec.uniform(8), 3)
    layer.deadline_gbps = 700.0
    s = torch.cuda.current_stream().cuda_stream
    layer.route(x, s)
    layer.pack(s)
    layer.load_schedule(sched)
    layer.dispatch(s)
    layer.experts(s)
    layer.combine(s)
    layer.aggregate(s)
    torch.cuda.synchronize()
    layer.check_status()
    assert torch.equal(layer.out, ref)
