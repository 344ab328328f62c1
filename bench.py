"""Benchmark of the Aurora MoE-layer hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--skew S]

Workload (BASELINE.json configs[1], "C2"): Mixtral-8x7B-shaped MoE layer,
hidden 4096, FFN 14336, 8 experts top-2, bf16, 16384 tokens, expert-parallel
over 8 ranks, synthetic Zipf-skewed routing (s = 1.0), random-init weights.
A step is one layer forward over the 16384 tokens: router + traffic matrix,
on-device Aurora schedule, token pack, scheduled dispatch, tcgen05 SwiGLU
experts, reversed-schedule combine, aggregation. With N GPUs each GPU drives
8/N ranks (N = 1: all eight ranks on one B200, the engine's peer stores land
in local HBM; N = 8: one rank per GPU over NVSwitch). Total work is fixed:
"scaling": "strong".

``--impl reference`` times the reference's CPU path: the oracle port
(oracle/, a restatement of the reference's build_schedule plus the CPU
restatement of router / SwiGLU experts / aggregation) on a bounded token
sample of the same workload, with all host threads.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE-layer all-to-all µs vs send/recv lower bound; layer tokens/s at 1/2/4/8 B200"
NVLINK_GBS = 900.0  # nominal per direction per GPU (the paper's big-switch B)
NVLINK_MEASURED_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skew", type=float, default=1.0)
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--ffn", type=int, default=14336)
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--topk", type=int, default=2)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--ranks", type=int, default=8, help="expert-parallel ranks (GPUs of the modelled cluster)")
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c3h", "c4", "c5"],
                    help="c2: Mixtral-8x7B layer (the headline); c3: C2's model colocated with a 16-expert "
                         "top-2 model (hidden 4096, FFN 7168; the config leaves F open) on the same 8 ranks by "
                         "Aurora's colocation plan (single GPU only); c4: C2 on an emulated heterogeneous "
                         "cluster (bandwidths 100/80/50/40 x2, PAPER.md:666; placement by "
                         "assign_exclusive_hetero; copy CTAs per rank follow bandwidth); c5: DeepSeek-style "
                         "64 experts top-6, hidden 5120, FFN 1536 (DeepSeek-V2 expert size; the config "
                         "leaves F open); c3h: C3 on C4's emulated heterogeneous cluster, placed by "
                         "colocate_heterogeneous (placement.py:129-157)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def apply_preset(args):
    if args.config == "c5":
        args.hidden, args.ffn, args.experts, args.topk = 5120, 1536, 64, 6
    return args


C4_BANDWIDTHS = (1.0, 1.0, 0.8, 0.8, 0.5, 0.5, 0.4, 0.4)  # PAPER.md:666 ratios 100/80/50/40, two ranks each


def workload(args):
    name = {"c2": "C2 Mixtral-8x7B MoE layer", "c3": "C3 Mixtral-8x7B + 16-expert top-2 layers colocated",
            "c3h": "C3 colocated layers on C4's heterogeneous emulation (colocate_heterogeneous)",
            "c4": "C4 Mixtral-8x7B MoE layer, heterogeneous emulation",
            "c5": "C5 DeepSeek-style 64-expert top-6 MoE layer"}[args.config]
    return {"workload": f"{name} (EP over {args.ranks} ranks)", "hidden": args.hidden, "ffn": args.ffn,
            "experts": args.experts, "top_k": args.topk, "tokens": args.tokens, "ranks": args.ranks,
            "skew": args.skew, "seed": args.seed, "gpus": args.gpus,
            **({"bandwidths": list(C4_BANDWIDTHS)} if args.config in ("c4", "c3h") else {}),
            "l2": "inputs larger than L2 (x >= 128 MiB, expert weights >= 2.6 GiB read every step)"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, path):
        self.path = path
        self.p = None

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
            self.f.close()

    def summary(self, device_index=0):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        try:
            rows = [r.split(", ") for r in open(self.path).read().strip().splitlines()]
            rows = [r for r in rows if len(r) >= 9 and r[0].strip() == str(device_index)]
            if not rows:
                return out
            sm = sorted(int(float(r[1])) for r in rows)
            out["sm_mhz"] = sm[len(sm) // 2]
            out["sm_max_mhz"] = int(float(rows[0][2]))
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            reasons = set()
            for r in rows:
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            out["reasons"] = sorted(reasons)
            out["samples"] = len(rows)
        except Exception:
            pass
        return out


# ------------------------------------------------------------------ reference arm / cpu baseline
def host_cores() -> int:
    """Host threads this process may use (the CPU legs run on all of them)."""
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_package():
    """The reference package ``moeplan`` from its offline install (baseline/_ref, made by
    ``pip install --target baseline/_ref``; it travels to the GPU box with the snapshot),
    or None. /root/reference itself is never read at run time."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "moeplan")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import moeplan
        return moeplan
    except Exception:
        return None


def reference_schedule_timing(counts, bandwidths=None, reps=30):
    """The reference's own CPU hot path on a traffic matrix: moeplan.build_schedule
    (commsched.py:291-324) and simulate_exclusive (sim.py:130-154), timed with
    time.perf_counter (median of ``reps``; single-threaded Python, 1 core), next to
    the C restatement (oracle/sched_oracle.c); plus whether both give the same phases."""
    import numpy as np
    from oracle.oracle import build_schedule_oracle
    d = np.asarray(counts, dtype=float).copy()
    np.fill_diagonal(d, 0)
    n = d.shape[0]

    def med(fn):
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            r = fn()
            ts.append(time.perf_counter() - t0)
        return 1e3 * sorted(ts)[len(ts) // 2], r

    port_ms, o = med(lambda: build_schedule_oracle(d, bandwidths))
    out = {"on": "this run's traffic matrix (off-diagonal token counts)", "n": n, "reps": reps, "cores": 1,
           "port_build_schedule_ms": port_ms, "port": "oracle/sched_oracle.c (C restatement, 1 thread)"}
    m = reference_package()
    if m is None:
        out["moeplan"] = "unavailable: baseline/_ref not installed"
        return out
    tm = m.TrafficMatrix(d)
    cl = (m.ClusterSpec.uniform(n) if bandwidths is None else
          m.ClusterSpec(tuple(m.GpuSpec(float(b), float(b)) for b in bandwidths)))
    ref_ms, sched = med(lambda: m.build_schedule(tm, cl))
    prof = m.LayerProfile(0.0, 0.0, 0.0, 0.0, tm)
    sim_ms, _ = med(lambda: m.simulate_exclusive(prof, m.DeploymentPlan.identity(n), cl))
    out.update({"moeplan_build_schedule_ms": ref_ms, "moeplan_simulate_exclusive_ms": sim_ms,
                "moeplan": "baseline/_ref (the reference itself, unmodified)",
                "phases": len(sched.phases),
                "port_identical": [(p.transfers, p.duration) for p in sched.phases] == o["phases"]})
    return out


def cpu_reference_step(x_bits, w_gate_bits, bias, w1, w3, w2, k, n, gpu_of_expert):
    """One pass of the CPU path over a token sample: router (oracle C), traffic
    matrix + permutation, the schedule by the reference itself (moeplan.build_schedule
    from baseline/_ref; the C restatement if it is not installed), fp32 SwiGLU experts
    (numpy BLAS, all threads), gate-weighted aggregation."""
    from oracle.oracle import build_schedule_oracle, moe_layer_oracle, pack_oracle, router_oracle
    import numpy as np
    import torch
    _, idx, wts = router_oracle(x_bits, w_gate_bits, bias, k)
    counts, _, _ = pack_oracle(idx, gpu_of_expert, n)
    d = counts.astype(float)
    np.fill_diagonal(d, 0)
    m = reference_package()
    if m is not None:
        m.build_schedule(m.TrafficMatrix(d), m.ClusterSpec.uniform(n))
    else:
        build_schedule_oracle(d)
    x = torch.from_numpy(x_bits.astype(np.int32) << 16).view(torch.float32).numpy()
    return moe_layer_oracle(x, idx, wts, w1, w3, w2)


def cpu_weights(args, seed=0):
    import torch
    from paper_2410_17043_b200.layer import zipf_bias
    H, F, E = args.hidden, args.ffn, args.experts
    g = torch.Generator().manual_seed(seed)
    w_gate = (torch.randn(E, H, generator=g) / math.sqrt(H)).to(torch.bfloat16)
    bias = zipf_bias(E, args.skew, g).numpy()
    ge = torch.Generator().manual_seed(seed + 7)
    # bf16 on the host (2.6 GiB at C2); the oracle widens one expert at a time
    w1 = [(torch.randn(F, H, generator=ge) / math.sqrt(H)).to(torch.bfloat16) for _ in range(E)]
    w3 = [(torch.randn(F, H, generator=ge) / math.sqrt(H)).to(torch.bfloat16) for _ in range(E)]
    w2 = [(torch.randn(H, F, generator=ge) / math.sqrt(F)).to(torch.bfloat16) for _ in range(E)]
    return w_gate, bias, w1, w3, w2


def run_cpu(args, sample_tokens, reps, seed=0, weights=None):
    """Times the CPU path (cpu_reference_step) on `sample_tokens` tokens of the
    workload with every host thread. Returns (tokens/s, seconds per rep, threads)."""
    import numpy as np
    import torch
    cores = host_cores()
    torch.set_num_threads(cores)
    E, k, n = args.experts, args.topk, args.ranks
    w_gate, bias, w1, w3, w2 = weights or cpu_weights(args, seed)
    gx = torch.Generator().manual_seed(seed + 5)
    x = torch.randn(sample_tokens, args.hidden, generator=gx).to(torch.bfloat16)
    xb = x.view(torch.int16).numpy().view(np.uint16)
    wb = w_gate.view(torch.int16).numpy().view(np.uint16)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        cpu_reference_step(xb, wb, bias, w1, w3, w2, k, n, [e // (E // n) for e in range(E)])
        times.append(time.perf_counter() - t0)
    med = sorted(times)[len(times) // 2]
    return sample_tokens / med, med, cores


def cpu_full_counts(args, weights, seed=0):
    """The full workload's traffic matrix computed on the host (oracle router over
    all T tokens of a CPU-generated input): what the reference arm schedules."""
    import numpy as np
    import torch
    from oracle.oracle import pack_oracle, router_oracle
    w_gate, bias = weights[0], weights[1]
    gx = torch.Generator().manual_seed(seed + 9)
    x = torch.randn(args.tokens, args.hidden, generator=gx).to(torch.bfloat16)
    _, idx, _ = router_oracle(x.view(torch.int16).numpy().view(np.uint16),
                              w_gate.view(torch.int16).numpy().view(np.uint16), bias, args.topk)
    E, n = args.experts, args.ranks
    counts, _, _ = pack_oracle(idx, [e // (E // n) for e in range(E)], n)
    return counts


def reference_arm(args):
    import torch.distributed as dist  # noqa: F401
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sample = 256
    reps = max(1, args.steps)
    weights = cpu_weights(args)
    for _ in range(min(args.warmup, 1)):
        run_cpu(args, sample, 1, weights=weights)
    tps, sec, cores = run_cpu(args, sample, reps, weights=weights)
    sched = reference_schedule_timing(cpu_full_counts(args, weights),
                                      list(C4_BANDWIDTHS[:args.ranks]) if args.config == "c4" else None)
    # the layer figure is the port (the reference has no token path); its schedule is the reference's own
    kind = "port"
    line = {"impl": "reference", "metric": METRIC, "value": tps, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": reps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload(args),
            "cpu_baseline": {"value": tps, "unit": "tokens/s", "cores": cores, "kind": kind,
                             "cpu_count": os.cpu_count(), "affinity": host_cores(),
                             "sample": f"{sample} tokens of the layer per step: oracle router + traffic matrix, "
                                       f"the schedule by moeplan.build_schedule (baseline/_ref), fp32 numpy "
                                       f"SwiGLU experts + aggregation on {cores} threads",
                             "schedule": sched,
                             "schedule_impl": ("reference: moeplan.build_schedule from baseline/_ref"
                                               if reference_package() is not None else "port")},
            "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------ our arm
def library_alltoall(layer, x, args, world, rank, stream, reps=5):
    """Unscheduled library all-to-all of the same dispatch rows. N = 1 (all ranks on
    one GPU): one torch.index_select gathering every rank's rows into receive order
    (the single-GPU stand-in: NCCL cannot run several ranks on one GPU). N > 1, one
    rank per GPU: the NCCL alltoallv the engine replaces -- pack by send list,
    device-to-host read of the split sizes, dist.all_to_all_single."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2410_17043_b200 import _lib
    sp = _lib.stream_ptr(stream)
    layer.route(x, sp)
    layer.exchange_counts()
    layer.pack(sp)
    torch.cuda.synchronize()
    n, Tr = layer.n, layer.cfg.tokens_per_rank
    counts = layer.counts.cpu().numpy()
    soff = layer.soff.cpu().numpy()
    sl = layer.send_list.cpu().numpy()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    if world == 1:
        idx = []
        for j in range(n):
            for i in [j] + [q for q in range(n) if q != j]:
                idx.append(sl[i, soff[i, j]:soff[i, j] + counts[i, j]] + i * Tr)
        idx = torch.from_numpy(np.concatenate(idx).astype(np.int64)).to(x.device)
        out = torch.empty(idx.numel(), x.shape[1], dtype=x.dtype, device=x.device)
        torch.index_select(x, 0, idx, out=out)
        torch.cuda.synchronize()
        ev[0].record(stream)
        for _ in range(reps):
            torch.index_select(x, 0, idx, out=out)
        ev[1].record(stream)
        torch.cuda.synchronize()
        return {"torch_index_select_us": ev[0].elapsed_time(ev[1]) / reps * 1e3, "rows": int(idx.numel()),
                "note": "one gather kernel moving every dispatched row into receive order (all ranks on one GPU)"}
    if os.environ.get("AURORA_BENCH_SAME_GPU", "0") == "1":
        return {"unavailable": "processes share one GPU (gloo host collectives): no NCCL"}
    # one process per GPU driving n_local ranks: the unscheduled NCCL alltoallv at process
    # granularity -- every row from this process's ranks to process q's ranks in one split
    # (rank order, then send-list order), rows between ranks of the same process included
    nl, rb, P = layer.n_local, layer.rank_base, n // layer.n_local
    idx, in_split, out_split = [], [], []
    for q in range(P):
        dst = range(q * nl, (q + 1) * nl)
        for i in range(rb, rb + nl):
            for j in dst:
                idx.append(sl[i - rb, soff[i, j]:soff[i, j] + counts[i, j]] + (i - rb) * Tr)
        in_split.append(int(sum(counts[i, j] for i in range(rb, rb + nl) for j in dst)))
        out_split.append(int(sum(counts[i, j] for i in range(q * nl, (q + 1) * nl) for j in range(rb, rb + nl))))
    lst = torch.from_numpy(np.concatenate(idx).astype(np.int64)).to(x.device)
    recv = torch.empty(sum(out_split), x.shape[1], dtype=x.dtype, device=x.device)
    tot = 0.0
    for r_ in range(reps + 1):
        dist.barrier()
        torch.cuda.synchronize()
        ev[0].record(stream)
        send = torch.index_select(x, 0, lst)
        c = layer.counts.cpu()  # alltoallv needs the split sizes on the host (a D2H sync every step)
        ins = [int(c[rb:rb + nl, q * nl:(q + 1) * nl].sum()) for q in range(P)]
        outs = [int(c[q * nl:(q + 1) * nl, rb:rb + nl].sum()) for q in range(P)]
        dist.all_to_all_single(recv, send, output_split_sizes=outs, input_split_sizes=ins)
        ev[1].record(stream)
        torch.cuda.synchronize()
        if r_:
            tot += ev[0].elapsed_time(ev[1])
    t = torch.tensor([tot / reps * 1e3], dtype=torch.float64, device=x.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"nccl_alltoallv_us": float(t.item()), "ranks_per_gpu": nl,
            "note": "pack (index_select) + D2H split sizes + dist.all_to_all_single between processes "
                    "(one split per GPU, its ranks' rows back to back), max over ranks",
            "symm_mem_all_to_all_vdev": "unavailable: needs NVSHMEM (not in this image)"}


def baseline_schedules(layer, x, sp, stream, reps=3):
    """SURVEY 8(f)3 / PAPER.md:747: the paper's SJF and RCS schedules of the same
    traffic matrix, executed by the same engine (host-built tables)."""
    import numpy as np
    import torch
    from paper_2410_17043_b200 import baselines as B
    from paper_2410_17043_b200.core import ClusterSpec, TrafficMatrix
    d = layer.counts.cpu().numpy().astype(float)
    np.fill_diagonal(d, 0)
    tm, cl = TrafficMatrix(d), ClusterSpec.uniform(layer.n)
    out = {}
    for name, sched in (("sjf", B.schedule_sjf(tm, cl)), ("rcs", B.schedule_rcs(tm, cl, 0))):
        if len(sched.phases) > layer.P:
            continue
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        disp = comb = 0.0
        for _ in range(reps):
            layer.route(x, sp)
            layer.pack(sp)
            layer.load_schedule(sched)
            ev[0].record(stream)
            layer.dispatch(sp)
            ev[1].record(stream)
            layer.experts(sp)
            ev[2].record(stream)
            layer.combine(sp)
            ev[3].record(stream)
            layer.aggregate(sp)
            torch.cuda.synchronize()
            disp += ev[0].elapsed_time(ev[1])
            comb += ev[2].elapsed_time(ev[3])
        layer.check_status()
        out[name] = {"dispatch_us": disp / reps * 1e3, "combine_us": comb / reps * 1e3,
                     "makespan_tokens": sched.makespan, "phases": len(sched.phases)}
    return out


GEMM_CAPTURE = "profiles/r02_ncu_gemm.json"


def n1_effect(layer, x, stream, steps):
    """N1 (north_star (4)): the arrival-driven expert GEMM -- GEMM1 a programmatic dependent
    of an LSU dispatch (one copy CTA per SM), each tile starting once its rows have landed --
    against the default plan (TMA dispatch on every SM, then GEMM1), alternated three times;
    plus one traced N1 step: when GEMM1's first tiles started relative to the dispatch CTAs."""
    import numpy as np
    import torch
    from paper_2410_17043_b200 import _lib
    if layer.G != 1 or not layer.combine_in_gemm:
        return {"unavailable": "one expert per rank with the fused combine only"}
    L = _lib.load()
    times = {"default": [], "n1": []}
    for _ in range(3):
        for name, on in (("default", False), ("n1", True)):
            layer.arrival = on
            for _ in range(2):
                layer(x)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                layer(x)
            e1.record(stream)
            torch.cuda.synchronize()
            layer.check_status()
            times[name].append(e0.elapsed_time(e1) / steps)
    layer.arrival = True
    eng = torch.zeros(4 * 4096, dtype=torch.int64, device=x.device)
    gt = torch.zeros(2 * 1024, dtype=torch.int64, device=x.device)
    L.aurora_debug_set_engine_trace(eng.data_ptr())
    L.aurora_debug_set_gemm_trace(gt.data_ptr())
    try:
        layer(x)
        torch.cuda.synchronize()
    finally:
        L.aurora_debug_set_engine_trace(None)
        L.aurora_debug_set_gemm_trace(None)
        layer.arrival = False
    layer.check_status()
    e = eng.view(-1, 4).cpu().numpy()
    e = e[e[:, 0] > 0]
    g = gt.view(-1, 2).cpu().numpy()
    g = g[g[:, 0] > 0]
    t0 = float(e[:, 0].min())
    trace = {"dispatch_ctas": int(len(e)), "dispatch_end_us": float(e[:, 2].max() - t0) / 1e3,
             "dispatch_local_rows_done_us": float(e[:, 1].max() - t0) / 1e3,
             "gemm1_ctas": int(len(g)), "gemm1_last_cta_entry_us": float(g[:, 0].max() - t0) / 1e3,
             "gemm1_first_cta_entry_us": float(g[:, 0].min() - t0) / 1e3,
             "gemm1_first_tile_us": float(g[g[:, 1] > 0][:, 1].min() - t0) / 1e3 if (g[:, 1] > 0).any() else None,
             "gemm1_ctas_started_before_dispatch_end": int((g[:, 0] < e[:, 2].max()).sum())}
    med = {k: float(np.median(v)) for k, v in times.items()}
    return {"default_ms_per_step": med["default"], "n1_ms_per_step": med["n1"], "runs": times,
            "speedup": med["default"] / med["n1"], "trace_us_from_dispatch_start": trace,
            "switch": "AURORA_N1=1", "default_on": False}


def placement_effect(layer, cfg, plan, bws, x, stream, steps):
    """C4: the Theorem-3 placement (assign_exclusive_hetero,
    placement.py:46-60: the k-th most loaded expert on the k-th fastest rank) against
    the identity placement on the same emulated cluster (per-rank copy CTAs and GEMM
    CTA pairs in proportion to the ranks' bandwidth / compute scale). Steps alternate
    between the two layers (same power state); per-rank GEMM work is reported too."""
    import numpy as np
    import torch
    from paper_2410_17043_b200 import DeploymentPlan
    from paper_2410_17043_b200.layer import AuroraMoELayer
    ident = AuroraMoELayer(cfg, DeploymentPlan.identity(cfg.ranks), bandwidths=bws, compute_scales=bws)
    layers = {"theorem3": layer, "identity": ident}
    for L in layers.values():
        for _ in range(2):
            L(x)
    torch.cuda.synchronize()
    times = {k: [] for k in layers}
    for _ in range(3):
        for name, L in layers.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                L(x)
            e1.record(stream)
            torch.cuda.synchronize()
            L.check_status()
            times[name].append(e0.elapsed_time(e1) / steps)
    out = {}
    for name, L in layers.items():
        rows = L.counts.cpu().numpy().sum(axis=0).astype(float)   # rows each rank's expert processes
        part = np.diff(L.gemm_part.cpu().numpy())                  # CTA pairs per rank
        tiles = np.ceil(rows / 256)                                # m-tiles (256 rows) per rank
        out[name] = {"assignment": list(L.plan.assignment_a), "ms_per_step": sorted(times[name])[1],
                     "ms_per_step_runs": times[name], "rows_per_rank": rows.tolist(),
                     "gemm_pairs_per_rank": part.tolist(),
                     "gemm_critical_rank": int(np.argmax(tiles / part)),
                     "gemm_work_ratio_max_over_mean": float((tiles / part).max() / (tiles.sum() / part.sum()))}
    out["speedup_theorem3_vs_identity"] = out["identity"]["ms_per_step"] / out["theorem3"]["ms_per_step"]
    del ident
    torch.cuda.empty_cache()
    return out


def gemm_traffic(args):
    """DRAM bytes (read + write) of the expert GEMM launches of one C2 step,
    from the committed ncu --set full capture; None for other workloads."""
    if args.config != "c2":
        return None
    try:
        rec = json.load(open(os.path.join(ROOT, GEMM_CAPTURE)))["grouped_gemm_2sm_kernel"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for launch in rec:
            for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                v, u = launch[key].split()
                tot += float(v) * scale[u]
        return tot
    except Exception:
        return None


def run_c3(args):
    """C3: two models colocated on the same ranks by Aurora's plan (colocation.py:
    Lina-style slots of model b, colocate_homogeneous pairing, placement.py:109-126).
    A step = one layer of each model over its 16384 tokens; value = both models'
    tokens per second. Single GPU (loopback)."""
    import numpy as np
    import torch
    from paper_2410_17043_b200 import _lib
    from paper_2410_17043_b200.colocation import ColocatedLayers, combined_bmax, lina_slots, plan_colocation
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        raise SystemExit("--config c3 runs on one GPU")
    n = args.ranks
    cfg_a = MoEConfig(hidden=4096, ffn=14336, experts=n, top_k=2, tokens=args.tokens, ranks=n, skew=args.skew,
                      seed=args.seed)
    cfg_b = MoEConfig(hidden=4096, ffn=7168, experts=2 * n, top_k=2, tokens=args.tokens, ranks=n, skew=1.5,
                      seed=args.seed + 1)
    g = torch.Generator(device="cuda").manual_seed(args.seed + 101)
    xa = torch.randn(cfg_a.tokens, cfg_a.hidden, device="cuda", generator=g).to(torch.bfloat16)
    xb = torch.randn(cfg_b.tokens, cfg_b.hidden, device="cuda", generator=g).to(torch.bfloat16)
    sp = _lib.stream_ptr()
    # deployment-time calibration: the routers alone give the traffic matrices
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
    cplan = plan_colocation(counts_a, slot_counts, slots)
    hetero = args.config == "c3h"
    kw, homo_pair, bws = {}, None, None
    if hetero:  # C4's cluster: per-rank copy CTAs and GEMM CTA pairs follow bandwidth / compute scale
        from paper_2410_17043_b200 import ClusterSpec, GpuSpec
        from paper_2410_17043_b200.colocation import expert_work, plan_colocation_hetero
        bws = C4_BANDWIDTHS[:n]
        kw = {"bandwidths": bws, "compute_scales": bws}
        cluster = ClusterSpec(tuple(GpuSpec(b, b) for b in bws))
        homo_plan = cplan
        cplan = plan_colocation_hetero(counts_a, slot_counts, slots, cluster, expert_work(4096, 14336),
                                       expert_work(4096, 7168))
        homo_pair = ColocatedLayers(cfg_a, cfg_b, homo_plan, **kw)
    pair = ColocatedLayers(cfg_a, cfg_b, cplan, **kw)
    if homo_pair is not None:
        homo_pair.interleave = pair.interleave
    for _ in range(args.warmup):
        pair(xa, xb)
    torch.cuda.synchronize()
    pair.check_status()
    st = torch.cuda.current_stream()
    clocks = ClockSampler(os.path.join(ROOT, "gpurun_out", "clocks_r0.csv")
                          if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else "/tmp/clocks_r0.csv")
    with clocks:
        time.sleep(0.3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.steps):
            pair(xa, xb)
        e1.record(st)
        torch.cuda.synchronize()
        time.sleep(0.2)
    pair.check_status()
    ms = e0.elapsed_time(e1) / args.steps
    # Table-1 interleaving vs the serial order (model a's layer, then model b's), alternated
    # three times so both see the same power state; the headline uses the layer's default
    il_default = pair.interleave
    il_runs = {"interleaved": [], "serial": []}
    for _ in range(3 if not hetero else 0):
        for name, il in (("interleaved", True), ("serial", False)):
            pair.interleave = il
            pair(xa, xb)
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(st)
            for _ in range(args.steps):
                pair(xa, xb)
            f1.record(st)
            torch.cuda.synchronize()
            pair.check_status()
            il_runs[name].append(f0.elapsed_time(f1) / args.steps)
    if not hetero:
        pair.interleave = True
        il_timeline = pair.timeline(xa, xb)
        pair.interleave = il_default
        il_med = {k: sorted(v)[1] for k, v in il_runs.items()}
    # end to end: both inputs in from pinned host memory, both outputs back, every step
    # pipelined like the C2 line: copy-engine streams move the next step's inputs in and the
    # previous step's outputs out under the layers, double-buffered device inputs / outputs
    NB = 2
    xah = [xa.cpu().pin_memory() for _ in range(NB)]
    xbh = [xb.cpu().pin_memory() for _ in range(NB)]
    oah = [torch.empty_like(xah[0]).pin_memory() for _ in range(NB)]
    obh = [torch.empty_like(xbh[0]).pin_memory() for _ in range(NB)]
    xad = [torch.empty_like(xa) for _ in range(NB)]
    xbd = [torch.empty_like(xb) for _ in range(NB)]
    oad = [torch.empty_like(xa) for _ in range(NB)]
    obd = [torch.empty_like(xb) for _ in range(NB)]
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    ev = {key: [torch.cuda.Event() for _ in range(NB)]
          for key in ("in_a", "in_b", "done_a", "done_b", "out_a", "out_b")}
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e2.record(st)
    for i in range(args.steps):
        bb = i % NB
        if i >= NB:  # step i-NB finished reading the input buffers
            h2d_s.wait_event(ev["done_b"][bb])
        with torch.cuda.stream(h2d_s):
            xad[bb].copy_(xah[bb], non_blocking=True)
            ev["in_a"][bb].record(h2d_s)
            xbd[bb].copy_(xbh[bb], non_blocking=True)
            ev["in_b"][bb].record(h2d_s)
        if i >= NB:  # the output buffers were drained to the host
            st.wait_event(ev["out_b"][bb])
        st.wait_event(ev["in_a"][bb])
        st.wait_event(ev["in_b"][bb])
        pair(xad[bb], xbd[bb], out_a=oad[bb], out_b=obd[bb])
        ev["done_a"][bb].record(st)
        ev["done_b"][bb].record(st)
        d2h_s.wait_event(ev["done_a"][bb])
        with torch.cuda.stream(d2h_s):
            oah[bb].copy_(oad[bb], non_blocking=True)
            ev["out_a"][bb].record(d2h_s)
        d2h_s.wait_event(ev["done_b"][bb])
        with torch.cuda.stream(d2h_s):
            obh[bb].copy_(obd[bb], non_blocking=True)
            ev["out_b"][bb].record(d2h_s)
    st.wait_event(ev["out_b"][(args.steps - 1) % NB])
    st.wait_event(ev["out_a"][(args.steps - 1) % NB])
    e3.record(st)
    torch.cuda.synchronize()
    e2e_ms = e2.elapsed_time(e3) / args.steps
    rows = float(pair.a.counts.sum().item()) * 14336 + float(pair.b.g_rows.sum().item()) * 7168
    flops = rows * 2 * 3 * 4096
    tokens = cfg_a.tokens + cfg_b.tokens
    line = {"metric": METRIC, "value": tokens / (ms * 1e-3), "unit": "tokens/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "config": workload(args),
            "colocation": {"pairing": list(cplan.plan.pairing),
                           "combined_bmax_tokens": combined_bmax(counts_a, slot_counts, cplan.plan),
                           "model_b": {"experts": 2 * n, "top_k": 2, "hidden": 4096, "ffn": 7168, "skew": 1.5}},
            "roofline": {"bound": "tensor", "achieved": flops / (ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                         "note": "both models' expert FLOPs over the whole step (upper bound on the GEMM time)"},
            "gpu_launches": (pair.a.kernels_per_step() + pair.b.kernels_per_step()) * args.steps,
            "e2e": {"value": tokens / (e2e_ms * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": int((xah[0].numel() + xbh[0].numel()) * 2),
                    "d2h_bytes_per_step": int((oah[0].numel() + obh[0].numel()) * 2), "ms_per_step": e2e_ms,
                    "path": "both layers' public forward on pinned host buffers",
                    "pipeline": "H2D of step i+1's inputs and D2H of step i-1's outputs under step i "
                                "(copy-engine streams, double-buffered device inputs / outputs)"},
            "clocks": clocks.summary(0),
            "interleave": ({"default_on": il_default, "switch": "AURORA_C3_INTERLEAVE=0 for the serial order",
                            "interleaved_ms_per_step": il_med["interleaved"], "serial_ms_per_step": il_med["serial"],
                            "speedup": il_med["serial"] / il_med["interleaved"], "runs": il_runs,
                            "timeline_ms": il_timeline,
                            "what": "Table 1 (PAPER.md:473-497) on one GPU: model b on a second stream, its gate "
                                    "and K2 beside model a's gate / dispatch, its dispatch right after model a's, "
                                    "its FFN behind model a's FFN, model a's aggregation beside it; combines fused"}
                           if not hetero else
                           {"default_on": False, "note": "off under the per-rank compute emulation: the two models' "
                                                         "FFNs would overlap on different SMs, giving every emulated "
                                                         "GPU twice its CTA pairs"}),
            "timeline_ms": {"a": pair.a.timeline(xa), "b": pair.b.timeline(xb)}}
    if hetero:
        # the same two models on the same emulated cluster, pairs placed by the homogeneous plan
        # (pair p on GPU p) vs colocate_heterogeneous's stage 2; alternated for equal power state
        res = {"colocate_heterogeneous": [], "homogeneous_plan": []}
        for p_ in (pair, homo_pair):
            for _ in range(2):
                p_(xa, xb)
        torch.cuda.synchronize()
        for _ in range(3):
            for name, p_ in (("colocate_heterogeneous", pair), ("homogeneous_plan", homo_pair)):
                f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                f0.record(st)
                for _ in range(args.steps):
                    p_(xa, xb)
                f1.record(st)
                torch.cuda.synchronize()
                p_.check_status()
                res[name].append(f0.elapsed_time(f1) / args.steps)
        med = {k: sorted(v)[1] for k, v in res.items()}
        line["placement"] = {
            "colocate_heterogeneous": {"ms_per_step": med["colocate_heterogeneous"], "runs": res["colocate_heterogeneous"],
                                       "gpu_of_a": list(cplan.gpu_of_a), "gpu_of_b": list(cplan.gpu_of_b)},
            "homogeneous_plan": {"ms_per_step": med["homogeneous_plan"], "runs": res["homogeneous_plan"],
                                 "gpu_of_a": list(homo_pair.cplan.gpu_of_a), "gpu_of_b": list(homo_pair.cplan.gpu_of_b)},
            "speedup": med["homogeneous_plan"] / med["colocate_heterogeneous"],
            "work_model": "LayerProfile work in the reference's time unit from measured rates (colocation.expert_work)"}
    print(json.dumps(line))
    return 0


def main():
    args = apply_preset(parse())
    if args.impl == "reference":
        return reference_arm(args)
    if args.config in ("c3", "c3h"):
        return run_c3(args)
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2410_17043_b200 import _lib
    from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # AURORA_BENCH_SAME_GPU=1 (testing the multi-process path on a one-GPU box): every rank on
    # cuda:0, gloo for the host-side collectives (NCCL refuses two ranks on one device); the
    # data path is the same peer-memory engine over CUDA IPC
    same_gpu = os.environ.get("AURORA_BENCH_SAME_GPU", "0") == "1"
    torch.cuda.set_device(0 if same_gpu else local_rank)
    if world > 1:
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            # NCCL INIT lines on stderr: which ranks / GPUs / transports the run used
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    n = args.ranks
    if n % world:
        raise SystemExit(f"{n} ranks do not split over {world} GPUs")
    n_local = n // world
    cfg = MoEConfig(hidden=args.hidden, ffn=args.ffn, experts=args.experts, top_k=args.topk, tokens=args.tokens,
                    ranks=n, skew=args.skew, seed=args.seed)
    plan, bws = None, None
    if args.config == "c4":
        # deployment-time placement (placement.py:46-60) from a calibration pass of the router
        from paper_2410_17043_b200 import ClusterSpec, GpuSpec, assign_exclusive_hetero
        bws = C4_BANDWIDTHS[:n]
        calib = AuroraMoELayer(cfg, rank_base=rank * n_local, n_local=n_local)
        gc_ = torch.Generator(device=calib.dev).manual_seed(args.seed + 101 + rank)
        xc = torch.randn(calib.T_local, cfg.hidden, device=calib.dev, generator=gc_).to(torch.bfloat16)
        calib.route(xc, _lib.stream_ptr())  # the router alone gives the traffic matrix
        if world > 1:  # calibration pass (host side, once): plain all-reduce of the rows
            dist.all_reduce(calib.counts)
        torch.cuda.synchronize()
        loads = calib.counts.cpu().numpy().sum(axis=0)
        plan = assign_exclusive_hetero(loads, ClusterSpec(tuple(GpuSpec(b, b) for b in bws)))
        del calib
        torch.cuda.empty_cache()
    # C4: each rank also gets a compute share in proportion to its GpuSpec compute_scale (= its
    # bandwidth ratio): the expert GEMMs' CTA pairs are partitioned among the ranks
    layer = AuroraMoELayer(cfg, plan, rank_base=rank * n_local, n_local=n_local, bandwidths=bws,
                           compute_scales=bws)
    if world > 1:
        from paper_2410_17043_b200 import dist as adist
        adist.connect_peers(layer)
    dev = layer.dev
    g = torch.Generator(device=dev).manual_seed(args.seed + 101 + rank)
    x = torch.randn(layer.T_local, cfg.hidden, device=dev, generator=g).to(torch.bfloat16)
    stream = torch.cuda.current_stream()
    sp = _lib.stream_ptr(stream)

    stages = ["route", "pack", "schedule", "dispatch", "experts", "combine", "aggregate"]

    def staged_step(ev, fused=False):
        """The same kernels run serially on one stream with events between
        stages: the per-stage breakdown (the timed steps overlap stages)."""
        ev[0].record(stream)
        layer.route(x, sp)
        layer.exchange_counts()
        ev[1].record(stream)
        layer.pack(sp)
        ev[2].record(stream)
        layer.schedule(sp)
        ev[3].record(stream)
        layer.dispatch(sp)
        ev[4].record(stream)
        if fused:  # the combine inside GEMM2's epilogue; "combine" = the receivers' wait
            layer.experts_combine(sp)
            ev[5].record(stream)
            layer.combine_wait(sp)
        else:
            layer.experts(sp)
            ev[5].record(stream)
            layer.combine(sp)
        ev[6].record(stream)
        layer.aggregate(sp)
        ev[7].record(stream)

    def a2a_overlapped(reps):
        """Dispatch as the layer runs it: K2 and the PDL-launched engine together,
        from the end of pack to the last dispatched row (schedule time included)."""
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
        for r_ in range(reps):
            layer.route(x, sp)
            layer.exchange_counts()
            layer.pack(sp)
            layer.progress.zero_()
            e[2 * r_].record(stream)
            layer.schedule(sp)
            layer.dispatch(sp, overlap_schedule=True)
            e[2 * r_ + 1].record(stream)
            layer.experts(sp)
            layer.combine(sp)
            layer.aggregate(sp)
        torch.cuda.synchronize()
        layer.check_status()
        return sum(e[2 * r_].elapsed_time(e[2 * r_ + 1]) for r_ in range(reps)) / reps * 1e3

    for _ in range(args.warmup):
        layer(x)
    torch.cuda.synchronize()
    layer.check_status()

    clocks = ClockSampler(os.path.join(ROOT, "gpurun_out", f"clocks_r{rank}.csv")
                          if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else f"/tmp/clocks_r{rank}.csv")
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with clocks:
        time.sleep(0.3)
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        # the dominant kernels' window inside every timed step: the layer records these two
        # events on its stream right after the dispatch launch and after GEMM2 (GEMM1 with the
        # SwiGLU epilogue, then GEMM2 with the fused combine) -- no extra sync, same launches
        gemm_ev = [{"dispatched": torch.cuda.Event(enable_timing=True),
                    "experts_done": torch.cuda.Event(enable_timing=True)} for _ in range(args.steps)]
        t_start.record(stream)
        for i_ in range(args.steps):
            layer.trace = gemm_ev[i_]
            layer(x)  # the public forward: overlapped streams, no host sync
        layer.trace = None
        t_end.record(stream)
        torch.cuda.synchronize()
        time.sleep(0.2)
    if world > 1:
        dist.barrier()
    total_ms = t_start.elapsed_time(t_end)
    layer.check_status()
    gemm_ms_steps = [e["dispatched"].elapsed_time(e["experts_done"]) for e in gemm_ev]
    gemm_ms = sum(gemm_ms_steps) / len(gemm_ms_steps)
    ms = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_per_step = float(ms.item()) / args.steps

    # ---- end to end through the public API with host buffers (pinned), copies timed,
    # right after the headline steps (same power regime as `value`; the diagnostics below
    # run the GPU for many more steps).
    # Serving-style pipeline: the copy engines move step i+1's input in and step
    # i-1's output out while the SMs run step i (double-buffered device input and
    # output, one stream per copy direction, events order the reuse of buffers).
    NB = 2
    xh = [x.cpu().pin_memory() for _ in range(NB)]
    outh = [torch.empty_like(xh[0]).pin_memory() for _ in range(NB)]
    xd = [torch.empty_like(x) for _ in range(NB)]
    od = [torch.empty_like(x) for _ in range(NB)]
    h2d_s, d2h_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ev = {key: [torch.cuda.Event() for _ in range(NB)] for key in ("in", "done", "out")}

    def e2e_steps(steps):
        for i in range(steps):
            b = i % NB
            if i >= NB:
                h2d_s.wait_event(ev["done"][b])   # step i-NB finished reading xd[b]
            with torch.cuda.stream(h2d_s):
                xd[b].copy_(xh[b], non_blocking=True)
            ev["in"][b].record(h2d_s)
            stream.wait_event(ev["in"][b])
            if i >= NB:
                stream.wait_event(ev["out"][b])   # od[b] drained to the host
            layer(xd[b], out=od[b])
            ev["done"][b].record(stream)
            d2h_s.wait_event(ev["done"][b])
            with torch.cuda.stream(d2h_s):
                outh[b].copy_(od[b], non_blocking=True)
            ev["out"][b].record(d2h_s)
        for b in range(NB):
            stream.wait_event(ev["out"][b])

    e2e_steps(2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    e0.record(stream)
    h2d_s.wait_event(e0)
    e2e_steps(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())
    layer.check_status()
    assert torch.equal(outh[(args.steps - 1) % NB], od[(args.steps - 1) % NB].cpu())

    # ---- sustained rate (diagnostic beside the headline): the 1 kW power limiter settles
    # over ~100 ms, so 60 more back-to-back steps report the rate after it has (last 40)
    sus = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    sus[0].record(stream)
    for i_ in range(60):
        layer(x)
        if i_ == 19:
            sus[1].record(stream)
    sus[2].record(stream)
    torch.cuda.synchronize()
    layer.check_status()
    sustained = {"first_20_ms_per_step": sus[0].elapsed_time(sus[1]) / 20,
                 "last_40_ms_per_step": sus[1].elapsed_time(sus[2]) / 40}

    # ---- per-stage breakdown (serial pass, not the headline number)
    # (with the combine fused into GEMM2, the fused and the engine step alternate so
    # both see the same power / clock state)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(8)] for _ in range(args.steps)]
    evf = [[torch.cuda.Event(enable_timing=True) for _ in range(8)] for _ in range(args.steps)]
    fused = layer.combine_in_gemm
    for s_ in range(args.steps):
        staged_step(evs[s_])
        if fused:
            staged_step(evf[s_], fused=True)
    torch.cuda.synchronize()
    layer.check_status()
    stage_ms = {st: sum(e[i].elapsed_time(e[i + 1]) for e in evs) / args.steps for i, st in enumerate(stages)}
    fused_ms = ({st: sum(e[i].elapsed_time(e[i + 1]) for e in evf) / args.steps for i, st in enumerate(stages)}
                if fused else None)
    serial_ms = sum(stage_ms.values())
    # ablation: the same engine with the schedule's pacing switched off
    layer.unpaced = 16
    for s_ in range(args.steps):
        staged_step(evs[s_])
    torch.cuda.synchronize()
    layer.check_status()
    layer.unpaced = 0
    unpaced_ms = {st: sum(e[i].elapsed_time(e[i + 1]) for e in evs) / args.steps for i, st in enumerate(stages)}
    baseline_sched = baseline_schedules(layer, x, sp, stream) if world == 1 else {}
    sched_dispatch_us = a2a_overlapped(args.steps)
    try:  # a diagnostic beside the headline: never let it take the bench line down
        library_a2a = library_alltoall(layer, x, args, world, rank, stream)
    except Exception as e:  # noqa: BLE001
        library_a2a = {"unavailable": f"{type(e).__name__}: {e}"[:200]}


    # ---- roofline of the dominant kernel (the tcgen05 expert GEMMs) and the all-to-all bound
    counts = layer.counts.cpu().numpy().astype(np.int64)
    if layer.G > 1:  # one GEMM row per (token, expert) pair
        gemm_rows = float(layer.g_rows.sum().item())
    else:
        gemm_rows = float(counts.sum(axis=0)[layer.rank_base:layer.rank_base + n_local].sum())
    gemm_flops = gemm_rows * 2 * 3 * cfg.hidden * cfg.ffn
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    # peak: the timed region is a short burst right after the warm-up (< 1 s of GEMMs), so the
    # burst figure applies; a window long enough for the 1 kW limiter to settle would use the
    # sustained one (B200_PROFILING.md)
    window_s = gemm_ms * args.steps * 1e-3
    regime = "burst" if window_s < 1.0 else "sustained"
    peak_tf = peaks.get("bf16_tflops" if regime == "burst" else "bf16_tflops_sustained")
    peak_src = f"measured (MEASURED_PEAKS.json {'bf16_tflops' if regime == 'burst' else 'bf16_tflops_sustained'})"
    if peak_tf is None:
        peak_tf, peak_src = (1650.0 if regime == "burst" else 1400.0), f"fallback (B200_PROFILING.md {regime})"
    achieved_tf = gemm_flops / (gemm_ms * 1e-3) / 1e12
    off = counts.copy()
    np.fill_diagonal(off, 0)
    bw_arr = np.asarray(bws if bws is not None else [1.0] * n, dtype=float)
    tmat = off / np.minimum.outer(bw_arr, bw_arr)  # time_normalize (commsched.py:181-190); B = 1 <-> 900 GB/s
    bmax_tokens = int(max(off.sum(axis=1).max(), off.sum(axis=0).max()))
    bmax_time = float(max(tmat.sum(axis=1).max(), tmat.sum(axis=0).max()))
    row_bytes = cfg.hidden * 2
    bound_us = bmax_time * row_bytes / (NVLINK_GBS * 1e9) * 1e6
    # loopback (all ranks on one GPU): every moved row is read and written once in this GPU's HBM
    peak_hbm = None
    try:
        peak_hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs")
    except Exception:
        pass
    peak_hbm = float(peak_hbm or 6650.0)  # fallback: B200_PROFILING.md
    moved_rows = float(counts.sum())
    loopback_floor_us = 2 * moved_rows * row_bytes / (peak_hbm * 1e9) * 1e6
    nph = int(layer.sched_i[0].item())
    line = {
        "metric": METRIC, "value": cfg.tokens / (ms_per_step * 1e-3), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": workload(args),
        "stage_ms_serial": stage_ms, "serial_ms_per_step": serial_ms,
        "sustained": dict(sustained, note="60 further back-to-back steps after the timed ones; the power "
                                           "limiter settles within ~20 steps (diagnostic, not the headline)"),
        "combine_fused": None if fused_ms is None else {
            "experts_plus_combine_ms": fused_ms["experts"] + fused_ms["combine"],
            "vs_engine_ms": stage_ms["experts"] + stage_ms["combine"],
            "wait_ms": fused_ms["combine"],
            "note": "the layer's default: the expert stage's last kernel (GEMM2's epilogue; the pre-reduction "
                    "when a rank hosts several experts) stores every row straight into its sender's return "
                    "buffer (peer memory) and its last CTA signals the senders; the engine rows above time the "
                    "reversed-schedule combine all-to-all (AURORA_COMBINE=engine)"},
        "overlap": ("K2 (on-device schedule) and the dispatch engine run concurrently: the engine is a programmatic "
                    "dependent launch of K2 and executes phase k as soon as K2 publishes it"
                    if layer.stream_schedule and not layer.overlap else f"AURORA_OVERLAP={layer.overlap}"),
        "engine": {"copy": "lsu" if layer.engine_lsu else "tma", "ctas_per_rank": layer.engine_ctas(False),
                   "cta_split": ["even", "volume", "bandwidth"][layer.split], "early_pace": bool(layer.early_pace)},
        "all_to_all": {
            "dispatch_us": stage_ms["dispatch"] * 1e3, "combine_us": stage_ms["combine"] * 1e3,
            "schedule_us": stage_ms["schedule"] * 1e3,
            "schedule_plus_dispatch_us": sched_dispatch_us,
            "schedule_plus_dispatch_note": "K2 and the dispatch engine overlapped as in the layer (PDL launch, "
                                           "engine follows K2's progress word); serial sum = schedule_us + dispatch_us",
            "unscheduled_dispatch_us": unpaced_ms["dispatch"] * 1e3,
            "unscheduled_combine_us": unpaced_ms["combine"] * 1e3,
            "baseline_schedules_on_engine": baseline_sched,
            "unscheduled_library": library_a2a,
            "bound_us_per_direction": bound_us, "b_max_tokens": bmax_tokens, "phases": nph,
            "loopback_hbm_floor_us": loopback_floor_us if world == 1 else None,
            "traffic_matrix": counts.tolist(),
            "ratio_dispatch_to_bound": (stage_ms["dispatch"] * 1e3) / bound_us if bound_us else None,
            # the bottleneck rank's traffic (b_max) over the measured time: comparable with the
            # 900 GB/s per direction per GPU the bound assumes
            "bottleneck_gbs_dispatch": bmax_tokens * row_bytes / (stage_ms["dispatch"] * 1e-3) / 1e9,
            "bottleneck_gbs_combine": bmax_tokens * row_bytes / (stage_ms["combine"] * 1e-3) / 1e9,
            "bound_basis": "max row / column sum of d_ij / min(B_i, B_j) (commsched.py:181-195; tokens when B = 1) "
                           "x hidden x 2 B / 900 GB/s NVLink per direction (the paper's big switch)",
            "transport": ("CUDA IPC between processes sharing one GPU (AURORA_BENCH_SAME_GPU=1: not NVLink)"
                          if same_gpu else "NVSwitch peer stores (CUDA IPC mappings of the peers' HBM)")
                         if world > 1 else
                         "loopback: all 8 ranks on one GPU, peer stores land in local HBM (not NVLink)",
        },
        "roofline": {"bound": "tensor", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": achieved_tf / peak_tf, "traffic": gemm_traffic(args),
                     "traffic_source": "not measured in this run: dram__bytes_read.sum + dram__bytes_write.sum of "
                                       "both GEMM launches from the committed ncu --set full capture ("
                                       + GEMM_CAPTURE + ", C2)",
                     "kernel": "aurora grouped_gemm_2sm_kernel x2 (GEMM1 + SwiGLU, GEMM2 + fused combine), "
                     "FLOPs = sum over (token, expert) rows of 2 * 3 * H * F",
                     "timing": "CUDA events on the layer's stream around the two GEMM launches inside every timed "
                               "step (mean over the timed steps)",
                     "gemm_ms_per_step": gemm_ms, "gemm_share_of_step": gemm_ms / ms_per_step,
                     "regime": regime, "peak_source": peak_src,
                     "frac_of_sustained": achieved_tf / float(peaks.get("bf16_tflops_sustained") or 1400.0),
                     "flops_per_step": gemm_flops},
        # route, pack, K2, engine, 2 GEMM, engine, aggregate (+ sort x3, gather, reduce with G > 1;
        # + local engine / GEMM pair when overlapped)
        "gpu_launches": layer.kernels_per_step() * args.steps,
        "e2e": {"value": cfg.tokens / (e2e_ms * 1e-3), "unit": "tokens/s",
                "h2d_bytes_per_step": int(xh[0].numel() * 2), "d2h_bytes_per_step": int(outh[0].numel() * 2),
                "ms_per_step": e2e_ms, "path": "AuroraMoELayer.__call__ on pinned host buffers",
                "pipeline": "H2D of step i+1 and D2H of step i-1 on copy-engine streams overlap step i "
                            "(double-buffered input/output)"},
        "clocks": clocks.summary(local_rank),
        "timeline_ms": layer.timeline(x),
    }
    if args.config == "c4" and world == 1:
        line["placement"] = placement_effect(layer, cfg, plan, bws, x, stream, args.steps)
    if args.config == "c2" and world == 1:
        line["arrival_driven_gemm"] = n1_effect(layer, x, stream, args.steps)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        weights = cpu_weights(args)
        tps, sec, cores = run_cpu(args, 256, 3, weights=weights)
        line["cpu_baseline"] = {
            "value": tps, "unit": "tokens/s", "cores": cores, "cpu_count": os.cpu_count(), "affinity": host_cores(),
            "kind": "port",
            "sample": "256 tokens of the layer per rep, median of 3: oracle router + traffic matrix, the schedule by "
                      "moeplan.build_schedule (baseline/_ref), fp32 numpy SwiGLU experts + aggregation",
            "schedule": reference_schedule_timing(counts, list(bws) if bws is not None else None),
            "schedule_impl": ("reference: moeplan.build_schedule from baseline/_ref"
                              if reference_package() is not None else "port")}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
