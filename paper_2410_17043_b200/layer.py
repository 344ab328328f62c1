"""The Aurora MoE layer on B200: router -> on-device schedule -> scheduled
NVSwitch dispatch -> tcgen05 experts -> reversed-schedule combine -> aggregate.

This is the execution the reference only simulates: ``simulate_exclusive``
(reference ``pkg/src/moeplan/sim.py:130-154``) models a layer as gate ->
all-to-all (``build_schedule``) -> FFN -> reversed all-to-all -> aggregation
behind barriers. Here every stage is a CUDA kernel from libaurora_b200.so and
the host never waits on the device inside :meth:`AuroraMoELayer.forward`.

Ranks and devices. The layer has ``n`` expert-parallel ranks (one expert per
rank, experts placed by a ``DeploymentPlan``: ``assignment_a[e]`` = rank of
expert e, reference core.py:253-304). A process drives ``n_local`` of them on
its GPU; with one process per GPU and ``n_local == 1`` the peer buffers are
CUDA-IPC mappings of the other GPUs' HBM and the engine's stores cross
NVSwitch. With fewer GPUs than ranks the remaining ranks share a GPU
("loopback"): identical kernels, identical tables, peer pointers that
happen to be local.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .core import DeploymentPlan

__all__ = ["MoEConfig", "AuroraMoELayer", "zipf_bias", "interleave_gate_up"]

PROGRESS_DONE = 1 << 20  # AURORA_PROGRESS_DONE (include/aurora_b200.h)


@dataclass(frozen=True)
class MoEConfig:
    """Shapes of one MoE layer."""

    hidden: int
    ffn: int
    experts: int
    top_k: int
    tokens: int          # global tokens T per layer call (T / ranks per rank)
    ranks: int           # expert-parallel ranks n
    skew: float = 1.0    # Zipf exponent of the router bias
    seed: int = 0

    @property
    def tokens_per_rank(self) -> int:
        return self.tokens // self.ranks

    def validate(self) -> None:
        if self.tokens % self.ranks or self.tokens_per_rank % 64:
            raise ValueError("tokens per rank must be a multiple of 64")
        if self.hidden % 256 or self.ffn % 128 or (2 * self.ffn) % 256:
            raise ValueError("hidden must be a multiple of 256 and ffn of 128")
        if self.experts % self.ranks or self.experts > 64:
            raise ValueError("experts must be a multiple of ranks (contiguous expert blocks per rank), <= 64")
        if not (1 <= self.top_k <= min(8, self.experts)):
            raise ValueError("top_k out of range")
        if not 1 <= self.ranks <= 32:
            raise ValueError("ranks must be 1..32 (the device scheduler keeps one matrix row per lane)")


def zipf_bias(experts: int, skew: float, gen: torch.Generator) -> torch.Tensor:
    """Router bias b_e = -s ln(rank_e + 1), rank = random permutation: the
    popularity law of workload.py:49-52 (1/(rank+1)^s) in logit space."""
    rank = torch.randperm(experts, generator=gen)
    return (-skew * torch.log(rank.double() + 1.0)).float()


def interleave_gate_up(w1: torch.Tensor, w3: torch.Tensor) -> torch.Tensor:
    """[G,F,H] gate and up projections -> [G,2F,H] in 128-row blocks
    (gate block b, up block b, ...), the layout the SwiGLU epilogue reads."""
    G, F, H = w1.shape
    return torch.stack([w1.view(G, F // 128, 128, H), w3.view(G, F // 128, 128, H)], dim=2).reshape(G, 2 * F, H)


class AuroraMoELayer:
    """One MoE layer, expert-parallel over ``cfg.ranks`` ranks.

    ``rank_base``/``n_local`` select the ranks this process drives
    (default: all of them, on the current device). ``peer_bufs`` is filled
    by :mod:`paper_2410_17043_b200.dist` for multi-GPU runs.
    """

    SCATTER_MAX_RANKS = 16  # gemm2sm.cu SC_MAXN

    def __init__(self, cfg: MoEConfig, plan: Optional[DeploymentPlan] = None, *, rank_base: int = 0,
                 n_local: Optional[int] = None, bandwidths=None, device=None, ctas_per_rank: Optional[int] = None,
                 weights: Optional[dict] = None, spin_limit: int = 1 << 26, gpu_of_expert=None,
                 compute_scales=None):
        cfg.validate()
        self.cfg = cfg
        self.L = _lib.load()
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        n = cfg.ranks
        self.n = n
        self.rank_base = rank_base
        self.n_local = n if n_local is None else n_local
        # experts per rank: 1 = the reference's exclusive deployment (DeploymentPlan,
        # core.py:253-304); > 1 = contiguous expert blocks e // G
        self.G = cfg.experts // n
        if gpu_of_expert is not None:  # explicit placement (e.g. a colocation plan, colocation.py)
            gpu_of = [int(g) for g in gpu_of_expert]
            if len(gpu_of) != cfg.experts or sorted(gpu_of) != sorted(r for r in range(n) for _ in range(self.G)):
                raise ValueError(f"gpu_of_expert must place exactly {self.G} expert(s) on each of {n} ranks")
            self.plan = DeploymentPlan(tuple(gpu_of)) if self.G == 1 else None
        elif self.G == 1:
            self.plan = plan if plan is not None else DeploymentPlan.identity(n)
            if self.plan.n != cfg.experts:
                raise ValueError("plan must cover every expert")
            gpu_of = list(self.plan.assignment_a)
        else:
            if plan is not None:
                raise ValueError("a DeploymentPlan places one expert per GPU; with several experts per "
                                 "rank pass gpu_of_expert (default: contiguous blocks)")
            self.plan = None
            gpu_of = [e // self.G for e in range(cfg.experts)]
        self.gpu_of = gpu_of
        sms = torch.cuda.get_device_properties(self.dev).multi_processor_count
        self.num_sms = sms
        # copy CTAs per rank: as many as stay co-resident (four TMA-engine CTAs per SM; the
        # engine clamps to its occupancy limit), capped at 96. Measured in loopback (C2, paced
        # dispatch): 16 / 24 / 32 / 37 / 55 / 74 CTAs per rank -> 336 / 253 / 217 / 204 / 170 /
        # 155 us (profiles/r01_engine_sweep.json)
        self.C = ctas_per_rank or max(1, min(96, (4 * sms) // self.n_local))
        self.spin_limit = spin_limit
        H, F, E, k = cfg.hidden, cfg.ffn, cfg.experts, cfg.top_k
        Tr = cfg.tokens_per_rank
        self.T_local = Tr * self.n_local
        dev = self.dev
        i32 = dict(dtype=torch.int32, device=dev)
        bf = dict(dtype=torch.bfloat16, device=dev)

        # ---- parameters (synthetic, seeded; experts hosted here only)
        if weights is None:
            weights = self.synthetic_weights(cfg, dev, [e for r in self.local_ranks for e in self.experts_of_rank(r)])
        self.w_gate = weights["w_gate"].to(dev, torch.bfloat16).contiguous()
        # the router's copy of the gate: fp32 (exact) in its shared-memory order, prepared once
        nf = self.L.aurora_route_gate_floats(cfg.experts, cfg.hidden)
        if nf < 0:
            raise ValueError(f"router: unsupported experts={cfg.experts} / hidden={cfg.hidden}")
        self.gate_prep = torch.empty(nf, dtype=torch.float32, device=dev)
        _lib.check(self.L.aurora_route_prepare_gate(self.w_gate.data_ptr(), cfg.experts, cfg.hidden,
                                                    self.gate_prep.data_ptr(), _lib.stream_ptr()),
                   "aurora_route_prepare_gate")
        self.bias = weights["bias"].to(dev, torch.float32).contiguous()
        self.w13 = weights["w13"].to(dev, torch.bfloat16).contiguous()   # [n_local, 2F, H] interleaved
        self.w2 = weights["w2"].to(dev, torch.bfloat16).contiguous()     # [n_local, H, F]
        self.gpu_of_expert = torch.tensor(gpu_of, **i32)
        self.local_of_expert = torch.tensor([self.experts_of_rank(g).index(e) for e, g in enumerate(gpu_of)], **i32)
        self.bw = None if bandwidths is None else torch.tensor(np.asarray(bandwidths, float), dtype=torch.float64,
                                                               device=dev)
        # emulated per-rank compute (C4: ClusterSpec.compute_scale, reference core.py:135-191): the
        # expert GEMMs' CTA pairs are split among the local ranks in proportion, each rank's tiles run
        # on its own share only (aurora_expert_ffn*'s cluster_part); pairs past the last share idle
        self.compute_scales = None if compute_scales is None else [float(c) for c in compute_scales]
        self.gemm_part = None
        if self.compute_scales is not None:
            if len(self.compute_scales) != n or min(self.compute_scales) <= 0:
                raise ValueError("compute_scales: one positive value per rank")
            # relative speeds must hold across processes too (one rank per GPU at N = 8): the process
            # whose ranks have the largest scale sum uses every CTA pair, the others leave pairs idle
            if n % self.n_local:
                raise ValueError("compute_scales: ranks must split evenly over the processes")
            sums = [sum(self.compute_scales[p:p + self.n_local]) for p in range(0, n, self.n_local)]
            mine = sum(self.compute_scales[r] for r in self.local_ranks)
            usable = max(self.n_local, min(sms // 2, int(round(sms // 2 * mine / max(sums)))))
            part = self.cluster_partition([self.compute_scales[r] for r in self.local_ranks], usable)
            self.gemm_part = torch.tensor(part, dtype=torch.int32, device=dev)

        # ---- routing / permutation state
        self.topk_idx = torch.empty(self.T_local, k, **i32)
        self.topk_w = torch.empty(self.T_local, k, dtype=torch.float32, device=dev)
        self.slot_dst = torch.empty(self.T_local, k, **i32)
        self.blk_cnt = torch.empty(self.T_local // 64, n, **i32)
        # traffic matrix, double-buffered by exchange step parity (aurora_exchange_counts): a peer
        # one step ahead writes its rows into the other buffer
        self.counts2 = torch.zeros(2, n, n, **i32)
        self.counts = self.counts2[0]
        self.xflag = torch.zeros(n, **i32)    # peer-visible: epoch of the last row received per rank
        self.xepoch = torch.zeros(1, **i32)   # exchange calls made (device side)
        self._xstep = 0
        self.send_list = torch.empty(self.n_local, Tr * k, **i32)
        self.pos = torch.empty(self.T_local, k, **i32)
        # E > 8: router logits workspace (the (tile, 8-expert pass) units run on a balanced grid)
        self.logits = (torch.empty(self.T_local, cfg.experts, dtype=torch.float32, device=dev)
                       if cfg.experts > 8 else None)
        # E > 8: the gate's contraction on the tensor cores, the deciding logits recomputed exactly
        # (aurora_route_tc; AURORA_ROUTER=fma selects the FMA router)
        self.router_tc = (self.logits is not None and os.environ.get("AURORA_ROUTER", "tc") != "fma"
                          and cfg.hidden <= 8192)
        if self.router_tc:
            nb = self.L.aurora_route_tc_bytes(cfg.experts, cfg.hidden)
            self.gate_tc = torch.empty(nb, dtype=torch.uint8, device=dev)
            _lib.check(self.L.aurora_route_prepare_gate_tc(self.w_gate.data_ptr(), cfg.experts, cfg.hidden,
                                                           self.gate_tc.data_ptr(), _lib.stream_ptr()),
                       "aurora_route_prepare_gate_tc")
            self.la_buf = torch.empty(self.T_local, 256, dtype=torch.bfloat16, device=dev)
            self.t_rows = torch.zeros(1, dtype=torch.int32, device=dev)  # GEMM row count (set by the call)
            self.n_fallback = torch.zeros(1, dtype=torch.int32, device=dev)  # uncertified tokens, cumulative

        # ---- schedule tables (written by K2 on the device)
        P = self.L.aurora_phase_cap(n)
        self.P = P
        self.phase_recv = torch.empty(P, n, **i32)
        self.phase_dur = torch.empty(P, dtype=torch.float64, device=dev)
        self.sched_i = torch.zeros(2, **i32)          # n_phases, status
        self.chunks = torch.empty(P, n, 4, **i32)
        self.rchunks = torch.empty(P, n, 4, **i32)
        self.n_in = torch.empty(n, **i32)
        self.n_out = torch.empty(n, **i32)
        # K2's progress word: phases whose engine entries are final (| DONE): the
        # dispatch starts on phase 0 while K2 is still computing later phases
        self.progress = torch.zeros(1, **i32)
        # buffer layout (written by K3 from the counts): local rows first in every receive buffer
        self.soff = torch.empty(n, n, **i32)
        self.roff = torch.empty(n, n, **i32)
        self.rtot = torch.empty(n, **i32)
        self.rloc = torch.empty(n, **i32)
        self.rrem = torch.empty(n, **i32)
        self.engine_status = torch.zeros(1, **i32)
        self.gemm_ticket = torch.zeros(1, **i32)  # fused combine: GEMM2's grid completion ticket
        # the expert GEMMs' dynamic tile order: one {next tile, clusters done} pair per stream the
        # layer launches GEMMs on (main, side), owned here -- no allocation inside a forward
        self.tile_ctrs = torch.zeros(2, 2, **i32)
        # overlap: the local rows' copy + expert GEMM run on a side stream while
        # K2 computes the schedule and the engine moves the network rows
        # Measured on B200 (profiles/r01_overlap_sweep.json): the expert GEMM runs
        # at the 1 kW power cap, so overlapping the copies only slows it, and
        # splitting it into local/network launches re-reads every expert's
        # weights. Serial is the default; the overlapped plans stay selectable.
        self.overlap = os.environ.get("AURORA_OVERLAP", "none")  # "none" | "schedule" | "full"
        if self.overlap == "none":
            self.overlap = False
        self.C_overlap = int(os.environ.get("AURORA_C_OVERLAP", "0"))  # copy CTAs/rank beside the GEMM
        self.unpaced = 0  # 16: ablation -- run the all-to-all without the schedule's pacing
        # the aggregation reads local (diagonal) rows straight from the expert output, so the
        # combine only moves rows that cross the network
        self.local_direct = os.environ.get("AURORA_LOCAL_DIRECT", "1") != "0"
        # the combine fused into GEMM2's epilogue (one expert per rank): output rows are stored
        # straight into their senders' return buffers while the GEMM runs, so no combine
        # all-to-all follows the experts; AURORA_COMBINE=engine runs the reversed-schedule
        # combine engine instead (needs local-direct aggregation either way)
        self.fused_combine = os.environ.get("AURORA_COMBINE", "fused") == "fused"
        # several experts per rank: dispatch rows straight into the packed per-expert groups
        # (engine mode bit 8; AURORA_GROUPED_DISPATCH=0: receive, sort, gather)
        self.grouped_dispatch = os.environ.get("AURORA_GROUPED_DISPATCH", "1") != "0"
        # grouped: finish single-expert rows in GEMM2's epilogue (per-row scattered stores)
        # instead of TMA-storing every row for the pre-reduction (AURORA_PACKED_SCATTER=0)
        self.packed_scatter = os.environ.get("AURORA_PACKED_SCATTER", "1") != "0"
        # the single-CTA GEMM (ablation; gemm.cu selects it for any AURORA_GEMM starting with '1') has no
        # scatter epilogue, and the pair kernel's scatter tables stop at 16 ranks (gemm2sm.cu SC_MAXN):
        # beyond that the combine runs on the reversed-schedule engine (up to 32 ranks)
        if os.environ.get("AURORA_GEMM", "").startswith("1") or n > self.SCATTER_MAX_RANKS:
            self.fused_combine = False
            self.packed_scatter = False
        # the engine's copy path: TMA bulk copies (default) or LSU 16-byte vectors (ablation)
        self.engine_lsu = 64 if os.environ.get("AURORA_ENGINE", "tma") == "lsu" else 0
        # TMA engine: release a receiver when a run has ~a flag round trip of rows left (mode bit 7)
        self.early_pace = 128 if os.environ.get("AURORA_EARLY_PACE", "1") != "0" else 0
        # deadline pacing: a run also starts when the schedule's clock (phase durations at this
        # link rate, GB/s per pair) reaches its phase, so a late hand-over flag no longer delays
        # the chain; 0 = flags only (AURORA_DEADLINE_GBPS)
        self.deadline_gbps = float(os.environ.get("AURORA_DEADLINE_GBPS", "0"))
        # how a process's copy CTAs are split among the ranks it drives (csrc/apportion.cuh):
        # by bandwidth when the cluster is heterogeneous (C4: a rank's copy rate follows its
        # bandwidth), else by volume (one rank per GPU: identity; loopback: the hot rank gets the
        # copy capacity its own GPU would have); AURORA_CTA_SPLIT=even|volume|bandwidth overrides
        split = os.environ.get("AURORA_CTA_SPLIT", "bandwidth" if bandwidths is not None else "volume")
        self.split = {"even": 0, "volume": 1, "bandwidth": 2}[split]
        self.trace = None
        self.side = torch.cuda.Stream(device=dev)
        self._ev_pack = torch.cuda.Event()
        self._ev_local = torch.cuda.Event()
        # the dispatch engine is a programmatic dependent launch of K2 and consumes
        # its phases while K2 computes the later ones (AURORA_STREAM_SCHEDULE=0:
        # K2, then the dispatch)
        self.stream_schedule = os.environ.get("AURORA_STREAM_SCHEDULE", "1") != "0"

        # ---- data buffers. A rank can receive at most every token once.
        self.cap = cfg.tokens
        self.recv = torch.empty(self.n_local * self.cap, H, **bf)
        self.hbuf = torch.empty(self.n_local * self.cap, F, **bf)
        self.ybuf = torch.empty(self.n_local * self.cap, H, **bf)
        self.ret_stride = Tr * k
        self.ret = torch.empty(self.n_local * self.ret_stride, H, **bf)
        self.out = torch.empty(self.T_local, H, **bf)
        # per rank {pace, done} arrival counters (peer-visible): pace paces run starts, done
        # counts runs whose stores have completed (the engine's exit condition)
        self.ctr_d = torch.zeros(n, 2, **i32)
        self.ctr_c = torch.zeros(n, 2, **i32)
        # several experts per rank: per-row expert metadata travels with the rows, the rows
        # are grouped by local expert for the GEMM and pre-reduced before the combine
        self.meta_bytes = ((k * 8 + 15) // 16) * 16
        if self.G > 1:
            E_loc = self.n_local * self.G
            self.meta_send = torch.zeros(self.n_local * Tr * k, self.meta_bytes, dtype=torch.uint8, device=dev)
            self.meta_recv = torch.zeros(self.n_local * self.cap, self.meta_bytes, dtype=torch.uint8, device=dev)
            self.max_entries = cfg.tokens * k  # every (token, expert) pair at most once
            self.g_off = torch.zeros(E_loc + 1, **i32)
            self.g_rows = torch.zeros(E_loc, **i32)
            self.g_src = torch.zeros(self.max_entries, **i32)
            self.inv = torch.empty(self.n_local * self.cap * k, **i32)
            blocks = (self.n_local * self.cap + 255) // 256
            self.sort_scratch = torch.empty(blocks * E_loc, **i32)
            self.a_g = torch.empty(self.max_entries, H, **bf)
            # grouped dispatch (default): rows land straight at their packed-group positions
            self.blk_cnt_e = torch.zeros(self.T_local // 64, E, **i32)
            self.cnt_e2 = torch.zeros(2, n, E, **i32)   # tokens per (sender rank, expert), parity-buffered
            self.cnt_e = self.cnt_e2[0]
            # per packed row {receiver-layout row, weight, single, 0} (grouped dispatch): rows with
            # one local expert are finished in GEMM2's epilogue instead of the pre-reduction
            self.ginfo = torch.zeros(self.max_entries, 4, **i32)
            self.h_g = torch.empty(self.max_entries, F, **bf)
            self.y_g = torch.empty(self.max_entries, H, **bf)
            self.overlap = False  # the local/network GEMM split assumes one expert per rank
        else:
            self.meta_send = self.meta_recv = None
        # arrival-driven expert GEMM (N1, one expert per rank): landed[g][i] = rows of block
        # (sender i -> local rank g) the dispatch has made visible; GEMM1 runs beside the dispatch
        # (an LSU copy engine, one CTA per SM, leaves the SMs' shared memory to the GEMM) and
        # starts each tile once its rows have landed. AURORA_N1=1 turns it on.
        self.landed = torch.zeros(self.n_local, n, **i32) if self.G == 1 else None
        self.arrival = os.environ.get("AURORA_N1", "0") == "1"
        self.nvtx = os.environ.get("AURORA_NVTX", "0") == "1"
        self.x = None
        self._tables_for(None)

    # ------------------------------------------------------------ helpers
    @property
    def local_ranks(self):
        return list(range(self.rank_base, self.rank_base + self.n_local))

    def expert_of_rank(self, r: int) -> int:
        """The single expert on rank r (exclusive deployment)."""
        return self.gpu_of.index(r)

    def experts_of_rank(self, r: int) -> list:
        """Experts hosted by rank r, in local-index order."""
        return [e for e, g in enumerate(self.gpu_of) if g == r]

    @staticmethod
    def synthetic_weights(cfg: MoEConfig, dev, experts) -> dict:
        """Seeded random-init parameters: W_g ~ N(0, 1/H), Zipf bias, expert
        weights N(0, 1/fan_in); generated per expert so any
        rank subset reproduces the same model."""
        H, F, E = cfg.hidden, cfg.ffn, cfg.experts
        g = torch.Generator(device="cpu").manual_seed(cfg.seed)
        w_gate = (torch.randn(E, H, generator=g) / math.sqrt(H)).to(torch.bfloat16)
        bias = zipf_bias(E, cfg.skew, g)
        w13, w2 = [], []
        for e in experts:
            ge = torch.Generator(device=dev).manual_seed(cfg.seed * 1000003 + 17 * e + 1)
            w1 = (torch.randn(1, F, H, generator=ge, device=dev) / math.sqrt(H)).to(torch.bfloat16)
            w3 = (torch.randn(1, F, H, generator=ge, device=dev) / math.sqrt(H)).to(torch.bfloat16)
            w13.append(interleave_gate_up(w1, w3)[0])
            w2.append((torch.randn(H, F, generator=ge, device=dev) / math.sqrt(F)).to(torch.bfloat16))
        return {"w_gate": w_gate, "bias": bias, "w13": torch.stack(w13), "w2": torch.stack(w2)}

    @staticmethod
    def cluster_partition(scales, clusters: int) -> list:
        """Prefix of CTA-pair counts per rank proportional to ``scales`` (largest
        remainder, at least one each): rank r's GEMM tiles run on clusters
        [part[r], part[r + 1])."""
        w = np.asarray(scales, dtype=float)
        if clusters < len(w):
            raise ValueError("fewer GEMM clusters than ranks")
        quota = w / w.sum() * (clusters - len(w))
        base = np.floor(quota).astype(int) + 1
        rest = clusters - int(base.sum())
        order = np.argsort(-(quota - np.floor(quota)), kind="stable")
        base[order[:rest]] += 1
        return [0] + np.cumsum(base).tolist()

    def _ptr_table(self, ptrs) -> torch.Tensor:
        return torch.tensor([int(p) for p in ptrs], dtype=torch.int64, device=self.dev)

    def _tables_for(self, x: Optional[torch.Tensor], peers: Optional[dict] = None) -> None:
        """Device pointer tables for the engine. ``peers`` (multi-GPU) maps
        buffer name -> list of n peer addresses; loopback uses local slices."""
        H = self.cfg.hidden
        esz = 2
        Tr = self.cfg.tokens_per_rank
        if peers is None:
            recv_p = [self.recv.data_ptr() + r * self.cap * H * esz for r in range(self.n)]
            ret_p = [self.ret.data_ptr() + r * self.ret_stride * H * esz for r in range(self.n)]
            ctr_d = [self.ctr_d.data_ptr() + 8 * r for r in range(self.n)]
            ctr_c = [self.ctr_c.data_ptr() + 8 * r for r in range(self.n)]
        else:
            recv_p, ret_p, ctr_d, ctr_c = peers["recv"], peers["ret"], peers["ctr_d"], peers["ctr_c"]
            self.t_counts2 = self._ptr_table(peers["counts2"])
            self.t_xflag = self._ptr_table(peers["xflag"])
        if self.landed is not None:  # receiver j's row of arrival credits
            self.t_landed = self._ptr_table(peers["landed"] if peers is not None else
                                            [self.landed.data_ptr() + (j - self.rank_base) * self.n * 4
                                             if self.rank_base <= j < self.rank_base + self.n_local else 0
                                             for j in range(self.n)])
        self.t_dst_d = self._ptr_table(recv_p)
        self.t_dst_c = self._ptr_table(ret_p)
        self.t_ctr_d = self._ptr_table(ctr_d)
        self.t_ctr_c = self._ptr_table(ctr_c)
        self.t_src_c = self._ptr_table([self.ybuf.data_ptr() + r * self.cap * H * esz for r in range(self.n_local)])
        if self.G > 1:  # second plane: expert metadata beside every dispatched row
            mb, k = self.meta_bytes, self.cfg.top_k
            self.t_src2 = self._ptr_table([self.meta_send.data_ptr() + r * Tr * k * mb for r in range(self.n_local)])
            meta_p = (peers["meta_recv"] if peers is not None else
                      [self.meta_recv.data_ptr() + r * self.cap * mb for r in range(self.n)])
            self.t_dst2 = self._ptr_table(meta_p)
            # grouped dispatch: every rank's rows go to its process's packed group buffer
            ag_p = peers["a_g"] if peers is not None else [self.a_g.data_ptr()] * self.n
            self.t_dst_g = self._ptr_table(ag_p)
            self.t_ginfo = self._ptr_table(peers["ginfo"] if peers is not None else [self.ginfo.data_ptr()] * self.n)
            if peers is not None:
                self.t_cnt_e2 = self._ptr_table(peers["cnt_e2"])
        self._src_tables = {}
        if x is not None:
            self._use_input(x)

    def _use_input(self, x: torch.Tensor) -> None:
        """Point the dispatch at ``x``. Tables are cached per input address, so
        alternating between a few (e.g. double-buffered) inputs never builds a
        table -- a host->device copy -- inside the forward."""
        key = x.data_ptr()
        t = self._src_tables.get(key)
        if t is None:
            Tr, H = self.cfg.tokens_per_rank, self.cfg.hidden
            t = self._ptr_table([key + r * Tr * H * 2 for r in range(self.n_local)])
            if len(self._src_tables) >= 8:
                self._src_tables.clear()
            self._src_tables[key] = t
        self.t_src_d = t
        self.x = x

    # ------------------------------------------------------------ stages
    def route(self, x: torch.Tensor, stream: int) -> None:
        cfg = self.cfg
        self.counts = self.counts2[self._xstep & 1]
        # only this process's rows: a peer may already have stored its rows for this step
        self.counts[self.rank_base:self.rank_base + self.n_local].zero_()
        if self.router_tc:
            _lib.check(self.L.aurora_route_tc(x.data_ptr(), self.w_gate.data_ptr(), self.gate_tc.data_ptr(),
                                              self.bias.data_ptr(), self.T_local, cfg.hidden, cfg.experts,
                                              cfg.top_k, self.gpu_of_expert.data_ptr(), self.n, self.rank_base,
                                              cfg.tokens_per_rank, self.topk_idx.data_ptr(), self.topk_w.data_ptr(),
                                              self.slot_dst.data_ptr(), self.blk_cnt.data_ptr(),
                                              self.counts.data_ptr(), self.logits.data_ptr(), self.la_buf.data_ptr(),
                                              self.t_rows.data_ptr(), None, self.n_fallback.data_ptr(), stream),
                       "aurora_route_tc")
        else:
            _lib.check(self.L.aurora_route(x.data_ptr(), self.gate_prep.data_ptr(), self.bias.data_ptr(),
                                           self.T_local, cfg.hidden, cfg.experts, cfg.top_k,
                                           self.gpu_of_expert.data_ptr(), self.n, self.rank_base,
                                           cfg.tokens_per_rank, self.topk_idx.data_ptr(), self.topk_w.data_ptr(),
                                           self.slot_dst.data_ptr(), self.blk_cnt.data_ptr(),
                                           self.counts.data_ptr(),
                                           None if self.logits is None else self.logits.data_ptr(),
                                           stream), "aurora_route")
        if self.grouped:
            self.cnt_e = self.cnt_e2[self._xstep & 1]
            self.cnt_e[self.rank_base:self.rank_base + self.n_local].zero_()
            _lib.check(self.L.aurora_expert_hist(self.topk_idx.data_ptr(), self.T_local, cfg.top_k, cfg.experts,
                                                 self.rank_base, cfg.tokens_per_rank, self.blk_cnt_e.data_ptr(),
                                                 self.cnt_e.data_ptr(), stream), "aurora_expert_hist")

    def exchange_counts(self, stream: Optional[int] = None) -> None:
        """Multi-GPU: complete the traffic matrix (each process owns its rows) with
        peer stores + flags on the stream (aurora_exchange_counts; no NCCL, no host
        sync). Loopback: nothing to do, every row was produced here."""
        if self.n_local == self.n:
            return
        if getattr(self, "t_counts2", None) is None:
            raise RuntimeError("multi-process layer: call dist.connect_peers(layer) first")
        s = _lib.stream_ptr() if stream is None else stream
        grouped = self.grouped
        _lib.check(self.L.aurora_exchange_counts(self.counts2.data_ptr(), self.t_counts2.data_ptr(),
                                                 self.cnt_e2.data_ptr() if grouped else None,
                                                 self.t_cnt_e2.data_ptr() if grouped else None,
                                                 self.cfg.experts, self.xflag.data_ptr(), self.t_xflag.data_ptr(),
                                                 self.xepoch.data_ptr(), self.n, self.rank_base, self.n_local,
                                                 self.spin_limit, self.engine_status.data_ptr(), s),
                   "aurora_exchange_counts")
        self._xstep += 1

    def engine_ctas(self, combine: bool, C: Optional[int] = None) -> int:
        """Copy CTAs per local rank the engine launches (clamped to co-residency)."""
        row2 = self.meta_bytes if (self.G > 1 and not combine) else 0
        lsu = self.engine_lsu
        if not combine and C is None:
            lsu, C = self.dispatch_engine()
        c = self.L.aurora_engine_ctas(self.n, self.n_local, C or self.C, self.cfg.hidden * 2, row2,
                                      1 if lsu else 0)
        if c < 1:
            _lib.check(-c, "aurora_engine_ctas")
        return c

    def cta_split(self, combine: bool) -> list:
        """Copy CTAs of every rank (host mirror of the device apportioning)."""
        from .apportion import apportion
        bw = None if self.bw is None else self.bw.cpu().numpy()
        return apportion(self.counts.cpu().numpy(), self.n, self.n_local, self.n_local * self.engine_ctas(combine),
                         self.split, combine, bw)

    def schedule(self, stream: int, dispatch_ctas: Optional[int] = None) -> None:
        """K2. ``dispatch_ctas``: copy CTAs per rank the dispatch will run with when it
        differs from ``self.C`` (the combine always runs with ``self.C``); the hand-over
        thresholds count one signal per copy CTA, so K2 and the engine must agree."""
        _lib.check(self.L.aurora_schedule_counts(
            self.counts.data_ptr(), None if self.bw is None else self.bw.data_ptr(), self.n,
            self.phase_recv.data_ptr(), self.phase_dur.data_ptr(), self.sched_i.data_ptr(),
            self.chunks.data_ptr(), self.rchunks.data_ptr(), self.n_in.data_ptr(), self.n_out.data_ptr(),
            self.sched_i[1:].data_ptr(), self.progress.data_ptr(), self.n_local,
            self.n_local * self.engine_ctas(False, dispatch_ctas), self.n_local * self.engine_ctas(True), self.split,
            stream),
            "aurora_schedule_counts")

    def pack(self, stream: int) -> None:
        cfg = self.cfg
        if self.grouped:
            _lib.check(self.L.aurora_pack_grouped(
                self.slot_dst.data_ptr(), self.blk_cnt.data_ptr(), self.counts.data_ptr(), self.T_local, cfg.top_k,
                self.n, self.rank_base, cfg.tokens_per_rank, self.send_list.data_ptr(), self.pos.data_ptr(),
                self.soff.data_ptr(), self.roff.data_ptr(), self.rtot.data_ptr(), self.rloc.data_ptr(),
                self.rrem.data_ptr(), self.topk_idx.data_ptr(), self.topk_w.data_ptr(),
                self.local_of_expert.data_ptr(), self.meta_send.data_ptr(), self.blk_cnt_e.data_ptr(),
                self.cnt_e.data_ptr(), self.gpu_of_expert.data_ptr(), cfg.experts, self.G, self.n_local,
                self.g_off.data_ptr(), self.g_rows.data_ptr(), self.t_ginfo.data_ptr(), stream),
                "aurora_pack_grouped")
            return
        _lib.check(self.L.aurora_pack(self.slot_dst.data_ptr(), self.blk_cnt.data_ptr(), self.counts.data_ptr(),
                                      self.T_local, cfg.top_k, self.n, self.rank_base, cfg.tokens_per_rank,
                                      self.send_list.data_ptr(), self.pos.data_ptr(), self.soff.data_ptr(),
                                      self.roff.data_ptr(), self.rtot.data_ptr(), self.rloc.data_ptr(),
                                      self.rrem.data_ptr(), self.topk_idx.data_ptr(), self.topk_w.data_ptr(),
                                      self.local_of_expert.data_ptr(),
                                      None if self.meta_send is None else self.meta_send.data_ptr(), stream),
                   "aurora_pack")

    # engine mode bits (include/aurora_b200.h): 1 combine, 2 system scope, 4 local only, 8 remote only
    def _engine(self, mode: int, stream: int) -> None:
        cfg = self.cfg
        combine = mode & 1
        lsu, C = (self.engine_lsu, self.C) if combine else self.dispatch_engine()
        landed = self.arrival_on and not combine
        src = self.t_src_c if combine else self.t_src_d
        dst = self.t_dst_c if combine else (self.t_dst_g if self.grouped else self.t_dst_d)
        ctr = self.t_ctr_c if combine else self.t_ctr_d
        sys_scope = 2 if self.n_local != self.n else 0  # peers on other GPUs
        plane2 = self.G > 1 and not combine
        grouped = 256 if (self.grouped and not combine) else 0
        _lib.check(self.L.aurora_engine(
            mode | sys_scope | lsu | self.early_pace | grouped, self.n, self.n_local, self.rank_base, self.counts.data_ptr(), self.chunks.data_ptr(),
            self.rchunks.data_ptr(), self.progress.data_ptr(), self.n_in.data_ptr(), self.n_out.data_ptr(),
            self.soff.data_ptr(), self.roff.data_ptr(), self.send_list.data_ptr(), self.send_list.shape[1],
            src.data_ptr(), dst.data_ptr(), cfg.hidden * 2,
            self.t_src2.data_ptr() if plane2 else None, self.t_dst2.data_ptr() if plane2 else None,
            self.meta_bytes if plane2 else 0,
            ctr.data_ptr(), C, self.P, self.spin_limit, self.engine_status.data_ptr(), self.split,
            None if self.bw is None else self.bw.data_ptr(), None,
            self.t_landed.data_ptr() if landed else None,
            self.phase_dur.data_ptr() if self.deadline_gbps > 0 else None,
            cfg.hidden * 2 / self.deadline_gbps if self.deadline_gbps > 0 else 0.0, stream),
            "aurora_engine")

    def dispatch(self, stream: int, part: str = "all", overlap_schedule: bool = False) -> None:
        """``overlap_schedule``: launched right after :meth:`schedule` on the same
        stream, start while K2 still runs (PDL) and follow its progress word."""
        self._engine({"all": 0, "local": 4, "remote": 8}[part] | self.unpaced | (32 if overlap_schedule else 0),
                     stream)

    def experts(self, stream: int, part: str = "all") -> None:
        """SwiGLU experts over this process's receive buffers: all rows, the
        local rows only (they need no schedule), or the network rows only."""
        cfg = self.cfg
        rb = self.rank_base
        if self.G > 1:
            self._experts_grouped(stream)
            return
        if part == "all":
            m_start, m_rows = 0, self.rtot[rb:].data_ptr()
        elif part == "local":
            m_start, m_rows = 0, self.rloc[rb:].data_ptr()
        else:
            m_start, m_rows = self.rloc[rb:].data_ptr(), self.rrem[rb:].data_ptr()
        _lib.check(self.L.aurora_expert_ffn(self.recv.data_ptr(), self.w13.data_ptr(), self.w2.data_ptr(),
                                            self.hbuf.data_ptr(), self.ybuf.data_ptr(), m_start or None, m_rows,
                                            self.n_local, self.cap, cfg.hidden, cfg.ffn, self._part(part),
                                            self._tctr(stream), self.num_sms, stream),
                   "aurora_expert_ffn")

    def _part(self, part: str = "all"):
        """The emulated-compute cluster partition (whole-buffer launches only)."""
        return self.gemm_part.data_ptr() if (self.gemm_part is not None and part == "all") else None

    def _tctr(self, stream: int) -> int:
        """The GEMM tile-counter pair of the stream a launch goes to."""
        return self.tile_ctrs[1 if stream == int(self.side.cuda_stream) else 0].data_ptr()

    @property
    def arrival_on(self) -> bool:
        """N1 in effect: one expert per rank, combine fused into GEMM2, K2 streamed to the dispatch."""
        return (self.arrival and self.G == 1 and self.combine_in_gemm and self.stream_schedule
                and not self.overlap and self.gemm_part is None)

    def dispatch_engine(self):
        """(LSU mode bit, copy CTAs per rank) of the dispatch: with N1 an LSU engine with one
        CTA per SM, which leaves the SMs' shared memory to the GEMM running beside it."""
        if self.arrival_on:
            return 64, max(1, (self.num_sms - 2) // self.n_local)
        return self.engine_lsu, self.C

    @property
    def grouped(self) -> bool:
        """Rows are dispatched straight into the packed per-expert groups (needs the TMA engine)."""
        return self.G > 1 and self.grouped_dispatch and not self.engine_lsu

    @property
    def combine_in_gemm(self) -> bool:
        """The combine runs inside the expert stage's last kernel (GEMM2's epilogue,
        or the pre-reduction when a rank hosts several experts); local rows are read
        in place by the aggregation."""
        return self.fused_combine and self.local_direct and not self.overlap

    def experts_combine(self, stream: int) -> None:
        """The experts with the combine fused into their last kernel: every output
        row goes straight to its sender's return buffer (peer memory), local rows
        stay in ybuf for the aggregation; see aurora_expert_ffn_combine /
        aurora_expert_reduce_combine."""
        cfg = self.cfg
        if self.G > 1:
            self._experts_grouped(stream, fused=True)
            return
        sys_scope = 1 if self.n_local != self.n else 0
        _lib.check(self.L.aurora_expert_ffn_combine(
            self.recv.data_ptr(), self.w13.data_ptr(), self.w2.data_ptr(), self.hbuf.data_ptr(),
            self.ybuf.data_ptr(), self.rtot[self.rank_base:].data_ptr(), self.n_local, self.cap, cfg.hidden,
            cfg.ffn, self.t_dst_c.data_ptr(), self.counts.data_ptr(), self.soff.data_ptr(), self.roff.data_ptr(),
            self.n, self.rank_base, self.t_ctr_c.data_ptr(), self.gemm_ticket.data_ptr(), sys_scope,
            self._part(), self.landed.data_ptr() if self.arrival_on else None, 1 if self.arrival_on else 0,
            self._tctr(stream), self.num_sms, stream), "aurora_expert_ffn_combine")

    def combine_wait(self, stream: int) -> None:
        """Receiving side of the fused combine: every expert rank's rows for this
        process's senders have landed (then the counters are re-armed)."""
        sys_scope = 1 if self.n_local != self.n else 0
        _lib.check(self.L.aurora_combine_wait(self.t_ctr_c.data_ptr(), self.rank_base, self.n_local, self.n,
                                              sys_scope, self.spin_limit, self.engine_status.data_ptr(), stream),
                   "aurora_combine_wait")

    def _experts_grouped(self, stream: int, fused: bool = False) -> None:
        """Several experts per rank: group the received rows by local expert,
        run the packed grouped GEMMs, pre-reduce each row's expert outputs."""
        cfg = self.cfg
        L, k, H = self.L, cfg.top_k, cfg.hidden
        E_loc = self.n_local * self.G
        skip = 0
        if self.grouped and not self.packed_scatter:
            _lib.check(L.aurora_expert_ffn_packed(self.a_g.data_ptr(), self.w13.data_ptr(), self.w2.data_ptr(),
                                                  self.h_g.data_ptr(), self.y_g.data_ptr(), self.g_off.data_ptr(),
                                                  self.g_rows.data_ptr(), E_loc, self.max_entries, H, cfg.ffn,
                                                  self._part(), self.G, self._tctr(stream), self.num_sms, stream),
                       "aurora_expert_ffn_packed")
            inv = None
        elif self.grouped:  # rows already sit in their groups (g_off / g_rows from the grouped pack);
            # single-expert rows are finished (w * y -> sender or ybuf) in GEMM2's epilogue
            _lib.check(L.aurora_expert_ffn_packed_scatter(
                self.a_g.data_ptr(), self.w13.data_ptr(), self.w2.data_ptr(), self.h_g.data_ptr(),
                self.y_g.data_ptr(), self.g_off.data_ptr(), self.g_rows.data_ptr(), E_loc, self.max_entries, H,
                cfg.ffn, self.ginfo.data_ptr(), self.G, self.t_dst_c.data_ptr(), self.counts.data_ptr(),
                self.soff.data_ptr(), self.roff.data_ptr(), self.n, self.rank_base, self.ybuf.data_ptr(), self.cap,
                1 if fused else 0, 1 if self.n_local != self.n else 0, self._part(), self._tctr(stream),
                self.num_sms, stream),
                "aurora_expert_ffn_packed_scatter")
            inv, skip = None, 1
        else:
            self._sort_and_gather(stream)
            inv = self.inv.data_ptr()
        if fused:
            _lib.check(L.aurora_expert_reduce_combine(
                self.y_g.data_ptr(), inv, self.meta_recv.data_ptr(), self.cap, self.meta_bytes,
                self.rtot.data_ptr(), self.n_local, self.rank_base, k, H, self.ybuf.data_ptr(),
                self.t_dst_c.data_ptr(), self.counts.data_ptr(), self.soff.data_ptr(), self.roff.data_ptr(),
                self.n, self.t_ctr_c.data_ptr(), self.gemm_ticket.data_ptr(), 1 if self.n_local != self.n else 0,
                skip, stream), "aurora_expert_reduce_combine")
            return
        _lib.check(L.aurora_expert_reduce(self.y_g.data_ptr(), inv, self.meta_recv.data_ptr(),
                                          self.cap, self.meta_bytes, self.rtot.data_ptr(), self.n_local,
                                          self.rank_base, k, H, self.ybuf.data_ptr(), skip, stream),
                   "aurora_expert_reduce")

    def _sort_and_gather(self, stream: int) -> None:
        """Ungrouped receive: sort the received rows by local expert, then gather them
        into the packed group buffer and run the packed GEMMs."""
        cfg = self.cfg
        L, k, H = self.L, cfg.top_k, cfg.hidden
        _lib.check(L.aurora_expert_sort(self.meta_recv.data_ptr(), self.cap, self.meta_bytes, self.rtot.data_ptr(),
                                        self.n_local, self.rank_base, k, self.G, self.g_off.data_ptr(),
                                        self.g_rows.data_ptr(), self.g_src.data_ptr(), self.inv.data_ptr(),
                                        self.sort_scratch.data_ptr(), self.sort_scratch.numel(), stream),
                   "aurora_expert_sort")
        E_loc = self.n_local * self.G
        _lib.check(L.aurora_gather_rows(self.recv.data_ptr(), self.a_g.data_ptr(), self.g_src.data_ptr(),
                                        self.g_off[E_loc:].data_ptr(), self.max_entries, H * 2, stream),
                   "aurora_gather_rows")
        _lib.check(L.aurora_expert_ffn_packed(self.a_g.data_ptr(), self.w13.data_ptr(), self.w2.data_ptr(),
                                              self.h_g.data_ptr(), self.y_g.data_ptr(), self.g_off.data_ptr(),
                                              self.g_rows.data_ptr(), E_loc, self.max_entries, H, cfg.ffn,
                                              self._part(), self.G, self._tctr(stream), self.num_sms, stream),
                   "aurora_expert_ffn_packed")

    def combine(self, stream: int) -> None:
        # local rows stay in the expert output; the aggregation reads them there
        self._engine(1 | (8 if self.local_direct else 0) | self.unpaced, stream)

    def aggregate(self, stream: int, out: Optional[torch.Tensor] = None) -> None:
        cfg = self.cfg
        out = self.out if out is None else out
        _lib.check(self.L.aurora_aggregate(self.ret.data_ptr(), self.ret_stride, self.soff.data_ptr(),
                                           self.pos.data_ptr(), self.slot_dst.data_ptr(), self.topk_w.data_ptr(),
                                           self.T_local, cfg.top_k, cfg.hidden, self.n, self.rank_base,
                                           cfg.tokens_per_rank, 1 if self.G > 1 else 0, out.data_ptr(),
                                           self.ybuf.data_ptr() if self.local_direct else None, self.cap,
                                           self.roff.data_ptr(), stream), "aurora_aggregate")

    # ------------------------------------------------------------ forward
    def forward(self, x: torch.Tensor, out: Optional[torch.Tensor] = None, *,
                dispatch_after: Optional[torch.cuda.Event] = None,
                dispatched: Optional[torch.cuda.Event] = None) -> torch.Tensor:
        r"""x: [tokens of the local ranks, hidden] bf16 on this GPU -> same shape,
        written to ``out`` when given (e.g. one of several pipelined output
        buffers), else to the layer's own ``self.out``.

        ``dispatch_after`` / ``dispatched``: events for running two layers on two
        streams (colocated models, :class:`~.colocation.ColocatedLayers`): the
        stream waits for ``dispatch_after`` before K2 + the dispatch, and records
        ``dispatched`` once the dispatch is launched, so the two layers' copy
        engines never run at the same time.

        Stream plan (no host synchronisation anywhere):
          route -> (counts exchange) -> pack -> K2 schedule ---------------------------+
                                                  \-> dispatch (PDL: local rows, then phase k
                                                       as soon as K2 publishes it) -> experts
          -> combine (reversed schedule) -> aggregate
        AURORA_OVERLAP=schedule|full instead runs the local rows' expert GEMM on a
        side stream beside K2 and the network dispatch (measured slower).
        """
        self._check_out(out, x)
        self.front(x)
        return self.back(out, dispatch_after=dispatch_after, dispatched=dispatched)

    def _check_out(self, out: Optional[torch.Tensor], x: Optional[torch.Tensor] = None) -> None:
        x = self.x if x is None else x
        if out is not None and (out.dtype != torch.bfloat16 or out.shape != x.shape or not out.is_contiguous()
                                or out.device != x.device):
            raise ValueError("out must be a contiguous bf16 tensor shaped like x on the same device")

    def _mark(self, k: str, st) -> None:
        tr = self.trace  # optional {point: cuda.Event} timeline (diagnostics)
        if tr and k in tr:
            tr[k].record(st)
            self._marked.add(k)
        if self.nvtx:  # host-side ranges around each stage's launches (AURORA_NVTX=1; nsys / ncu --nvtx)
            if k != "start":
                torch.cuda.nvtx.range_pop()
            if k != "end":
                torch.cuda.nvtx.range_push(self.NVTX_STAGES.get(k, "aurora: after " + k))

    def front(self, x: torch.Tensor) -> None:
        """The forward up to the permutation (router, counts exchange, pack) on the
        current stream; :meth:`back` continues it. ``forward`` = front + back."""
        if x.dtype != torch.bfloat16 or x.shape != (self.T_local, self.cfg.hidden) or not x.is_contiguous():
            raise ValueError(f"x must be contiguous bf16 [{self.T_local}, {self.cfg.hidden}]")
        if self.x is None or x.data_ptr() != self.x.data_ptr():
            self._use_input(x)
        main = torch.cuda.current_stream(self.dev)
        s = int(main.cuda_stream)
        self._marked = set()
        self._mark("start", main)
        self.route(x, s)
        self.exchange_counts(s)
        self.pack(s)
        self._mark("packed", main)

    def back(self, out: Optional[torch.Tensor] = None, *, dispatch_after: Optional[torch.cuda.Event] = None,
             dispatched: Optional[torch.cuda.Event] = None) -> torch.Tensor:
        """The forward from K2 on (schedule, dispatch, experts, combine, aggregate) on
        the current stream, after :meth:`front` of the same batch: :meth:`send` then
        :meth:`finish` (or the AURORA_OVERLAP split)."""
        if self.overlap:
            if dispatch_after is not None or dispatched is not None:
                raise ValueError("dispatch events exclude AURORA_OVERLAP (a second dispatch on the side stream)")
            return self._back_overlap(out)
        self.send(dispatch_after=dispatch_after, dispatched=dispatched)
        return self.finish(out)

    def send(self, *, dispatch_after: Optional[torch.cuda.Event] = None,
             dispatched: Optional[torch.cuda.Event] = None) -> None:
        """K2 and the dispatch on the current stream. ``dispatch_after``: the dispatch
        waits for this event (K2 still runs before it, so it overlaps what the event
        guards); ``dispatched`` is recorded when the dispatch has finished."""
        if self.overlap:
            raise ValueError("AURORA_OVERLAP layers run back() as a whole")
        if (dispatch_after is not None or dispatched is not None) and self.arrival_on:
            raise ValueError("dispatch events exclude N1 (GEMM1 launched right behind the dispatch)")
        main = torch.cuda.current_stream(self.dev)
        s = int(main.cuda_stream)
        if self.stream_schedule and dispatch_after is None:
            self.progress.zero_()  # stream-ordered before both K2 and the engine read it
            self.schedule(s)
            self.dispatch(s, overlap_schedule=True)
        else:
            self.schedule(s)
            if dispatch_after is not None:
                main.wait_event(dispatch_after)
            self.dispatch(s)
        if dispatched is not None:
            dispatched.record(main)
        if not self.arrival_on:  # N1: GEMM1 must directly follow the dispatch (PDL)
            self._mark("dispatched", main)

    def finish(self, out: Optional[torch.Tensor] = None, *,
               experts_after: Optional[torch.cuda.Event] = None) -> torch.Tensor:
        """Experts (+ fused combine), combine, aggregation on the current stream, after
        :meth:`send`. ``experts_after``: the expert GEMMs wait for this event."""
        self._check_out(out)
        main = torch.cuda.current_stream(self.dev)
        s = int(main.cuda_stream)
        if experts_after is not None:
            if self.arrival_on:
                raise ValueError("experts_after excludes N1 (GEMM1 launched right behind the dispatch)")
            main.wait_event(experts_after)
        if self.combine_in_gemm:
            self.experts_combine(s)
        else:
            self.experts(s)
        return self._tail(out, main)

    def _tail(self, out, main) -> torch.Tensor:
        s = int(main.cuda_stream)
        self._mark("experts_done", main)
        if self.combine_in_gemm:
            self.combine_wait(s)
        else:
            self.combine(s)
        self._mark("combined", main)
        self.aggregate(s, out)
        self._mark("end", main)
        return self.out if out is None else out

    def _back_overlap(self, out) -> torch.Tensor:
        """AURORA_OVERLAP=schedule|full: the local rows' dispatch + expert GEMM on the
        side stream beside K2 and the network dispatch (measured slower)."""
        self._check_out(out)
        main = torch.cuda.current_stream(self.dev)
        s = int(main.cuda_stream)
        mark = self._mark
        self._ev_pack.record(main)
        self.side.wait_event(self._ev_pack)
        ss = int(self.side.cuda_stream)
        self.dispatch(ss, "local")
        mark("local_copied", self.side)
        self.experts(ss, "local")
        mark("local_gemm_done", self.side)
        self._ev_local.record(self.side)
        # the remote dispatch may run with fewer copy CTAs beside the local GEMM
        # (AURORA_C_OVERLAP): K2 counts its hand-over thresholds for the CTAs the
        # dispatch will actually launch
        c_disp = (self.C_overlap or self.C) if self.overlap != "schedule" else self.C
        self.schedule(s, dispatch_ctas=c_disp)
        mark("scheduled", main)
        if self.overlap == "schedule":
            # only the (latency-bound) scheduler hides under the local GEMM;
            # the bandwidth-bound dispatch runs after it
            main.wait_event(self._ev_local)
            mark("joined", main)
            self.dispatch(s, "remote")
            mark("dispatched", main)
        else:
            c_full = self.C
            self.C = c_disp
            try:
                self.dispatch(s, "remote")
            finally:
                self.C = c_full
            mark("dispatched", main)
            main.wait_event(self._ev_local)
            mark("joined", main)
        self.experts(s, "remote")
        return self._tail(out, main)

    TRACE_POINTS = ("start", "packed", "local_copied", "local_gemm_done", "scheduled", "dispatched", "joined",
                    "experts_done", "combined", "end")
    # NVTX range opened at each trace point (the stage that starts there)
    NVTX_STAGES = {"start": "aurora: route + pack", "packed": "aurora: schedule + dispatch",
                   "local_copied": "aurora: local experts", "scheduled": "aurora: remote dispatch",
                   "dispatched": "aurora: experts", "joined": "aurora: remote experts",
                   "experts_done": "aurora: combine", "combined": "aurora: aggregate"}

    def timeline(self, x: torch.Tensor) -> dict:
        """One traced forward: ms from start to each point (diagnostics)."""
        self.trace = {k: torch.cuda.Event(enable_timing=True) for k in self.TRACE_POINTS}
        try:
            self.forward(x)
            torch.cuda.synchronize(self.dev)
            t0 = self.trace["start"]
            return {k: round(t0.elapsed_time(e), 4) for k, e in self.trace.items() if k in self._marked}
        finally:
            self.trace = None

    __call__ = forward

    def kernels_per_step(self) -> int:
        """Launches of this library's kernels in one forward (bench's gpu_launches)."""
        n = 1 if self.logits is None else (4 if self.router_tc else 2)  # router (+ rows, GEMM, exact pass / tail)
        n += 1 if self.grouped else 0                      # per-expert histogram
        n += 3                                             # pack, K2, dispatch engine
        if self.overlap:
            n += 3                                         # local dispatch + local GEMMs split off
        if self.G == 1:
            n += 2                                         # GEMM1 (+SwiGLU), GEMM2
        else:
            n += (0 if self.grouped else 4) + 2 + 1        # [sort x3, gather], GEMMs, pre-reduction
        n += 1                                             # combine engine or the fused combine's wait
        n += 1                                             # aggregate
        return n

    def capture(self, x: torch.Tensor, out: Optional[torch.Tensor] = None, warmup: int = 2):
        """CUDA graph of one forward on these exact input / output buffers (serving
        loops with fixed buffers: one graph launch instead of ~15 kernel launches
        and their host-side argument marshalling). Returns (graph, output); replay
        with ``graph.replay()`` after writing the next batch into ``x``. Every kernel
        reads its sizes and schedule from device memory, so replays see new routing.
        One process driving every rank only: the multi-process traffic-matrix
        exchange alternates buffers by step parity, which one graph cannot follow."""
        if self.n_local != self.n:
            raise NotImplementedError("graph capture of the multi-process layer (parity-alternating exchange)")
        s = torch.cuda.Stream(device=self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):  # first launches on this stream: kernel attributes, GEMM tile counters
            for _ in range(warmup):
                self.forward(x, out)
        torch.cuda.current_stream(self.dev).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            y = self.forward(x, out)
        return g, y

    def check_status(self) -> None:
        """Debug path: raise if the device scheduler or engine reported an error."""
        st, es = int(self.sched_i[1].item()), int(self.engine_status.item())
        if st != 0:
            raise RuntimeError(f"device scheduler status {st}")
        if es != 0:
            raise RuntimeError(f"engine status {es} (timeout)")

    def load_schedule(self, sched) -> None:
        """Replace this batch's engine tables with an arbitrary CommSchedule in
        token units (e.g. baselines.schedule_sjf of the same counts) -- the
        schedule ablation of SURVEY 8(f)3. Host -> device copy; diagnostics only."""
        from .baselines import to_engine_tables
        ch, rch, n_in, n_out = to_engine_tables(sched, self.n, self.cta_split(False), self.cta_split(True))
        if ch.shape[0] > self.P:
            raise ValueError(f"{ch.shape[0]} phases exceed the table capacity {self.P}")
        P = ch.shape[0]
        self.chunks[:P].copy_(torch.from_numpy(ch))
        self.rchunks[:P].copy_(torch.from_numpy(rch))
        self.n_in.copy_(torch.from_numpy(n_in))
        self.n_out.copy_(torch.from_numpy(n_out))
        if P:  # deadline pacing reads the phase durations
            self.phase_dur[:len(sched.phases)].copy_(torch.tensor([ph.duration for ph in sched.phases],
                                                                  dtype=torch.float64))
        self.sched_i[0] = len(sched.phases)
        self.progress.fill_(len(sched.phases) | PROGRESS_DONE)

    def schedule_objects(self):
        """The current batch's schedule as reference-shaped CommSchedule (debug / drop-in parity)."""
        from .commsched import CommSchedule, Phase
        nph = int(self.sched_i[0].item())
        pr = self.phase_recv[:nph].cpu().numpy()
        pd = self.phase_dur[:nph].cpu().numpy()
        phases = tuple(Phase(tuple((i, int(j)) for i, j in enumerate(row) if j >= 0), float(d))
                       for row, d in zip(pr, pd))
        return CommSchedule(self.n, phases, math.fsum(p.duration for p in phases))
