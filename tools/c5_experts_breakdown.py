"""C5 (E > n) expert-stage breakdown: sort by local expert, row gather, the two
grouped GEMMs, pre-reduction. Usage: python tools/c5_experts_breakdown.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_17043_b200 import _lib
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig

cfg = MoEConfig(hidden=5120, ffn=1536, experts=64, top_k=6, tokens=16384, ranks=8, skew=1.0, seed=0)
layer = AuroraMoELayer(cfg)
layer.grouped_dispatch = False  # this breakdown times the receive / sort / gather path
x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
s = _lib.stream_ptr()
st = torch.cuda.current_stream()
L = layer.L
for _ in range(2):
    layer(x)
torch.cuda.synchronize()
k, H = cfg.top_k, cfg.hidden
E_loc = layer.n_local * layer.G
names = ["sort", "gather", "gemms", "reduce"]
tot = {n_: 0.0 for n_ in names}
R = 5
for _ in range(R):
    layer.route(x, s); layer.pack(s); layer.schedule(s); layer.dispatch(s)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record(st)
    L.aurora_expert_sort(layer.meta_recv.data_ptr(), layer.cap, layer.meta_bytes, layer.rtot.data_ptr(), layer.n_local,
                         layer.rank_base, k, layer.G, layer.g_off.data_ptr(), layer.g_rows.data_ptr(),
                         layer.g_src.data_ptr(), layer.inv.data_ptr(), layer.sort_scratch.data_ptr(),
                         layer.sort_scratch.numel(), s)
    ev[1].record(st)
    L.aurora_gather_rows(layer.recv.data_ptr(), layer.a_g.data_ptr(), layer.g_src.data_ptr(),
                         layer.g_off[E_loc:].data_ptr(), layer.max_entries, H * 2, s)
    ev[2].record(st)
    L.aurora_expert_ffn_packed(layer.a_g.data_ptr(), layer.w13.data_ptr(), layer.w2.data_ptr(), layer.h_g.data_ptr(),
                               layer.y_g.data_ptr(), layer.g_off.data_ptr(), layer.g_rows.data_ptr(), E_loc,
                               layer.max_entries, H, cfg.ffn, None, layer.G, layer.tile_ctrs[0].data_ptr(), layer.num_sms, s)
    ev[3].record(st)
    L.aurora_expert_reduce(layer.y_g.data_ptr(), layer.inv.data_ptr(), layer.meta_recv.data_ptr(), layer.cap,
                           layer.meta_bytes, layer.rtot.data_ptr(), layer.n_local, layer.rank_base, k, H,
                           layer.ybuf.data_ptr(), 0, s)
    ev[4].record(st)
    layer.combine(s); layer.aggregate(s)
    torch.cuda.synchronize()
    for i, n_ in enumerate(names):
        tot[n_] += ev[i].elapsed_time(ev[i + 1]) / R
rows = int(layer.g_rows.sum().item())
print({n_: round(v * 1e3, 1) for n_, v in tot.items()}, "rows", rows, "gather GB/s",
      round(2 * rows * H * 2 / (tot["gather"] * 1e-3) / 1e9), flush=True)
