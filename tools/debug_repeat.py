"""Diagnostics: back-to-back layer calls (no host sync) with per-call device
snapshots of the scheduler / engine state."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
cfg = MoEConfig(hidden=256, ffn=256, experts=8, top_k=2, tokens=2048, ranks=8, skew=0.5, seed=2)
layer = AuroraMoELayer(cfg, spin_limit=1 << 16)
x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
N = 6
snap = torch.zeros(N, 8, dtype=torch.int32, device="cuda")
tl = []
for it in range(N):
    layer.trace = {k: torch.cuda.Event(enable_timing=True) for k in layer.TRACE_POINTS}
    layer(x)
    tl.append(layer.trace)
    layer.trace = None
    snap[it, 0] = layer.progress[0]
    snap[it, 1] = layer.engine_status[0]
    snap[it, 2:4] = layer.sched_i
torch.cuda.synchronize()
for it in range(N):
    t0 = tl[it]["start"]
    print(it, "prog", hex(int(snap[it, 0])), "eng", int(snap[it, 1]), "sched", snap[it, 2:4].tolist(),
          {k: round(t0.elapsed_time(e), 3) for k, e in tl[it].items() if k in ("packed", "dispatched", "experts_done", "combined", "end")})
