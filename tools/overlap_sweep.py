"""Time the C2 layer under each overlap mode / copy-CTA count (diagnostics)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig

cfg = MoEConfig(hidden=4096, ffn=14336, experts=8, top_k=2, tokens=16384, ranks=8, skew=1.0, seed=0)
layer = AuroraMoELayer(cfg)
x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
res = {}
for mode, cov, c in [("none", 0, 18), ("schedule", 0, 18), ("schedule", 0, 32), ("full", 4, 18), ("full", 8, 18),
                     ("full", 16, 18), ("none", 0, 32)]:
    layer.overlap = False if mode == "none" else mode
    layer.C_overlap = cov
    layer.C = c
    for _ in range(3):
        layer(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        layer(x)
    e1.record()
    torch.cuda.synchronize()
    layer.check_status()
    key = f"{mode}/Cov{cov}/C{c}"
    res[key] = {"ms": e0.elapsed_time(e1) / 10, "timeline": layer.timeline(x)}
    print(key, round(res[key]["ms"], 3), res[key]["timeline"], flush=True)
json.dump(res, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "overlap_sweep.json"), "w"), indent=1)
