"""C5 sweep: DeepSeek-style 64 experts top-6, hidden 5120, FFN 1536,
16384 tokens, routing skew s = 0..2, 2 / 4 / 8 expert-parallel ranks (loopback on
one GPU): layer tokens/s, scheduled vs unscheduled all-to-all, and the bound."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig

out = []
for n in (2, 4, 8):
    for s in (0.0, 1.0, 2.0):
        cfg = MoEConfig(hidden=5120, ffn=1536, experts=64, top_k=6, tokens=16384, ranks=n, skew=s, seed=0)
        layer = AuroraMoELayer(cfg)
        x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
        for _ in range(3):
            layer(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            layer(x)
        e1.record()
        torch.cuda.synchronize()
        layer.check_status()
        ms = e0.elapsed_time(e1) / 5
        tl = layer.timeline(x)
        layer.unpaced = 16
        tl_u = layer.timeline(x)
        layer.unpaced = 0
        c = layer.counts.cpu().numpy().astype(np.int64)
        np.fill_diagonal(c, 0)
        bmax = int(max(c.sum(1).max(), c.sum(0).max()))
        rec = {"ranks": n, "skew": s, "ms": ms, "tokens_per_s": cfg.tokens / ms * 1e3,
               "b_max_tokens": bmax, "bound_us": bmax * cfg.hidden * 2 / 900e9 * 1e6,
               "phases": int(layer.sched_i[0]), "timeline": tl, "timeline_unscheduled": tl_u}
        print(json.dumps(rec), flush=True)
        out.append(rec)
        del layer
        torch.cuda.empty_cache()
json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                                 "c5_sweep.json"), "w"), indent=1)
