"""Copy-CTA count sweep of the TMA engine (C2, loopback): dispatch / combine
medians, paced and unpaced, without the GEMM between them."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_17043_b200 import _lib
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig

cfg = MoEConfig(hidden=4096, ffn=14336, experts=8, top_k=2, tokens=16384, ranks=8, skew=1.0, seed=0)
x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
s = _lib.stream_ptr()
st = torch.cuda.current_stream()
res = {}
layer = AuroraMoELayer(cfg)
layer(x)
torch.cuda.synchronize()
for C in (16, 24, 32, 37, 55, 74, 16, 24, 32, 37, 55, 74):
    layer.C = C
    for unpaced in (0, 16):
        layer.unpaced = unpaced
        dd, cc = [], []
        for _ in range(9):
            layer.route(x, s); layer.pack(s); layer.schedule(s)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record(st); layer.dispatch(s); ev[1].record(st)
            ev[2].record(st); layer.combine(s); ev[3].record(st)
            torch.cuda.synchronize()
            dd.append(ev[0].elapsed_time(ev[1]) * 1e3); cc.append(ev[2].elapsed_time(ev[3]) * 1e3)
        layer.check_status()
        key = f"C{C}/{'unpaced' if unpaced else 'paced'}"
        r = {"dispatch_us": round(sorted(dd)[4], 1), "combine_us": round(sorted(cc)[4], 1)}
        res.setdefault(key, []).append(r)
        print(key, r, flush=True)
json.dump(res, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                                 "engine_sweep.json"), "w"), indent=1)
