"""One in-layer K2 launch on a C2-shaped traffic matrix (skew 1), for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
torch.manual_seed(0)
from paper_2410_17043_b200 import _lib
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig

cfg = MoEConfig(hidden=256, ffn=256, experts=8, top_k=2, tokens=16384, ranks=8, skew=float(os.environ.get("SKEW", "1.0")), seed=0)
layer = AuroraMoELayer(cfg)
x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
layer(x)
torch.cuda.synchronize()
s = _lib.stream_ptr()
for _ in range(3):
    layer.schedule(s)
torch.cuda.synchronize()
print("phases", len(layer.schedule_objects().phases))
