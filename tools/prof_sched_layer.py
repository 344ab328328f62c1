"""Section cycles of the in-layer K2 launch (int32 counts, uniform cluster)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_17043_b200 import _lib
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig

L = _lib.load()
names = ["w0:snap+mask", "w0:match", "w0:update+publish", "w1:strip+chunks busy", "w1:", "prologue", "kernel", "w1:total"]
for n, T in ((8, 16384), (16, 16384)):
    cfg = MoEConfig(hidden=256, ffn=256, experts=n, top_k=2, tokens=T, ranks=n, skew=1.0, seed=0)
    layer = AuroraMoELayer(cfg)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    layer(x)
    torch.cuda.synchronize()
    prof = torch.zeros(8, dtype=torch.int64, device="cuda")
    L.aurora_debug_set_schedule_profile(prof.data_ptr())
    s = _lib.stream_ptr()
    for _ in range(3):
        layer.schedule(s)
    torch.cuda.synchronize()
    L.aurora_debug_set_schedule_profile(None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        layer.schedule(s)
    e1.record()
    torch.cuda.synchronize()
    pv = prof.cpu().tolist()
    pv[4] = f"close={pv[4] >> 32}/publish={pv[4] & 0xffffffff}"
    print(f"n={n}: {e0.elapsed_time(e1) / 20 * 1000:.1f} us/launch;",
          " ".join(f"{k}={v}" for k, v in zip(names, pv)), flush=True)
