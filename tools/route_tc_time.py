"""Router A/B at the C5 shape (64 experts top-6, hidden 5120, 16384 tokens): the FMA router
(aurora_route: balanced units + top-k tail) vs the tensor-core router (aurora_route_tc: grouped
GEMM for approximate logits, exact candidate pass + certificate, top-k tail); CUDA-event time per
call, alternated, and the number of uncertified (fallback) tokens."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2410_17043_b200 import _lib
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig

skew = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
cfg = MoEConfig(hidden=5120, ffn=1536, experts=64, top_k=6, tokens=16384, ranks=8, skew=skew, seed=0)
layers = {}
for mode in ("fma", "tc"):
    os.environ["AURORA_ROUTER"] = mode
    layers[mode] = AuroraMoELayer(cfg)
os.environ.pop("AURORA_ROUTER")
g = torch.Generator(device="cuda").manual_seed(3)
x = torch.randn(cfg.tokens, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
s = _lib.stream_ptr()
res = {m: [] for m in layers}
for rep in range(3):
    for mode, layer in layers.items():
        for _ in range(3):
            layer.route(x, s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            layer.route(x, s)
        e1.record()
        torch.cuda.synchronize()
        res[mode].append(e0.elapsed_time(e1) / 20 * 1000)
same = all(torch.equal(getattr(layers["tc"], a), getattr(layers["fma"], a))
           for a in ("topk_idx", "topk_w", "slot_dst", "blk_cnt", "counts"))
calls = 3 * 23
print(f"skew {skew}: fma {min(res['fma']):.1f} us, tc {min(res['tc']):.1f} us per route (best of 3 x 20); "
      f"fallback tokens {int(layers['tc'].n_fallback.item()) / calls:.1f} per call of {cfg.tokens}; "
      f"identical outputs {same}")
