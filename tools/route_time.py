"""Router (K1) time for one shape: median of CUDA-event timed layer.route calls and a
digest of its outputs (routing, weights, logits) to compare variants bit for bit.

    python tools/route_time.py TOKENS HIDDEN EXPERTS TOPK [RANKS]
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_17043_b200 import _lib  # noqa: E402
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig  # noqa: E402


def main(tokens, hidden, experts, topk, ranks=8):
    cfg = MoEConfig(hidden=hidden, ffn=256, experts=experts, top_k=topk, tokens=tokens, ranks=ranks, skew=1.0,
                    seed=0)
    layer = AuroraMoELayer(cfg)
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    s = _lib.stream_ptr()
    st = torch.cuda.current_stream()
    for _ in range(5):
        layer.route(x, s)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):  # back to back (the host enqueues ahead, as in the layer), mean per call
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(20):
            layer.route(x, s)
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / 20)
    h = hashlib.sha256()
    for t in (layer.topk_idx, layer.topk_w, layer.counts, layer.blk_cnt):
        h.update(t.cpu().numpy().tobytes())
    print(json.dumps({"tokens": tokens, "hidden": hidden, "experts": experts, "top_k": topk,
                      "route_us_median": round(float(np.median(ts)), 2), "route_us_min": round(float(np.min(ts)), 2),
                      "digest": h.hexdigest()[:16]}))


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
