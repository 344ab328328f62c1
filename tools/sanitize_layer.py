"""Small MoE-layer forwards for compute-sanitizer (racecheck / synccheck /
memcheck): the TMA dispatch engine with pacing, K2 streamed to it (PDL), the
combine fused into GEMM2 / the pre-reduction, and the reversed-schedule
combine engine. Few copy CTAs per rank so every CTA stays co-resident under
instrumentation; a bounded spin limit turns a lost signal into an error
instead of a hang.  Usage: compute-sanitizer --tool racecheck python tools/sanitize_layer.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig  # noqa: E402


def run(cfg, **modes):
    layer = AuroraMoELayer(cfg, ctas_per_rank=2, spin_limit=1 << 22)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    ref = None
    for fused in (True, False):
        layer.fused_combine = fused
        for k, v in modes.items():
            setattr(layer, k, v)
        out = layer(x)
        torch.cuda.synchronize()
        layer.check_status()
        ref = out.clone() if ref is None else ref
        assert torch.equal(out, ref), (cfg, fused)
    print("ok", cfg.experts, cfg.top_k, cfg.ranks, flush=True)


if __name__ == "__main__":
    run(MoEConfig(hidden=256, ffn=256, experts=4, top_k=2, tokens=512, ranks=4, skew=1.0, seed=1))
    run(MoEConfig(hidden=256, ffn=128, experts=16, top_k=4, tokens=512, ranks=4, skew=1.0, seed=2))
    print("sanitize: done")
