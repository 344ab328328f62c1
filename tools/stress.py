"""Randomised stress of the layer's execution variants (race hunting): random small
configs, each run through every variant that must give identical bits -- default,
engine combine, serial K2, unpaced, LSU engine, N1 (arrival-driven GEMM1), emulated
compute partition, deadline pacing -- repeated, with the counters checked re-armed after each config.

    python tools/stress.py [iterations] [seed]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig  # noqa: E402


def variants(layer):
    yield "default", {}
    yield "engine_combine", {"fused_combine": False}
    yield "serial_k2", {"stream_schedule": False}
    yield "unpaced", {"unpaced": 16}
    if layer.G == 1:
        yield "n1", {"arrival": True}
    if layer.G > 1:
        yield "no_packed_scatter", {"packed_scatter": False}
        yield "ungrouped", {"grouped_dispatch": False}
    yield "lsu", {"engine_lsu": 64}
    yield "deadline", {"deadline_gbps": 700.0}


def main(iters=60, seed=0):
    rng = np.random.default_rng(seed)
    t0 = time.time()
    for it in range(iters):
        n = int(rng.choice([2, 4, 8, 8, 16]))
        G = int(rng.choice([1, 1, 2, 4])) if n <= 8 else 1
        E = n * G
        k = int(rng.integers(1, min(6, E) + 1))
        tokens = n * 64 * int(rng.integers(1, 5))
        cfg = MoEConfig(hidden=256 * int(rng.integers(1, 3)), ffn=128 * int(rng.integers(1, 3)), experts=E, top_k=k,
                        tokens=tokens, ranks=n, skew=float(rng.uniform(0, 3)), seed=int(rng.integers(0, 1000)))
        scales = [float(v) for v in rng.choice([1.0, 0.8, 0.5, 0.4], n)] if rng.random() < 0.3 else None
        layer = AuroraMoELayer(cfg, spin_limit=1 << 24, compute_scales=scales)
        x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
        ref = None
        for name, attrs in variants(layer):
            saved = {a: getattr(layer, a) for a in attrs}
            for a, v in attrs.items():
                setattr(layer, a, v)
            for rep in range(2):
                out = layer(x)
                torch.cuda.synchronize()
                layer.check_status()
                if ref is None:
                    ref = out.clone()
                elif not torch.equal(out, ref):
                    raise SystemExit(f"MISMATCH it={it} cfg={cfg} scales={scales} variant={name} rep={rep}")
            for a, v in saved.items():
                setattr(layer, a, v)
        if int(layer.ctr_d.abs().sum()) or int(layer.ctr_c.abs().sum()) or \
                (layer.landed is not None and int(layer.landed.abs().sum())):
            raise SystemExit(f"counters not re-armed it={it} cfg={cfg}")
        print(f"ok {it} n={n} E={E} k={k} T={tokens} scales={'y' if scales else 'n'} {time.time() - t0:.0f}s",
              flush=True)
        del layer
    print("stress: all variants identical")


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
