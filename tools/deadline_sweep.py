"""Deadline pacing ("time-triggered issue from prefix-sum start
times"): the TMA engine starts a run when the hand-over arrives OR when the
schedule's own clock reaches the run's phase (aurora_debug_set_deadline), on the
C2 layer's all-to-all (loopback, 3 skews x 2 seeds), against flag-only pacing and
the unpaced engine; then the layer step with the best rate, alternated with the
default.

    python tools/deadline_sweep.py [out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig  # noqa: E402
from tools.schedule_sweep import a2a  # noqa: E402

RATES = (400, 550, 700, 900, 1200)  # GB/s per sender assumed by the deadline clock


def set_deadline(layer, gbps):
    layer.deadline_gbps = float(gbps)


def step_ms(layer, x, steps=10):
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    layer(x)
    a.record(st)
    for _ in range(steps):
        layer(x)
    b.record(st)
    torch.cuda.synchronize()
    layer.check_status()
    return a.elapsed_time(b) / steps


def main(out=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                          "deadline_sweep.json")):
    res = {"rates_gbps": RATES, "cases": []}
    for skew in (0.0, 1.0, 2.0):
        for seed in (0, 1):
            cfg = MoEConfig(hidden=4096, ffn=14336, experts=8, top_k=2, tokens=16384, ranks=8, skew=skew, seed=seed)
            layer = AuroraMoELayer(cfg)
            layer.fused_combine = False  # a2a() also times the reversed-schedule combine engine
            g = torch.Generator(device="cuda").manual_seed(100 + seed)
            x = torch.randn(cfg.tokens, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
            ref = layer(x).clone()
            case = {"skew": skew, "seed": seed}
            for rep in range(2):
                for gb in (0,) + RATES + ("unpaced",):
                    layer.unpaced = 16 if gb == "unpaced" else 0
                    set_deadline(layer, 0 if gb == "unpaced" else gb)
                    case.setdefault(str(gb), []).append(a2a(layer, x)["dispatch_us"])
                layer.unpaced = 0
            set_deadline(layer, RATES[2])
            same = bool(torch.equal(layer(x), ref))
            set_deadline(layer, 0)
            case = {k: (float(np.median(v)) if isinstance(v, list) else v) for k, v in case.items()}
            case["outputs_identical_with_deadlines"] = same
            print(json.dumps(case), flush=True)
            res["cases"].append(case)
            del layer
            torch.cuda.empty_cache()
    keys = ("0",) + tuple(str(r) for r in RATES) + ("unpaced",)
    res["mean_dispatch_us"] = {k: float(np.mean([c[k] for c in res["cases"]])) for k in keys}
    best = min(RATES, key=lambda r: res["mean_dispatch_us"][str(r)])
    # the layer step (skew 1), deadline at the best rate vs flags only, alternated
    cfg = MoEConfig(hidden=4096, ffn=14336, experts=8, top_k=2, tokens=16384, ranks=8, skew=1.0, seed=0)
    layer = AuroraMoELayer(cfg)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    runs = {"flags": [], "deadline": []}
    for _ in range(3):
        for name, gb in (("flags", 0), ("deadline", best)):
            set_deadline(layer, gb)
            runs[name].append(step_ms(layer, x))
    set_deadline(layer, 0)
    res["layer_step_ms"] = {"best_rate_gbps": best, "runs": runs,
                            "median": {k: float(np.median(v)) for k, v in runs.items()}}
    print(json.dumps({"mean_dispatch_us": res["mean_dispatch_us"], "layer_step_ms": res["layer_step_ms"]}))
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
