"""Does the schedule pay on the engine?

On the C2 layer (16384 tokens, 8 ranks, loopback on one B200) for seeds 0-2 x
Zipf skews 0 / 1 / 2: dispatch + combine time of the same TMA copy engine
executing (a) Aurora's schedule (K2, build_schedule bit-exact), (b) the paper's
SJF and RCS baselines (baselines.py:91-109, host-built tables), (c) no schedule
(every pair at once, unpaced) -- all-to-all only, no GEMM in between (its
power-capped clocks would skew the copies). Also a sweep of the early pace
release (rows before a run's end at which the next sender may start).

    python tools/schedule_sweep.py [out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_17043_b200 import _lib  # noqa: E402
from paper_2410_17043_b200 import baselines as B  # noqa: E402
from paper_2410_17043_b200.core import ClusterSpec, TrafficMatrix  # noqa: E402
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig  # noqa: E402

L = _lib.load()
st = torch.cuda.current_stream()
s = _lib.stream_ptr()


def a2a(layer, x, sched=None, reps=7):
    """median dispatch / combine us of the engine on this batch (sched: host tables or K2)"""
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    dd, cc = [], []
    for _ in range(reps):
        layer.route(x, s)
        layer.pack(s)
        if sched is None:
            layer.schedule(s)
        else:
            layer.load_schedule(sched)
        ev[0].record(st)
        layer.dispatch(s)
        ev[1].record(st)
        ev[2].record(st)
        layer.combine(s)
        ev[3].record(st)
        torch.cuda.synchronize()
        dd.append(ev[0].elapsed_time(ev[1]) * 1e3)
        cc.append(ev[2].elapsed_time(ev[3]) * 1e3)
    layer.check_status()
    return {"dispatch_us": float(np.median(dd)), "combine_us": float(np.median(cc))}


def main(out=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                          "schedule_sweep.json")):
    res = {"cases": []}
    for skew in (0.0, 1.0, 2.0):
        for seed in (0, 1, 2):
            cfg = MoEConfig(hidden=4096, ffn=14336, experts=8, top_k=2, tokens=16384, ranks=8, skew=skew, seed=seed)
            layer = AuroraMoELayer(cfg)
            layer.fused_combine = False  # time the reversed-schedule combine engine too
            g = torch.Generator(device="cuda").manual_seed(100 + seed)
            x = torch.randn(cfg.tokens, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
            layer(x)
            torch.cuda.synchronize()
            d = layer.counts.cpu().numpy().astype(float)
            np.fill_diagonal(d, 0)
            tm, cl = TrafficMatrix(d), ClusterSpec.uniform(8)
            bmax = float(max(d.sum(0).max(), d.sum(1).max()))
            case = {"skew": skew, "seed": seed, "b_max_tokens": bmax,
                    "bound_us": bmax * cfg.hidden * 2 / 900e9 * 1e6,
                    "loopback_hbm_floor_us": 2 * layer.counts.sum().item() * cfg.hidden * 2 / 6.55e12 * 1e6}
            sj, rc = B.schedule_sjf(tm, cl), B.schedule_rcs(tm, cl, seed)
            case["makespan_tokens"] = {"aurora": bmax, "sjf": sj.makespan, "rcs": rc.makespan}
            for rep in range(2):  # alternate the arms twice (same power state)
                for name, sc in (("aurora", None), ("sjf", sj), ("rcs", rc), ("unpaced", None)):
                    layer.unpaced = 16 if name == "unpaced" else 0
                    r = a2a(layer, x, sc)
                    case.setdefault(name, []).append(r)
                layer.unpaced = 0
            for name in ("aurora", "sjf", "rcs", "unpaced"):
                runs = case[name]
                case[name] = {k: float(np.median([r[k] for r in runs])) for k in runs[0]}
            a = case["aurora"]
            case["aurora_total_vs"] = {k: (case[k]["dispatch_us"] + case[k]["combine_us"]) /
                                          (a["dispatch_us"] + a["combine_us"]) for k in ("sjf", "rcs", "unpaced")}
            print(json.dumps(case), flush=True)
            res["cases"].append(case)
            del layer
            torch.cuda.empty_cache()
    # early pace release sweep on one case (skew 1, seed 0)
    cfg = MoEConfig(hidden=4096, ffn=14336, experts=8, top_k=2, tokens=16384, ranks=8, skew=1.0, seed=0)
    layer = AuroraMoELayer(cfg)
    layer.fused_combine = False
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    layer(x)
    sweep = {}
    for rows in (0, 1, 2, 4, 8, 16, 64, 1 << 20):
        if rows == 0:
            layer.early_pace = 0
        else:
            layer.early_pace = 128
            L.aurora_debug_set_early_rows(rows)
        sweep[str(rows)] = a2a(layer, x)
        print("early rows", rows, sweep[str(rows)], flush=True)
    L.aurora_debug_set_early_rows(2)
    layer.early_pace = 128
    res["early_pace_rows_sweep"] = sweep
    agg = {k: float(np.mean([c["aurora_total_vs"][k] for c in res["cases"]])) for k in ("sjf", "rcs", "unpaced")}
    wins = {k: sum(c["aurora_total_vs"][k] > 1.0 for c in res["cases"]) for k in ("sjf", "rcs")}
    res["summary"] = {"mean_total_time_ratio_vs_aurora": agg, "cases_aurora_faster": wins,
                      "cases": len(res["cases"])}
    print(json.dumps(res["summary"]))
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
