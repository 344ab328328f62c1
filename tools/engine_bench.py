"""Engine microbenchmark on the C2 layer (loopback): dispatch / combine time for
the TMA and LSU copy paths, schedule-paced and unpaced, plus K2+dispatch
overlapped. Usage: python tools/engine_bench.py [--config c5]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_17043_b200 import _lib
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig

c5 = "--config" in sys.argv and sys.argv[sys.argv.index("--config") + 1] == "c5"
cfg = (MoEConfig(hidden=5120, ffn=1536, experts=64, top_k=6, tokens=16384, ranks=8, skew=1.0, seed=0) if c5 else
       MoEConfig(hidden=4096, ffn=14336, experts=8, top_k=2, tokens=16384, ranks=8, skew=1.0, seed=0))
layer = AuroraMoELayer(cfg)
x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
s = _lib.stream_ptr()
st = torch.cuda.current_stream()
for _ in range(2):
    layer(x)
torch.cuda.synchronize()
layer.check_status()
res = {}
def a2a_only(reps=12):
    """dispatch / combine medians without the GEMM in between (its power-capped clocks skew the copies)"""
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    dd, cc = [], []
    for _ in range(reps):
        layer.route(x, s); layer.pack(s); layer.schedule(s)
        ev[0].record(st); layer.dispatch(s); ev[1].record(st)
        ev[2].record(st); layer.combine(s); ev[3].record(st)
        torch.cuda.synchronize()
        dd.append(ev[0].elapsed_time(ev[1]) * 1e3); cc.append(ev[2].elapsed_time(ev[3]) * 1e3)
    layer.check_status()
    return {"dispatch_us": round(sorted(dd)[reps // 2], 1), "combine_us": round(sorted(cc)[reps // 2], 1)}


for early in (0, 128, 0, 128):  # A/B of the early pace release, interleaved
    layer.early_pace = early
    r = a2a_only()
    res[f"tma/{'early' if early else 'end'}_pace_nogemm"] = r
    print("early pace" if early else "pace at run end", r, flush=True)
layer.early_pace = 128
for eng in ("tma", "lsu"):
    layer.engine_lsu = 64 if eng == "lsu" else 0
    for paced in (True, False):
        layer.unpaced = 0 if paced else 16
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        d = cmb = 0.0
        R = 5
        for _ in range(R):
            layer.route(x, s); layer.pack(s); layer.schedule(s)
            ev[0].record(st); layer.dispatch(s); ev[1].record(st)
            layer.experts(s)
            ev[2].record(st); layer.combine(s); ev[3].record(st)
            layer.aggregate(s)
            torch.cuda.synchronize()
            d += ev[0].elapsed_time(ev[1]); cmb += ev[2].elapsed_time(ev[3])
        layer.check_status()
        res[f"{eng}/{'paced' if paced else 'unpaced'}"] = {"dispatch_us": round(d / R * 1e3, 1), "combine_us": round(cmb / R * 1e3, 1)}
        print(eng, "paced" if paced else "unpaced", res[f"{eng}/{'paced' if paced else 'unpaced'}"], flush=True)
layer.unpaced = 0
for eng in ("tma", "lsu"):
    layer.engine_lsu = 64 if eng == "lsu" else 0
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    t = 0.0
    for _ in range(5):
        layer.route(x, s); layer.pack(s); layer.progress.zero_()
        ev[0].record(st); layer.schedule(s); layer.dispatch(s, overlap_schedule=True); ev[1].record(st)
        layer.experts(s); layer.combine(s); layer.aggregate(s)
        torch.cuda.synchronize()
        t += ev[0].elapsed_time(ev[1])
    layer.check_status()
    res[f"{eng}/schedule+dispatch"] = round(t / 5 * 1e3, 1)
    print(eng, "schedule+dispatch overlapped", res[f"{eng}/schedule+dispatch"], flush=True)
json.dump(res, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                                 "engine_bench.json"), "w"), indent=1)

# K2's own cycles when it runs alone vs. beside the PDL-launched engine
layer.engine_lsu = 0
prof = torch.zeros(8, dtype=torch.int64, device="cuda")
L = _lib.load()
L.aurora_debug_set_schedule_profile(prof.data_ptr())
for mode in ("alone", "overlapped"):
    tot = torch.zeros(8, dtype=torch.int64)
    for _ in range(5):
        layer.route(x, s); layer.pack(s); layer.progress.zero_()
        layer.schedule(s)
        if mode == "alone":
            torch.cuda.synchronize()
        layer.dispatch(s, overlap_schedule=(mode == "overlapped"))
        torch.cuda.synchronize()
        tot += prof.cpu()
    print("K2", mode, "kernel cycles", int(tot[6]) // 5, "match", int(tot[1]) // 5, "w1 total", int(tot[7]) // 5, flush=True)
L.aurora_debug_set_schedule_profile(None)
layer.check_status()
