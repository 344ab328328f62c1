"""K2 in-layer A/B: launch time and section cycles of the scheduler variants
(aurora_debug_set_schedule_variant: 0 = cell-lane decomposition + strip (default),
1 = per-step masks, 2 = cell-lane decomposition + row-lane strip, 3 = row-lane
incremental decomposition + strip), identical outputs checked. Layer shapes are small: K2
only sees the traffic matrix, which depends on routing (tokens, ranks, skew)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
torch.manual_seed(0)
from paper_2410_17043_b200 import _lib
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig

L = _lib.load()
VARIANTS = tuple(int(v) for v in os.environ.get("K2_VARIANTS", "3,0,3,0").split(","))
names = ["w0:snap+mask", "w0:match", "w0:update+publish", "w1:strip busy", "w1:close/publish", "prologue", "kernel", "w1:total"]
for skew in (0.0, 1.0, 2.0):
    cfg = MoEConfig(hidden=256, ffn=256, experts=8, top_k=2, tokens=16384, ranks=8, skew=skew, seed=0)
    layer = AuroraMoELayer(cfg)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
    layer(x)
    torch.cuda.synchronize()
    s = _lib.stream_ptr()
    res = {}
    for var in VARIANTS:
        L.aurora_debug_set_schedule_variant(var)
        prof = torch.zeros(8, dtype=torch.int64, device="cuda")
        L.aurora_debug_set_schedule_profile(prof.data_ptr())
        for _ in range(3):
            layer.schedule(s)
        torch.cuda.synchronize()
        L.aurora_debug_set_schedule_profile(None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            layer.schedule(s)
        e1.record()
        torch.cuda.synchronize()
        sched = layer.schedule_objects()
        key = [(p.transfers, p.duration) for p in sched.phases]
        if var in res:
            assert res[var][0] == key
        res[var] = (key, e0.elapsed_time(e1) / 50 * 1000, prof.cpu().tolist())
        pv = res[var][2]
        pv[4] = f"{pv[4] >> 32}/{pv[4] & 0xffffffff}"
        print(f"skew {skew} variant {var}: {res[var][1]:.1f} us/launch, {len(key)} phases;",
              " ".join(f"{k}={v}" for k, v in zip(names, pv)), flush=True)
    assert all(res[v][0] == res[VARIANTS[0]][0] for v in res), "variants disagree"
    L.aurora_debug_set_schedule_variant(0)
print("identical phases across variants")
