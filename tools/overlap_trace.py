"""Timeline of K2 + PDL dispatch on the C2 layer: when K2 publishes each
phase vs. when the engine's copy CTAs finish (globaltimer ns)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_17043_b200 import _lib
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig

cfg = MoEConfig(hidden=4096, ffn=14336, experts=8, top_k=2, tokens=16384, ranks=8, skew=1.0, seed=0)
layer = AuroraMoELayer(cfg)
x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
s = _lib.stream_ptr()
L = _lib.load()
layer(x); layer(x)
torch.cuda.synchronize()
st = torch.zeros(512, dtype=torch.int64, device="cuda")
et = torch.zeros(4 * 1024, dtype=torch.int64, device="cuda")
out = {}
L.aurora_debug_set_schedule_trace(st.data_ptr()); L.aurora_debug_set_engine_trace(et.data_ptr())
for mode in ("overlapped", "serial", "queued"):
    st.zero_(); et.zero_()
    layer.route(x, s); layer.pack(s); layer.progress.zero_()
    if mode != "queued":
        torch.cuda.synchronize()
    layer.schedule(s)
    if mode == "serial":
        torch.cuda.synchronize()
    layer.dispatch(s, overlap_schedule=(mode != "serial"))
    torch.cuda.synchronize()
    nph = int(layer.sched_i[0])
    pub = st[1:nph + 1].cpu().numpy()
    e = et.view(-1, 4)[:layer.n_local * layer.C].cpu().numpy()
    t0 = min(pub.min(), e[:, 0].min(), st[0].item())
    r = lambda v: round(float(v - t0) / 1e3, 1)
    ends = e[:, 2].reshape(layer.n_local, layer.C)
    out[mode] = {"phases": nph, "k2_start_us": r(st[0].item()), "publish_us": [r(v) for v in pub[::4]], "last_publish_us": r(pub[-1]),
                 "engine_start_us": r(e[:, 0].min()), "local_done_us": r(e[:, 1].max()),
                 "rank_end_us": [r(v) for v in ends.max(axis=1)]}
    print(mode, json.dumps(out[mode]), flush=True)
L.aurora_debug_set_schedule_trace(None); L.aurora_debug_set_engine_trace(None)
layer.check_status()
json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "overlap_trace.json"), "w"), indent=1)
st_ = torch.cuda.current_stream()
for sync_before in (True, False):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    tt = []
    for _ in range(5):
        layer.route(x, s); layer.pack(s); layer.progress.zero_()
        if sync_before:
            torch.cuda.synchronize()
        ev[0].record(st_); layer.schedule(s); layer.dispatch(s, overlap_schedule=True); ev[1].record(st_)
        layer.experts(s); layer.combine(s); layer.aggregate(s)
        torch.cuda.synchronize()
        tt.append(ev[0].elapsed_time(ev[1]) * 1e3)
    print("events schedule+dispatch, sync before" if sync_before else "events schedule+dispatch, queued", [round(v, 1) for v in tt], flush=True)

# K2's effective SM clock inside the queued layer sequence (cycles / ns)
prof = torch.zeros(8, dtype=torch.int64, device="cuda")
L.aurora_debug_set_schedule_profile(prof.data_ptr())
L.aurora_debug_set_schedule_trace(st.data_ptr())
for it in range(5):
    st.zero_()
    layer.route(x, s); layer.pack(s); layer.progress.zero_()
    layer.schedule(s); layer.dispatch(s, overlap_schedule=True)
    layer.experts(s); layer.combine(s); layer.aggregate(s)
    torch.cuda.synchronize()
    nph = int(layer.sched_i[0])
    ns = int(st[nph].item() - st[0].item())
    cyc = int(prof[6].item())
    print(f"queued iter {it}: K2 {cyc} cycles in {ns / 1e3:.1f} us -> {cyc / ns * 1e3:.0f} MHz", flush=True)
L.aurora_debug_set_schedule_profile(None)
L.aurora_debug_set_schedule_trace(None)
