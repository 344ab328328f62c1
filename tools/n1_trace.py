import sys, json, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2410_17043_b200 import _lib
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig
cfg = MoEConfig(hidden=4096, ffn=14336, experts=8, top_k=2, tokens=16384, ranks=8, skew=1.0, seed=0)
layer = AuroraMoELayer(cfg)
x = torch.randn(cfg.tokens, cfg.hidden, device="cuda").to(torch.bfloat16)
L = _lib.load()
out = {}
for on in (False, True, False, True):
    layer.arrival = on
    for _ in range(3): layer(x)
    torch.cuda.synchronize()
    eng = torch.zeros(4 * 4096, dtype=torch.int64, device="cuda"); gt = torch.zeros(2 * 1024, dtype=torch.int64, device="cuda")
    L.aurora_debug_set_engine_trace(eng.data_ptr()); L.aurora_debug_set_gemm_trace(gt.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); layer(x); e1.record(); torch.cuda.synchronize()
    L.aurora_debug_set_engine_trace(None); L.aurora_debug_set_gemm_trace(None)
    e = eng.view(-1, 4).cpu().numpy(); e = e[e[:, 0] > 0]; g = gt.view(-1, 2).cpu().numpy(); g = g[g[:, 0] > 0]
    t0 = e[:, 0].min()
    r = {"step_ms": e0.elapsed_time(e1), "eng_ctas": len(e), "eng_local_done_us": (np.percentile(e[:,1],[50,100]) - t0).tolist() if (e[:,1]>0).all() else None,
         "eng_end_us_p50_p100": (np.percentile(e[:, 2], [50, 100]) - t0).tolist(),
         "gemm_ctas": len(g), "gemm_entry_us_min_p50_max": (np.percentile(g[:, 0], [0, 50, 100]) - t0).tolist(),
         "gemm_first_tile_us_min_p50_max": (np.percentile(g[:, 1], [0, 50, 100]) - t0).tolist()}
    out[f"{'n1' if on else 'default'}_{len(out)}"] = r
    print(json.dumps(r), flush=True)
json.dump(out, open("gpurun_out/n1trace.json", "w"), indent=1)
