"""Would K2 pace an 8-GPU all-to-all? For the C2 layer run back to back (K2 at the clock it
gets right after the expert GEMM, as in steady state), record when K2 publishes each phase
(%globaltimer) and compare with when an engine following the schedule at the NVLink rate
would need it: phase k's data starts after sum_{j<k} dur_j x hidden x 2 B / 900 GB/s. The
largest publish-minus-need is the delay K2 would add to the 94 us bound at N = 8 (the
engine in loopback starts later anyway: local rows first). Both matcher variants.

    python tools/k2_n8_projection.py [out.json]
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_17043_b200 import _lib
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig

L = _lib.load()
NVLINK = 900e9
out = {"nvlink_gbps": NVLINK / 1e9, "cases": []}
for skew in (0.0, 1.0, 2.0):
    cfg = MoEConfig(hidden=4096, ffn=14336, experts=8, top_k=2, tokens=16384, ranks=8, skew=skew, seed=0)
    layer = AuroraMoELayer(cfg)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(cfg.tokens, cfg.hidden, device="cuda", generator=g).to(torch.bfloat16)
    s = _lib.stream_ptr()
    layer(x); layer(x)
    torch.cuda.synchronize()
    st = torch.zeros(512, dtype=torch.int64, device="cuda")
    case = {"skew": skew}
    for variant in (3, 0):
        L.aurora_debug_set_schedule_variant(variant)
        lags, k2s = [], []
        for it in range(4):
            layer(x)  # the previous step's GEMM sets the clock K2 sees
            L.aurora_debug_set_schedule_trace(st.data_ptr())
            st.zero_()
            layer(x)
            torch.cuda.synchronize()
            L.aurora_debug_set_schedule_trace(None)
            nph = int(layer.sched_i[0])
            raw = st[1:nph + 1].cpu().numpy().astype(np.float64)
            raw[raw == 0] = np.inf  # counts never published on their own (batched releases)
            pub = (raw - st[0].item()) / 1e3  # us after K2 start
            dur = layer.phase_dur[:nph].cpu().numpy()
            need = np.concatenate([[0.0], np.cumsum(dur)[:-1]]) * cfg.hidden * 2 / NVLINK * 1e6
            # publication is batched (up to 4 phases per release store): phase k is usable
            # once a publish covering it happened -- the recorded time of the first count >= k + 1
            usable = np.minimum.accumulate(pub[::-1])[::-1]
            lags.append(float(np.max(usable - need)))
            k2s.append(float(pub[-1]))
        case[f"variant{variant}"] = {"k2_last_publish_us": float(np.median(k2s)),
                                     "max_publish_minus_need_us": float(np.median(lags)),
                                     "bound_us": float(np.sum(dur) * cfg.hidden * 2 / NVLINK * 1e6),
                                     "phases": nph}
    L.aurora_debug_set_schedule_variant(0)
    print(json.dumps(case), flush=True)
    out["cases"].append(case)
    del layer
    torch.cuda.empty_cache()
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                           "gpurun_out", "k2_n8_projection.json")
json.dump(out, open(path, "w"), indent=1)
