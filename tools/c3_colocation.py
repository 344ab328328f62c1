"""C3: Mixtral-shaped model a (8 experts) + a 16-expert top-2 model b (hidden 4096,
FFN 7168 -- the config leaves F open) colocated on 8 ranks by Aurora's plan, vs a
random pairing (colocate_rec, baselines.py:112-115). Loopback on one GPU."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_17043_b200.colocation import ColocatedLayers, ColocationPlan, combined_bmax, lina_slots, plan_colocation
from paper_2410_17043_b200.core import DeploymentPlan
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig

n = 8
cfg_a = MoEConfig(hidden=4096, ffn=14336, experts=8, top_k=2, tokens=16384, ranks=n, skew=1.0, seed=0)
cfg_b = MoEConfig(hidden=4096, ffn=7168, experts=16, top_k=2, tokens=16384, ranks=n, skew=1.5, seed=1)
xa = torch.randn(cfg_a.tokens, cfg_a.hidden, device="cuda").to(torch.bfloat16)
xb = torch.randn(cfg_b.tokens, cfg_b.hidden, device="cuda").to(torch.bfloat16)
cal_a = AuroraMoELayer(cfg_a)
cal_a(xa)
torch.cuda.synchronize()
counts_a = cal_a.counts.cpu().numpy()
del cal_a
cal_b = AuroraMoELayer(cfg_b)
cal_b(xb)
torch.cuda.synchronize()
loads_b = np.bincount(cal_b.topk_idx.cpu().numpy().ravel(), minlength=16)
slots = lina_slots(loads_b)
slot_of = [0] * 16
for s, (e1, e2) in enumerate(slots):
    slot_of[e1] = slot_of[e2] = s
cal_s = AuroraMoELayer(cfg_b, gpu_of_expert=slot_of, weights={"w_gate": cal_b.w_gate, "bias": cal_b.bias,
                                                                "w13": cal_b.w13, "w2": cal_b.w2})
cal_s(xb)
torch.cuda.synchronize()
slot_counts = cal_s.counts.cpu().numpy()
del cal_b, cal_s
torch.cuda.empty_cache()
aurora = plan_colocation(counts_a, slot_counts, slots)
rng = np.random.default_rng(0)
rand_pair = tuple(int(v) for v in rng.permutation(n))
rand_plan = DeploymentPlan.from_pairing(rand_pair)
gpu_of_b_rand = [0] * 16
for s, (e1, e2) in enumerate(slots):
    gpu_of_b_rand[e1] = gpu_of_b_rand[e2] = rand_plan.assignment_b[s]
rand = ColocationPlan(rand_plan, slots, tuple(rand_plan.assignment_a), tuple(gpu_of_b_rand))
res = {}
for name, cp in (("aurora", aurora), ("random", rand)):
    pair = ColocatedLayers(cfg_a, cfg_b, cp)
    for _ in range(3):
        pair(xa, xb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        pair(xa, xb)
    e1.record()
    torch.cuda.synchronize()
    pair.check_status()
    ms = e0.elapsed_time(e1) / 5
    res[name] = {"pairing": list(cp.plan.pairing), "combined_bmax_tokens": combined_bmax(counts_a, slot_counts, cp.plan),
                 "ms_both_layers": ms, "tokens_per_s": (cfg_a.tokens + cfg_b.tokens) / ms * 1e3,
                 "timeline_a": pair.a.timeline(xa), "timeline_b": pair.b.timeline(xb)}
    print(name, json.dumps(res[name]), flush=True)
    del pair
    torch.cuda.empty_cache()
json.dump(res, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                                 "c3_colocation.json"), "w"), indent=1)
