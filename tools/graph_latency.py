"""Per-layer latency, eager forward vs one CUDA-graph replay (layer.capture), at
serving-size batches of the C2 layer: where the GPU work is short the ~15
launches and their host-side argument marshalling show. Usage:
python tools/graph_latency.py [tokens ...]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_17043_b200.layer import AuroraMoELayer, MoEConfig

sizes = [int(a) for a in sys.argv[1:]] or [512, 2048, 8192, 16384]
out = {}
for T in sizes:
    cfg = MoEConfig(hidden=4096, ffn=14336, experts=8, top_k=2, tokens=T, ranks=8, skew=1.0, seed=0)
    layer = AuroraMoELayer(cfg)
    x = torch.randn(T, cfg.hidden, device="cuda").to(torch.bfloat16)
    o = torch.empty_like(x)
    for _ in range(3):
        layer(x, out=o)
    torch.cuda.synchronize()
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        layer(x, out=o)
    e1.record()
    t_host = (time.perf_counter() - t0) / reps * 1e3
    torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) / reps
    g, y = layer.capture(x, o)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / reps
    layer.check_status()
    out[T] = {"eager_ms": round(eager, 3), "graph_ms": round(graph, 3), "eager_host_enqueue_ms": round(t_host, 3)}
    print(T, out[T], flush=True)
    del layer, x, o, g, y
    torch.cuda.empty_cache()
print(json.dumps(out))
