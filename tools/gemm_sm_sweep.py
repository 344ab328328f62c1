"""Expert GEMM time vs the number of SMs it may use (C2 GEMM1 shape): what reserving SMs for
overlapped work (C3 interleaving) would cost. Usage: python tools/gemm_sm_sweep.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_17043_b200 import _lib
L = _lib.load()
G, m, N, K, ep = 8, 4096, 2 * 14336, 4096, 1
a = torch.randn(G * m, K, device="cuda").to(torch.bfloat16)
b = (torch.randn(G * N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
c = torch.empty(G * m, N // 2, device="cuda", dtype=torch.bfloat16)
rows = torch.full((G,), m, dtype=torch.int32, device="cuda")
ctr = torch.zeros(2, dtype=torch.int32, device="cuda")
for rep in range(2):
  for sms in (148, 140, 132, 116):
    run = lambda: L.aurora_grouped_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), None, rows.data_ptr(), G, m, N, K, ep, ctr.data_ptr(), sms, _lib.stream_ptr())
    for _ in range(3): run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): run()
    e1.record(); torch.cuda.synchronize()
    print(sms, round(e0.elapsed_time(e1) / 10, 3), "ms", flush=True)
