"""Grouped-GEMM microbenchmark (K5) at the layer's shapes: TFLOP/s of
aurora_grouped_gemm for C2 GEMM1/GEMM2 and C5 GEMM1/GEMM2 (64 groups, 1536
rows each). Usage: python tools/gemm_bench.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2410_17043_b200 import _lib

L = _lib.load()
cases = {  # name: (G, rows per group, N, K, epilogue)
    "c2_gemm1": (8, 4096, 2 * 14336, 4096, 1), "c2_gemm2": (8, 4096, 4096, 14336, 0),
    "c5_gemm1": (64, 1536, 2 * 1536, 5120, 1), "c5_gemm2": (64, 1536, 5120, 1536, 0),
}
for name, (G, m, N, K, ep) in cases.items():
    a = torch.randn(G * m, K, device="cuda").to(torch.bfloat16)
    b = (torch.randn(G * N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    c = torch.empty(G * m, N // 2 if ep else N, device="cuda", dtype=torch.bfloat16)
    rows = torch.full((G,), m, dtype=torch.int32, device="cuda")
    ctr = torch.zeros(2, dtype=torch.int32, device="cuda")
    run = lambda: L.aurora_grouped_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), None, rows.data_ptr(), G, m, N,
                                        K, ep, ctr.data_ptr(), 0, _lib.stream_ptr())
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    # cuBLAS on the same shape (batched, one matmul per group) for reference
    a3, b3 = a.view(G, m, K), b.view(G, N, K)
    cub = lambda: torch.bmm(a3, b3.transpose(1, 2))
    for _ in range(3):
        cub()
    e0.record()
    for _ in range(10):
        cub()
    e1.record()
    torch.cuda.synchronize()
    ms_cb = e0.elapsed_time(e1) / 10
    fl = 2.0 * G * m * N * K
    print(f"{name}: {ms * 1e3:8.1f} us  {fl / ms / 1e9:7.1f} TFLOP/s   cuBLAS bmm {ms_cb * 1e3:8.1f} us "
          f"{fl / ms_cb / 1e9:7.1f} TFLOP/s", flush=True)
    del a, b, c
