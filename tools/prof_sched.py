"""Per-section cycle counts of the K2 scheduler (diagnostics entry point)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_17043_b200 import _lib
L = _lib.load()
rng = np.random.default_rng(0)
for n in (4, 8, 16):
    pop = 1.0 / (rng.permutation(n) + 1.0)
    m = np.round(np.outer(rng.uniform(1800, 2200, n), pop / pop.sum()) * rng.uniform(0.9, 1.1, (n, n)))
    np.fill_diagonal(m, 0)
    d = torch.tensor(m, dtype=torch.float64, device="cuda")
    prof = torch.zeros(8, dtype=torch.int64, device="cuda")
    sc = torch.zeros(4 * n * n * n, dtype=torch.int32, device="cuda")
    ds = torch.zeros(4 * n * n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        L.aurora_debug_schedule_cycles(d.data_ptr(), n, prof.data_ptr(), sc.data_ptr(), ds.data_ptr(), _lib.stream_ptr())
    torch.cuda.synchronize()
    p = prof.cpu().tolist()
    print(f"n={n}: cycles snap+mask={p[0]} match={p[1]} update={p[2]} strip={p[3]} total={p[4]}")
