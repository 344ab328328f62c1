"""Device latency of the K2 scheduler kernel (CUDA events, 200 launches)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2410_17043_b200 import _lib

L = _lib.load()
rng = np.random.default_rng(0)
for n in (2, 4, 8, 16, 32):
    pop = 1.0 / (rng.permutation(n) + 1.0) ** 1.0
    m = np.round(np.outer(rng.uniform(1800, 2200, n), pop / pop.sum()) * rng.uniform(0.9, 1.1, (n, n)))
    np.fill_diagonal(m, 0)
    d = torch.tensor(m, dtype=torch.float64, device="cuda")
    R, P = L.aurora_raw_phase_cap(n), L.aurora_phase_cap(n)
    rp = torch.empty(R * n, dtype=torch.int32, device="cuda"); rd = torch.empty(R, dtype=torch.float64, device="cuda")
    pr = torch.empty(P * n, dtype=torch.int32, device="cuda"); pd = torch.empty(P, dtype=torch.float64, device="cuda")
    sc = torch.zeros(4, dtype=torch.int32, device="cuda"); bm = torch.zeros(1, dtype=torch.float64, device="cuda")
    s = _lib.stream_ptr()
    call = lambda: L.aurora_schedule_f64(d.data_ptr(), None, n, rp.data_ptr(), rd.data_ptr(), sc.data_ptr(),
                                         pr.data_ptr(), pd.data_ptr(), sc[1:].data_ptr(), bm.data_ptr(), sc[2:].data_ptr(), s)
    for _ in range(5): call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200): call()
    e1.record(); torch.cuda.synchronize()
    print(f"n={n}: {e0.elapsed_time(e1)/200*1000:.1f} us per schedule; raw={int(sc[0])} phases={int(sc[1])} status={int(sc[2])}")
