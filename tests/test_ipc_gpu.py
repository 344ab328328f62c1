"""The multi-GPU path through real CUDA IPC: two processes on one device, each
driving 4 of the 8 ranks -- and eight processes, one rank each (the N = 8
deployment's shape) -- peer tables from dist.connect_peers, system-scope
flags, gloo for the host collectives; output identical to the single-process
(loopback) layer, with K2 serial and overlapped, one and two experts per rank."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("variant,procs", [("e8", 2), ("e16", 2), ("e8", 8), ("e16", 8)])
def test_two_processes_cuda_ipc(variant, procs):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ipc_two_process.py"), variant, str(procs)],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count("identical to loopback: True") == 2, r.stdout
