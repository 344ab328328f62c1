"""The multi-GPU path through real CUDA IPC: two processes on one device, each
driving 4 of the 8 ranks, peer tables from dist.connect_peers, system-scope
flags, gloo for the host collectives; output identical to the single-process
(loopback) layer, with K2 serial and overlapped, one and two experts per rank."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("variant", ["e8", "e16"])
def test_two_processes_cuda_ipc(variant):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ipc_two_process.py"), variant],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count("identical to loopback: True") == 2, r.stdout
