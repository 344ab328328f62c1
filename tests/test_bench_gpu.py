"""bench.py's multi-process path end to end on one GPU: torchrun with two
processes sharing cuda:0 (AURORA_BENCH_SAME_GPU=1: CUDA IPC peer tables, the
counts exchange by peer stores, the fused combine across processes, max-over-
ranks timing), and the contract keys of the JSON line."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_processes_same_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, AURORA_BENCH_SAME_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--tokens", "4096", "--hidden", "1024", "--ffn", "1024",
           "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    d = lines[0]
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0 and d["gpu_launches"] > 0
    assert "sharing one GPU" in d["all_to_all"]["transport"]
    assert "unavailable" in d["all_to_all"]["unscheduled_library"]
    assert 0 < d["roofline"]["gemm_ms_per_step"] <= d["ms_per_step"]
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
