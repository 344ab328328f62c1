"""Copy-CTA apportioning (csrc/apportion.cuh) and its host mirror
(paper_2410_17043_b200/apportion.py) agree bit-for-bit; every rank gets at
least one CTA and the totals are exact."""
import os
import subprocess

import numpy as np

from paper_2410_17043_b200.apportion import apportion

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_apportion_matches_device_header(tmp_path):
    exe = tmp_path / "apportion_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-o", str(exe), os.path.join(ROOT, "tests/native/apportion_check.cpp")],
                   check=True)
    rng = np.random.default_rng(3)
    cases, lines = [], []
    for it in range(600):
        n = int(rng.choice([1, 2, 3, 4, 6, 8, 12, 16, 32]))
        nl = int(rng.choice([d for d in range(1, n + 1) if n % d == 0]))
        ctot = nl * int(rng.integers(1, 40)) + int(rng.integers(0, nl))
        mode, comb = int(it % 3), int(rng.integers(0, 2))
        bw = rng.choice([1.0, 0.8, 0.5, 0.4, 100.0, 37.5], size=n)
        counts = rng.integers(0, 3000, size=(n, n)) * (rng.random((n, n)) < 0.8)
        if it % 17 == 0:
            counts[:] = 0
        cases.append((n, nl, ctot, mode, comb, bw, counts))
        lines.append(f"{n} {nl} {ctot} {mode} {comb} " + " ".join(repr(float(b)) for b in bw) + " "
                     + " ".join(str(int(v)) for v in counts.ravel()))
    out = subprocess.run([str(exe)], input="\n".join(lines) + "\n", capture_output=True, text=True, check=True)
    got = [list(map(int, ln.split())) for ln in out.stdout.strip().splitlines()]
    assert len(got) == len(cases)
    for (n, nl, ctot, mode, comb, bw, counts), dev in zip(cases, got):
        host = apportion(counts, n, nl, ctot, mode, bool(comb), bw)
        assert host == dev, (n, nl, ctot, mode, comb)
        for g0 in range(0, n, nl):
            assert sum(host[g0:g0 + nl]) == ctot and min(host[g0:g0 + nl]) >= 1


def test_apportion_volume_follows_load():
    counts = np.array([[100, 10, 10, 10], [10, 100, 10, 10], [10, 10, 100, 10], [3000, 3000, 3000, 100]])
    C = apportion(counts, 4, 4, 40, 1, False)  # dispatch: rank 3 sends the most
    assert C[3] == max(C) and sum(C) == 40
    C = apportion(counts, 4, 4, 40, 1, True)   # combine: returns follow column sums
    assert sum(C) == 40 and C[3] == min(C) and C[0] == C[1] == C[2]
    assert apportion(counts, 4, 1, 16, 1, False) == [16] * 4  # one rank per process: identity
