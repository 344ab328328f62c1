"""The K2 fast-path matchers (csrc/fastmatch.cuh, fastmatch8b.cuh, fastmatch8d.cuh, fastmatch16.cuh; host+device) are bit-exact with
the oracle's perfect_matching / hopcroft_karp restatement (matching.py:20-112)
on 300k random bitmask graphs -- checked on the host, no GPU needed."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fastmatch_matches_oracle(tmp_path):
    exe = tmp_path / "fastmatch_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-o", str(exe), os.path.join(ROOT, "tests/native/fastmatch_check.cpp"),
                    "-x", "c", os.path.join(ROOT, "oracle/sched_oracle.c"), "-lm"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches: 0" in r.stdout
