"""The reference arm of bench.py (CPU only): one JSON line with the contract
keys, the reference's own build_schedule timed on the workload's traffic
matrix next to the C restatement, and both giving the same phases."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    cmd = [sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1",
           "--tokens", "2048", "--hidden", "256", "--ffn", "256"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "tokens/s"
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["cores"] >= 1 and cb["kind"] in ("port", "reference")
    assert d["e2e"] == {"value": d["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    sch = cb["schedule"]
    assert sch["port_build_schedule_ms"] > 0
    if "moeplan_build_schedule_ms" in sch:  # reference installed (baseline/_ref)
        assert sch["port_identical"] is True and sch["moeplan_build_schedule_ms"] > 0
