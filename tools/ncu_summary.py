"""Summarise ncu --set full reports into profiles/: per kernel launch the
time, DRAM traffic and throughput, SM clock, occupancy and the top stall
reasons. Usage: python tools/ncu_summary.py out.json rep1.ncu-rep [rep2 ...]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]


def summarise(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = {}
    for r in data:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        m = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                m[k] = f"{r[i]} {units[i]}".strip()
        stalls = []
        for i, k in enumerate(hdr):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        m["top_stalls_per_issue"] = {s: round(v, 3) for v, s in sorted(stalls, reverse=True)[:5]}
        out.setdefault(name, []).append(m)
    return out


def main(dst, *reps):
    res = {}
    for rep in reps:
        for k, v in summarise(rep).items():
            res.setdefault(k, []).extend(v)
    json.dump(res, open(dst, "w"), indent=1)
    for k, v in res.items():
        print(k, v[0].get("gpu__time_duration.sum"), v[0].get("dram__bytes_read.sum"), v[0].get("top_stalls_per_issue"))


if __name__ == "__main__":
    main(*sys.argv[1:])
