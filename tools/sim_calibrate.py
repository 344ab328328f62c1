"""calibrate the reference's timeline model with measured kernels.

Reads a bench line (profiles/r01_bench_c2.json: per-stage times and the step's
traffic matrix), fits the reference's LayerProfile work parameters in its own
time unit (one token over one link direction at B = 1, i.e. hidden x 2 B /
900 GB/s), and runs the reference simulator -- moeplan.sim.simulate_exclusive
(sim.py:130-154) with Aurora's build_schedule and with the SJF / RCS baselines
(baselines.py:91-109) -- to predict the layer on 8 GPUs (one expert each).
Runs in the build container, where the reference package is importable
(PYTHONPATH=baseline/_ref or /root/reference/pkg/src); never on the GPU box. Also
writes the experiment CSV (experiment.py:26-39) with measured and predicted rows.

    PYTHONPATH=baseline/_ref python tools/sim_calibrate.py [bench.json] [out.json]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(src=os.path.join(ROOT, "profiles", "r02_bench_c2.json"),
         dst=os.path.join(ROOT, "profiles", "r02_sim_calibration.json")):
    from moeplan import baselines as RB
    from moeplan.core import ClusterSpec, LayerProfile, TrafficMatrix
    from moeplan.sim import simulate_exclusive

    line = json.loads(open(src).read().strip().splitlines()[-1])
    cfg, st, a2a = line["config"], line["stage_ms_serial"], line["all_to_all"]
    counts = np.asarray(a2a["traffic_matrix"], dtype=float)
    n, H = counts.shape[0], cfg["hidden"]
    tau_us = H * 2 / 900e9 * 1e6  # one token at B = 1 (the paper's big switch)
    rows = counts.sum()            # (token, expert) rows the expert GEMMs processed (all ranks, loopback)
    # loopback ran every rank's gate / aggregation on one GPU: one GPU's share is 1/n of it
    # (both are HBM-bound over the rank's own tokens); FFN: GPU time per (token, expert) row
    prof = LayerProfile(gate_work=(st["route"] + st["pack"]) * 1e3 / n / tau_us,
                        agg_work=st["aggregate"] * 1e3 / n / tau_us,
                        ffn_work_per_token=st["experts"] * 1e3 / rows / tau_us,
                        ffn_base_work=0.0,
                        d_first=TrafficMatrix(counts))  # the diagonal (local rows) is dropped, core.py:95
    cluster = ClusterSpec.uniform(n)
    ident = tuple(range(n))
    out = {"source": os.path.relpath(src, ROOT), "time_unit_us": tau_us,
           "fitted_profile": {"gate_work": prof.gate_work, "agg_work": prof.agg_work,
                              "ffn_work_per_token": prof.ffn_work_per_token, "ffn_base_work": 0.0},
           "measured_loopback": {"ms_per_step": line["ms_per_step"], "dispatch_us": a2a["dispatch_us"],
                                 "combine_us": a2a["combine_us"], "schedule_us": a2a["schedule_us"],
                                 "note": "1 x B200, all 8 ranks on one GPU: the expert GEMMs of all ranks "
                                         "run one after another"},
           "predicted_8gpu": {}}
    for name, fn in (("aurora", None), ("sjf", RB.schedule_sjf),
                     ("rcs", lambda d, c: RB.schedule_rcs(d, c, 0))):
        r = simulate_exclusive(prof, ident, cluster, schedule_fn=fn)
        out["predicted_8gpu"][name] = {
            "layer_us": r.inference_time * tau_us,
            "spans_us": {k: [v.start * tau_us, v.end * tau_us] for k, v in r.spans.items()},
            "all_to_all_us": (r.spans["N"].duration + r.spans["C"].duration) * tau_us,
            "utilization": r.utilization}
    a = out["predicted_8gpu"]["aurora"]
    out["summary"] = (f"reference model, 8 GPUs, measured kernel rates: layer {a['layer_us']:.0f} us "
                      f"(all-to-all {a['all_to_all_us']:.0f} us = 2 x b_max); SJF "
                      f"{out['predicted_8gpu']['sjf']['layer_us']:.0f} us, RCS "
                      f"{out['predicted_8gpu']['rcs']['layer_us']:.0f} us; loopback measured "
                      f"{line['ms_per_step'] * 1e3:.0f} us for all 8 ranks on one GPU")
    json.dump(out, open(dst, "w"), indent=1)
    print(out["summary"])
    # the experiment CSV (experiment.py:26-39): measured loopback rows (this repo's report.py)
    # followed by the reference simulator's 8-GPU predictions as its own ResultRow objects
    import moeplan.experiment as mexp
    sys.path.insert(0, ROOT)
    from paper_2410_17043_b200.report import measured_rows
    rows = measured_rows(line)
    for name, pr in out["predicted_8gpu"].items():
        rows.append(mexp.ResultRow("exclusive-homo", f"{name}-predicted-8gpu", 0, n, 0.0, cfg["seed"],
                                   pr["spans_us"]["N"][1] / tau_us - pr["spans_us"]["N"][0] / tau_us,
                                   pr["spans_us"]["C"][1] / tau_us - pr["spans_us"]["C"][0] / tau_us,
                                   pr["layer_us"] / tau_us, pr["utilization"]))
    csv_path = os.path.splitext(dst)[0] + ".csv"
    open(csv_path, "w").write(mexp.csv_text(rows))
    print("wrote", os.path.relpath(csv_path, ROOT))


if __name__ == "__main__":
    main(*sys.argv[1:])
