"""C5 plan-search RATE (BASELINE.json configs[4]: 4-model cascade, 10M-request
trace, 128-GPU pool, full TP/PP/DP enumeration).  The full sweep is ~10^13
(row, plan) pairs -- intractable for any exact method in a bench run, and the
reference CPU planner cannot even materialise its plan sets (~3*10^12 plans per
small-model row) -- so this reports RATES on sampled filter waves and an
EXTRAPOLATED 1-GPU sweep time (labelled as such):

  * routing of the full 10M-request trace over the default decile grid
    (cg_route_grid: K1-K3 + K2 quality), measured;
  * per stage, one representative unique row evaluated through cg_stage_row
    with the rate-sampling options (pilot off, `max_waves` filter waves spread
    by `wave_stride` over the row's whole plan-index space): plans/s,
    request-steps/s, stable fraction;
  * extrapolation: sum over the sweep's unique rows of plans / (that stage's
    sampled plans/s).  Bounds come from the sampled waves only, so they are
    looser than in a full run: the estimate is conservative (an upper bound
    on the time the same kernels would need).

  python tools/c5_rate_probe.py [waves_per_row] [out.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_04203_b200 import engine as eng, workloads as W  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 6
out_path = sys.argv[2] if len(sys.argv) > 2 else None
name = "C5"
t0 = time.time()
parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs(name)]
t = eng.concat_traces(parts) if len(parts) > 1 else parts[0]
n, C = int(t["arrival_s"].shape[0]), int(t["scores"].shape[0])
cfg, N = W.planner_config(name, t["scores"])
gen_s = time.time() - t0
E = eng.Engine(0)
dev = {k: torch.from_numpy(np.ascontiguousarray(t[k])).cuda() for k in t}
tb = eng.TraceBuffers(dev["arrival_s"].data_ptr(), dev["input_tokens"].data_ptr(), dev["output_tokens"].data_ptr(),
                      dev["scores"].data_ptr(), on_device=True, keep={"n": n, "stages": C, "t": dev})
E.route_grid(tb, {})  # warm-up
cands = E.route_grid(tb, {})
rst = dict(E.last_stats)

# unique rows per stage (the reference's row cache key: stage + the workload's 5 doubles)
keys = ("arrival_rate", "mean_input_tokens", "mean_output_tokens", "p95_input_tokens", "p95_output_tokens")
rows = [dict() for _ in range(C)]
for c in cands:
    for i in range(C):
        w = c["stage_workloads"][i]
        if w["arrival_rate"] > 0:
            rows[i][tuple(w[k] for k in keys)] = w

report = {"config": W.__dict__.get("CONFIGS", {}).get(name, {}).get("models", None), "requests": n, "stages": C,
          "total_gpus": N, "candidates": len(cands),
          "routing": {"ms_route": rst["ms_route"], "ms_quality": rst["ms_quality"], "ms_k1": rst["ms_k1"],
                      "k1_GBps": rst["k1_bytes"] / rst["ms_k1"] / 1e6 if rst["ms_k1"] else None,
                      "ms_total_route_grid": rst["ms_total"]},
          "stages_detail": [], "kind": "extrapolated", "waves_per_row": M}
E.set_option("pilot", 0)
total_s = rst["ms_total"] / 1000.0
for i in range(C):
    if not rows[i]:
        continue
    model = cfg["models"][i]
    wl = sorted(rows[i].values(), key=lambda w: w["arrival_rate"])
    rep_w = wl[len(wl) // 2]  # the median-rate workload of this stage
    E.set_option("max_waves", 1)
    E.set_option("wave_stride", 1)
    E.row(cfg["hardware"], cfg["cost_model"], model, rep_w, N)
    probe = dict(E.last_stats)
    waves_total = max(1, probe["waves_total"])
    stride = max(1, waves_total // M)
    E.set_option("max_waves", M)
    E.set_option("wave_stride", stride)
    t1 = time.time()
    E.row(cfg["hardware"], cfg["cost_model"], model, rep_w, N)
    wall = time.time() - t1
    st = dict(E.last_stats)
    ms = st["ms_total"]  # host wall of the row call: filter waves + K4 + bookkeeping
    rate = st["plans_in_waves"] / (ms / 1000.0) if ms > 0 else None
    plans = st["plans_enumerated"]
    est_row_s = plans / rate if rate else 0.0
    stage_s = est_row_s * len(rows[i])
    total_s += stage_s
    report["stages_detail"].append({
        "stage": i, "model": model["id"], "unique_rows": len(rows[i]), "plans_per_row": plans,
        "sampled_workload": rep_w, "waves_total": st["waves_total"], "waves_run": st["waves_run"],
        "wave_stride": stride, "plans_sampled": st["plans_in_waves"], "plans_stable_sampled": st["plans_stable"],
        "plans_simulated_sampled": st["plans_simulated_full"] + st["plans_pruned"],
        "request_steps_sampled": st["request_steps"], "ms_row_call_sampled": ms, "ms_k4_sampled": st["ms_k4"],
        "wall_s_sampled": wall, "plans_per_s": rate,
        "request_steps_per_s": st["request_steps"] / (st["ms_k4"] / 1000.0) if st["ms_k4"] > 0 else None,
        "est_row_s": est_row_s, "est_stage_s": stage_s})
    print(json.dumps(report["stages_detail"][-1]), flush=True)
E.set_option("max_waves", 0)
E.set_option("wave_stride", 1)
report["est_sweep_s_1gpu"] = total_s
report["est_sweep_s_8gpu_ideal"] = total_s / 8.0
report["plans_per_sweep"] = int(sum(d["plans_per_row"] * d["unique_rows"] for d in report["stages_detail"]))
report["note"] = ("rates measured on sampled waves (pilot off, bounds from the sampled waves only); sweep time "
                  "EXTRAPOLATED as sum over unique rows of plans / stage rate; the reference CPU planner cannot "
                  "materialise the plan sets at N=128 (~3e12 plans per small-model row)")
print(json.dumps({k: v for k, v in report.items() if k != "stages_detail"}), flush=True)
if out_path:
    with open(out_path, "w") as f:
        json.dump(report, f, indent=1)
