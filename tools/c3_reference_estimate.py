"""Reference CPU time of the C3 plan search (3-model Llama 8B->70B->405B,
1M-request trace, 64-GPU pool), extrapolated -- the full run takes hours.

Measured on this host with the compiled reference (oracle/_ref, all threads):
  * route_trace on the 1M trace (one call; the sweep makes 121 + 3);
  * StageEvaluator::row of the 8B and 70B models at N = 32 (490,772 and
    112,564 plans), on the C3 all-accept / stage-1 workloads -> plans/s.
The reference's cost is its queueing simulations: one per STABLE plan (the
unstable ones are rejected by an O(S) test).  Its simulations/s is measured
on those rows (the stable count of each row comes from the GPU engine's
identical filter) and applied to the C3 sweep's exact stable-plan count.
Dispatch cost per simulation grows with dp, and dp is larger at N = 64, so
this underestimates the reference: a lower bound.

  python tools/c3_reference_estimate.py > profiles/round1_c3_reference_estimate.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
os.environ.setdefault("CASCADE_PLANNER_THREADS", str(os.cpu_count() or 1))
from paper_2506_04203_b200 import engine as eng, workloads as W
from oracle import refpy

parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs("C3")]
t = eng.concat_traces(parts)
cfg, N = W.planner_config("C3", t["scores"])
C = t["scores"].shape[0]
t0 = time.perf_counter()
r_all = refpy.route(t, [0.0] * (C - 1), [True] * C)["result"]
route_s = time.perf_counter() - t0
r_mid = refpy.route(t, [101.0] + [0.0] * (C - 2), [True] * C)["result"]   # everything escalated once
rates = {}
for stage, wl, name in ((0, r_all["stage_workloads"][0], "8B"), (1, r_mid["stage_workloads"][1], "70B")):
    t0 = time.perf_counter()
    row = refpy.row(cfg["hardware"], cfg["cost_model"], cfg["models"][stage], wl, 32)
    el = time.perf_counter() - t0
    rates[name] = {"budget": 32, "seconds": el}
E = eng.Engine(0)
for stage, wl, name in ((0, r_all["stage_workloads"][0], "8B"), (1, r_mid["stage_workloads"][1], "70B")):
    E.row(cfg["hardware"], cfg["cost_model"], cfg["models"][stage], wl, 32)
    rates[name]["stable_plans"] = E.last_stats["plans_stable"]
    rates[name]["sims_per_s"] = rates[name]["stable_plans"] / rates[name]["seconds"]
E.sweep(t, cfg["models"], cfg["hardware"], cfg["cost_model"], N, cfg["sweep"])
st = E.last_stats
gpu_ms = st["ms_total"]
# plan-space sizes (exact counts of the reference recursion)
plans_n32 = {"8B": 490772, "70B": 112564}
plans_n64 = {"8B": 393136346, "70B": 63673523, "405B": 586}
rows = {"8B": 1, "70B": 11, "405B": st["unique_rows"] - 12}
for k in rates:
    rates[k]["plans_per_s"] = plans_n32[k] / rates[k]["seconds"]
sims_per_s = max(rates["8B"]["sims_per_s"], rates["70B"]["sims_per_s"])  # the faster (optimistic) rate
est = st["plans_stable"] / sims_per_s + (st["candidates"] + 3) * route_s
print(json.dumps({
    "workload": "C3: Llama 8B->70B->405B, 1M-request bursty trace, 64-GPU pool, default decile grid",
    "kind": "extrapolated lower bound (reference rates measured at N=32, dp grows with N)",
    "host_threads": refpy.max_threads(), "route_trace_s": route_s, "row_rates": rates,
    "rows_by_model": rows, "plans_per_row_n64": plans_n64,
    "gpu_plans_enumerated": st["plans_enumerated"], "stable_plans_in_sweep": st["plans_stable"],
    "reference_sims_per_s_used": sims_per_s, "gpu_sweep_ms": gpu_ms,
    "reference_sweep_s_estimate": est, "speedup_estimate": est / (gpu_ms / 1e3)}, indent=1))
