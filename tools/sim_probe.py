"""Validation simulator at scale: every Pareto-front plan of a sweep replayed
over the full trace on the GPU (one batch) vs the reference's sim::run on the
CPU (timed on a few plans), reports compared bit for bit.

  python tools/sim_probe.py [C2|C3] [reference plans]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from paper_2506_04203_b200 import engine as eng, workloads as W
from oracle import refpy
from parity_util import diff_json

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
nref = int(sys.argv[2]) if len(sys.argv) > 2 else 2
parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs(name)]
t = eng.concat_traces(parts) if len(parts) > 1 else parts[0]
cfg, N = W.planner_config(name, t["scores"])
E = eng.Engine(0)
res = E.sweep(t, cfg["models"], cfg["hardware"], cfg["cost_model"], N, cfg["sweep"])
plans = [p["plan_ref"] for p in res["front"]["points"]]
n = int(t["arrival_s"].shape[0])
for rep in range(2):
    t0 = time.perf_counter()
    reps = E.simulate_many(plans, t, cfg["models"], cfg["hardware"], cfg["cost_model"], {})
    wall = time.perf_counter() - t0
    print(json.dumps({"config": name, "requests": n, "plans": len(plans), "gpu_wall_s": wall,
                      "gpu_ms_engine": E.last_sim["ms_total"], "launches": E.last_sim["gpu_launches"]}), flush=True)
ref_s, same = 0.0, True
for i in range(min(nref, len(plans))):
    r = refpy.simulate(t, cfg, [plans[i]], {})
    ref_s += r["elapsed_s"]
    same &= not diff_json(reps[i], r["result"])
print(json.dumps({"reference_plans": min(nref, len(plans)), "reference_s": ref_s,
                  "reference_s_per_plan": ref_s / max(1, min(nref, len(plans))), "identical": same}))
