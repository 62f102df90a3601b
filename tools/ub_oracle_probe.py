"""Diagnostic: how much of K4's work is due to bounds that are not yet tight?
Runs the sweep twice; the second run's K4 bounds start at the exact final
rows (option ub_oracle).  Results must be identical either way."""
import json, os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2506_04203_b200 import engine as eng, workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs(name)]
t = eng.concat_traces(parts) if len(parts) > 1 else parts[0]
cfg, N = W.planner_config(name, t["scores"])
E = eng.Engine(0)
E.set_option("ub_oracle", 1)
res = []
for rep in range(3):
    r = E.sweep(t, cfg["models"], cfg["hardware"], cfg["cost_model"], N, cfg["sweep"])
    st = E.last_stats
    res.append(r)
    print(json.dumps({k: st[k] for k in ("ms_total", "ms_k4", "request_steps", "plans_simulated_full",
                                         "plans_pruned", "plans_bound_skipped", "plans_seeded")}), flush=True)
print("identical:", json.dumps(res[0], sort_keys=True) == json.dumps(res[2], sort_keys=True))
