"""Sweep time vs filter-wave size (option wave_plans, 2^20 plans per wave).
python tools/wave_probe.py C2 16,32,64"""
import json, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2506_04203_b200 import engine as eng, workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
sizes = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "16,64").split(",")]
parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs(name)]
t = eng.concat_traces(parts) if len(parts) > 1 else parts[0]
cfg, N = W.planner_config(name, t["scores"])
E = eng.Engine(0)
ref = None
for w in sizes:
    E.set_option("wave_plans", w)
    for rep in range(2):
        r = E.sweep(t, cfg["models"], cfg["hardware"], cfg["cost_model"], N, cfg["sweep"])
    st = E.last_stats
    same = ref is None or json.dumps(r, sort_keys=True) == ref
    ref = ref or json.dumps(r, sort_keys=True)
    print(json.dumps({"wave_plans": w, "identical": same, **{k: round(st[k], 2) if isinstance(st[k], float) else st[k]
          for k in ("ms_total", "ms_k4", "request_steps", "plans_pruned", "plans_bound_skipped", "gpu_launches")}}), flush=True)
