"""A/B of engine options on full sweeps: results must be identical.
  python tools/opt_probe.py C2,C3 key=v1,v2"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2506_04203_b200 import engine as eng, workloads as W

key, vals = sys.argv[2].split("=")
for name in sys.argv[1].split(","):
    parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs(name)]
    t = eng.concat_traces(parts) if len(parts) > 1 else parts[0]
    cfg, N = W.planner_config(name, t["scores"])
    E = eng.Engine(0)
    ref = None
    for v in vals.split(","):
        E.set_option(key, int(v))
        for rep in range(2):
            r = E.sweep(t, cfg["models"], cfg["hardware"], cfg["cost_model"], N, cfg["sweep"])
        st = E.last_stats
        js = json.dumps(r, sort_keys=True)
        print(json.dumps({"cfg": name, key: int(v), "ms_k4": round(st["ms_k4"], 1), "ms_total": round(st["ms_total"], 1),
                          "steps": st["request_steps"], "pruned": st["plans_pruned"], "full": st["plans_simulated_full"],
                          "identical": None if ref is None else js == ref}), flush=True)
        ref = ref or js
