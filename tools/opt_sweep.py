"""Sweep time for values of one engine option.  python tools/opt_sweep.py C2 pilot_min_plans 0,4096"""
import json, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2506_04203_b200 import engine as eng, workloads as W

name, opt = sys.argv[1], sys.argv[2]
vals = [int(x) for x in sys.argv[3].split(",")]
parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs(name)]
t = eng.concat_traces(parts) if len(parts) > 1 else parts[0]
cfg, N = W.planner_config(name, t["scores"])
E = eng.Engine(0)
ref = None
for v in vals:
    E.set_option(opt, v)
    for rep in range(2):
        r = E.sweep(t, cfg["models"], cfg["hardware"], cfg["cost_model"], N, cfg["sweep"])
    st = E.last_stats
    same = ref is None or json.dumps(r, sort_keys=True) == ref
    ref = ref or json.dumps(r, sort_keys=True)
    print(json.dumps({opt: v, "identical": same, **{k: round(st[k], 2) if isinstance(st[k], float) else st[k]
          for k in ("ms_total", "ms_k4", "request_steps", "plans_simulated_full", "plans_pruned", "plans_seeded")}}), flush=True)
