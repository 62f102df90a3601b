import sys, os, json, time
sys.path.insert(0, '.')
from paper_2506_04203_b200 import engine as eng, workloads as W
for name in sys.argv[1].split(","):
    parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs(name)]
    t = eng.concat_traces(parts) if len(parts) > 1 else parts[0]
    cfg, N = W.planner_config(name, t["scores"])
    E = eng.Engine(0)
    ref = None
    for pack in (0, 1, 2):
        E.set_option("k4_pack", pack)
        for rep in range(2):
            r = E.sweep(t, cfg["models"], cfg["hardware"], cfg["cost_model"], N, cfg["sweep"])
        st = E.last_stats
        same = None if ref is None else json.dumps(r, sort_keys=True) == ref
        ref = ref or json.dumps(r, sort_keys=True)
        print(json.dumps({"cfg": name, "pack": pack, "ms_k4": round(st["ms_k4"], 1), "ms_total": round(st["ms_total"], 1),
                          "overflow": st["plans_overflow"], "identical": same}), flush=True)
