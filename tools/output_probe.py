"""Output serialisation at scale: sweep.json / front.json of a full sweep
rendered by the GPU writer vs the reference's nlohmann dump(2) of the same
result (oracle/_ref), byte-compared and timed.

  python tools/output_probe.py [C2|C4] [reps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2506_04203_b200 import engine as eng, workloads as W
from oracle import refpy

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs(name)]
t = eng.concat_traces(parts) if len(parts) > 1 else parts[0]
cfg, N = W.planner_config(name, t["scores"])
E = eng.Engine(0)
t0 = time.perf_counter()
res = E.sweep(t, cfg["models"], cfg["hardware"], cfg["cost_model"], N, cfg["sweep"])
sweep_s = time.perf_counter() - t0
for r in range(reps):
    t0 = time.perf_counter()
    E.sweep(t, cfg["models"], cfg["hardware"], cfg["cost_model"], N, cfg["sweep"], raw=True, files=True)
    both = time.perf_counter() - t0
    ms_sweep = E.last_stats["ms_total"]
    print(json.dumps({"config": name, "evaluations": len(res["evaluations"]), "sweep_plus_files_s": both,
                      "sweep_ms": ms_sweep, "files_ms": both * 1e3 - ms_sweep,
                      "sweep_json_bytes": len(E.last_files["sweep.json"])}), flush=True)
ref = refpy.dump_sweep(res)
print(json.dumps({"reference_dump_s": ref["elapsed_s"],
                  "sweep_json_identical": ref["sweep.json"] == E.last_files["sweep.json"],
                  "front_json_identical": ref["front.json"] == E.last_files["front.json"]}))
