"""K4 phase breakdown (development): runs a config's sweep on the profiling
build (CG_BUILD_VARIANT=prof, -DCG_K4_PROF) and prints, per one-lane-per-plan
kernel class, the warp cycles spent claiming plans, stepping, checking and
finishing, plus claim-round and SIMT-occupancy counts.

    CG_BUILD_VARIANT=prof python -m paper_2506_04203_b200.build   # once
    python tools/k4_prof_probe.py C3
"""
import ctypes
import json
import os
import sys

os.environ["CG_BUILD_VARIANT"] = "prof"
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2506_04203_b200 import engine as eng, workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs(name, None)]
t = eng.concat_traces(parts) if len(parts) > 1 else parts[0]
cfg, N = W.planner_config(name, t["scores"])
E = eng.Engine(0)
for kv in filter(None, os.environ.get("CG_OPTS", "").split(",")):
    k, v = kv.split("=")
    E.set_option(k, int(v))
L = eng.library()
L.cg_k4prof_read.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_uint64 * 64)()
E.sweep(t, cfg["models"], cfg["hardware"], cfg["cost_model"], N, cfg["sweep"])  # warm-up
L.cg_k4prof_reset()
E.sweep(t, cfg["models"], cfg["hardware"], cfg["cost_model"], N, cfg["sweep"])
L.cg_k4prof_read(buf)
st = E.last_stats
print(json.dumps({k: st[k] for k in ("ms_k4", "request_steps", "plans_pruned", "plans_bound_skipped",
                                     "plans_simulated_full")}))
names = {1: "claim_take", 12: "claim_setup", 2: "steps", 3: "check", 4: "finish"}
for ri, R in enumerate((4, 8, 16, 32)):
    p = list(buf[ri * 16:(ri + 1) * 16])
    tot = p[0]
    if not tot:
        continue
    trips = max(p[9], 1)
    out = {"R": R, "warps": p[11], "warp_cycles": tot,
           "share": {v: round(p[k] / tot, 3) for k, v in names.items()},
           "claim_rounds": p[5], "claim_iters": p[6], "lane_attempts": p[8], "takes": p[7],
           "trips": p[9], "simt_occupancy": round(p[10] / (32.0 * trips), 3),
           "cycles_per_trip_steps": round(p[2] / trips, 1),
           "cycles_per_claim_round": round((p[1] + p[12]) / max(p[5], 1), 1),
           "trips_per_claim_round": round(trips / max(p[5], 1), 2)}
    print(json.dumps(out), flush=True)
