"""Times one full sweep of a named config on the GPU engine (host trace)."""
import sys, os, time, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2506_04203_b200 import engine as eng, workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
count = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
prunes = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs(name, count)]
t = eng.concat_traces(parts) if len(parts) > 1 else parts[0]
cfg, N = W.planner_config(name, t["scores"])
E = eng.Engine(0)
for kv in filter(None, os.environ.get("CG_OPTS", "").split(",")):  # e.g. CG_OPTS=k4_pack=4,pilot=0
    k, v = kv.split("=")
    E.set_option(k, int(v))
for prune in prunes:
    E.set_option("prune", prune)
    for rep in range(reps):
        t0 = time.time()
        res = E.sweep(t, cfg["models"], cfg["hardware"], cfg["cost_model"], N, cfg["sweep"])
        dt = time.time() - t0
        st = E.last_stats
        print(f"{name} prune={prune} rep={rep}: wall {dt:.3f}s evals={len(res['evaluations'])} front={len(res['front']['points'])}", flush=True)
        print("  ", json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in st.items()}), flush=True)
