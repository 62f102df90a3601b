"""Wall time of the unmodified reference planner's outerplan::sweep (oracle/_ref)
on the bench configurations, on this host's cores, at 1 thread and at all
threads (CASCADE_PLANNER_THREADS).  Traces come from the reference's own
generator.  C3's complete run is tools/make_c3_golden.py (1,852.8 s on 16 threads).

    python tools/reference_cpu_times.py C1,C2 [out.json]
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

names = (sys.argv[1] if len(sys.argv) > 1 else "C1,C2").split(",")
out = sys.argv[2] if len(sys.argv) > 2 else None
if os.environ.get("_REF_CHILD"):
    from oracle import refpy
    from paper_2506_04203_b200 import workloads as W
    name = os.environ["_REF_CHILD"]
    t = W.build_trace(name, refpy.generate_trace)
    cfg, N = W.planner_config(name, t["scores"])
    t0 = time.time()
    r = refpy.sweep(t, cfg, N)
    print(json.dumps({"config": name, "sweep_s": time.time() - t0,
                      "evaluations": len(r["result"]["evaluations"]),
                      "threads": int(os.environ["CASCADE_PLANNER_THREADS"])}))
    sys.exit(0)
res = []
cores = os.cpu_count() or 1
for name in names:
    for th in sorted({1, cores}):
        if name == "C2" and th == 1:
            continue  # ~50 min on one thread: the survey measured 8 threads
        env = dict(os.environ, _REF_CHILD=name, CASCADE_PLANNER_THREADS=str(th))
        p = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True, timeout=7200)
        line = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else json.dumps({"config": name, "error": p.stderr[-500:]})
        print(line, flush=True)
        res.append(json.loads(line))
doc = {"host_cores": cores, "runs": res,
       "C3_full_sweep": {"sweep_s": 1852.755475282669, "threads": 16, "source": "tests/golden/c3_full.json"}}
if out:
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
