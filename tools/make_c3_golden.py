"""Full-size C3 parity fixture from the UNMODIFIED reference planner.

Runs cascade::outerplan::sweep of the compiled reference (oracle/_ref) on the
complete C3 workload -- 3-model Llama 8B -> 70B -> 405B cascade, the 1M-request
heterogeneous bursty trace from the reference's own cli::generate_trace, the
64-GPU pool, the default decile grid -- on all host threads, and writes the
whole SweepResult plus the measured wall time to tests/golden/c3_full.json.
tests/test_gpu_fullsize.py compares the engine's C3 sweep (the bench
workload) against it field by field.  Takes about an hour on 16 threads and
~30 GB of host memory (the reference materialises its plan sets), so it runs
once, on the GPU box's host:

    CASCADE_PLANNER_THREADS=16 python tools/make_c3_golden.py [out.json]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import refpy  # noqa: E402
from paper_2506_04203_b200 import workloads as W  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tests", "golden", "c3_full.json")
os.environ.setdefault("CASCADE_PLANNER_THREADS", str(os.cpu_count() or 1))
t0 = time.time()
trace = W.build_trace("C3", refpy.generate_trace)
cfg, N = W.planner_config("C3", trace["scores"])
gen_s = time.time() - t0
t1 = time.time()
res = refpy.sweep(trace, cfg, N)
wall = time.time() - t1
doc = {"name": "c3_full", "config_name": "C3", "trace_specs": W.trace_specs("C3"), "config": cfg,
       "total_gpus": N, "result": res["result"],
       "reference": {"sweep_wall_s": wall, "elapsed_s": res.get("elapsed_s"),
                     "threads": int(os.environ["CASCADE_PLANNER_THREADS"]), "host_cores": os.cpu_count(),
                     "trace_generation_s": gen_s}}
with open(out, "w") as f:
    json.dump(doc, f)
print(json.dumps({"out": out, "sweep_wall_s": wall, "evaluations": len(res["result"]["evaluations"])}))
