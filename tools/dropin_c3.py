"""End-to-end C3 through the reference's own C++ pipeline with the engine
dropped in (oracle/_ref/dropin_check --gpu-only): cli::cmd_plan on the 1M-line
C3 JSONL trace (GPU ingest, sweep, output files) and outerplan::sweep through
the C++ binding on the parsed records (AoS -> SoA, pageable copies, result
rebuild).  The reference's CPU sweep of the same workload took 1,852.8 s on 16
threads (tests/golden/c3_full.json).

    python tools/dropin_c3.py [out.json]
"""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2506_04203_b200 import engine as eng, workloads as W  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else None
t = W.build_trace("C3", eng.generate_trace)
cfg, N = W.planner_config("C3", t["scores"])
d = tempfile.mkdtemp(prefix="dropin_c3_")
C = t["scores"].shape[0]
with open(os.path.join(d, "trace.jsonl"), "w") as f:
    arr, inp, outt, sc = t["arrival_s"], t["input_tokens"], t["output_tokens"], t["scores"]
    for r in range(arr.shape[0]):
        f.write(json.dumps({"arrival_s": float(arr[r]), "input_tokens": float(inp[r]),
                            "per_stage": [{"output_tokens": float(outt[i, r]), "score": float(sc[i, r])}
                                          for i in range(C)]}) + "\n")
with open(os.path.join(d, "config.json"), "w") as f:
    json.dump(cfg, f)
res = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "dropin_check"), os.path.join(d, "config.json"),
                      os.path.join(d, "trace.jsonl"), "0", os.path.join(d, "out"), "0", "--gpu-only", "3"],
                     capture_output=True, text=True, timeout=1800)
line = res.stdout.strip().splitlines()[-1] if res.stdout.strip() else ""
rep = json.loads(line) if line else {"error": res.stderr[-2000:]}
rep["trace_bytes"] = os.path.getsize(os.path.join(d, "trace.jsonl"))
rep["reference_cpu_sweep_s"] = 1852.755475282669
print(json.dumps(rep))
if out:
    with open(out, "w") as f:
        json.dump(rep, f, indent=1)
