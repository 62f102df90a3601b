"""K2 quality forms on a large trace (cg_route_grid, default decile grid):
  python tools/quality_probe.py C5 [reps]
Times ms_quality for the block-parallel exact form (1) and the one-chain form
(0) and checks that every candidate's quality is bit-identical."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
from paper_2506_04203_b200 import engine as eng, workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs(name)]
t = eng.concat_traces(parts) if len(parts) > 1 else parts[0]
C = t["scores"].shape[0]
E = eng.Engine(0)
dev = {k: torch.from_numpy(np.ascontiguousarray(t[k])).cuda() for k in t}
tb = eng.TraceBuffers(dev["arrival_s"].data_ptr(), dev["input_tokens"].data_ptr(), dev["output_tokens"].data_ptr(),
                      dev["scores"].data_ptr(), on_device=True, keep={"n": t["arrival_s"].shape[0], "stages": C, "t": dev})
res = {}
for form in (1, 0):
    E.set_option("quality_form", form)
    ms = []
    for rep in range(reps):
        r = E.route_grid(tb, {})
        ms.append(E.last_stats["ms_quality"])
        route_ms = E.last_stats["ms_route"]
    res[form] = r
    print(json.dumps({"config": name, "quality_form": form, "n": int(t["arrival_s"].shape[0]), "candidates": len(r),
                      "ms_quality": ms, "ms_route": route_ms, "quality_blocks": E.last_stats["quality_blocks"],
                      "quality_blocks_seq": E.last_stats["quality_blocks_seq"]}), flush=True)
q1 = np.array([c["quality"] for c in res[1]])
q0 = np.array([c["quality"] for c in res[0]])
print(json.dumps({"bit_identical": bool(np.array_equal(q1.view(np.uint64), q0.view(np.uint64)))}))
