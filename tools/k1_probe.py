"""Routing/aggregation pass (K1) on a large trace, for the HBM roofline:
one cg_route over the C5 trace (10M requests, 4 stages) and the C3 trace."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from paper_2506_04203_b200 import engine as eng, workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs(name)]
t = eng.concat_traces(parts) if len(parts) > 1 else parts[0]
C = t["scores"].shape[0]
E = eng.Engine(0)
import torch
dev = {k: torch.from_numpy(np.ascontiguousarray(t[k])).cuda() for k in t}
tb = eng.TraceBuffers(dev["arrival_s"].data_ptr(), dev["input_tokens"].data_ptr(), dev["output_tokens"].data_ptr(),
                      dev["scores"].data_ptr(), on_device=True, keep={"n": t["arrival_s"].shape[0], "stages": C, "t": dev})
for rep in range(3):
    r = E.route_trace(tb, [60.0] * (C - 1), [True] * C)
print(name, "n", t["arrival_s"].shape[0], "C", C, "ratios", [round(x, 4) for x in r["ratios"]], flush=True)
