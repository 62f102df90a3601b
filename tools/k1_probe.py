"""Routing phase (K1-K3 + K2) over a large trace for the HBM roofline:
cg_route_grid with the default decile grid over the C3 / C5 traces.

  python tools/k1_probe.py C5 3 [forms]   forms: comma list of engine k1_form values
Every form's routing result must be identical (checked here)."""
import os, sys, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from paper_2506_04203_b200 import engine as eng, workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
forms = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]
parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs(name)]
t = eng.concat_traces(parts) if len(parts) > 1 else parts[0]
C = t["scores"].shape[0]
E = eng.Engine(0)
import torch
dev = {k: torch.from_numpy(np.ascontiguousarray(t[k])).cuda() for k in t}
tb = eng.TraceBuffers(dev["arrival_s"].data_ptr(), dev["input_tokens"].data_ptr(), dev["output_tokens"].data_ptr(),
                      dev["scores"].data_ptr(), on_device=True, keep={"n": t["arrival_s"].shape[0], "stages": C, "t": dev})
first = None
for form in forms:
    E.set_option("k1_form", form)
    for rep in range(reps):
        res = E.route_grid(tb, {})
        st = E.last_stats
        same = None
        if first is None:
            first = res
        else:
            same = json.dumps(res, sort_keys=True) == json.dumps(first, sort_keys=True)
        print(json.dumps({"config": name, "k1_form": form, "n": int(t["arrival_s"].shape[0]), "C": C,
                          "candidates": len(res), "ms_k1": st["ms_k1"], "k1_bytes": st["k1_bytes"],
                          "k1_GBps": st["k1_bytes"] / st["ms_k1"] / 1e6 if st["ms_k1"] else None,
                          "ms_route": st["ms_route"], "ms_quality": st["ms_quality"], "ms_total": st["ms_total"],
                          "identical_to_first_form": same}), flush=True)
