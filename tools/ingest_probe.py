"""Trace ingest (cascade::read_trace_jsonl) at scale: the C3 1M-request trace
written by the reference writer, read by the GPU engine and by the reference
reader (CPU, oracle/_ref), bit-identity checked.

  python tools/ingest_probe.py [C3|C5] [reps]"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from paper_2506_04203_b200 import engine as eng, workloads as W
from oracle import refpy

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs(name)]
t = eng.concat_traces(parts) if len(parts) > 1 else parts[0]
n = int(t["arrival_s"].shape[0])
d = tempfile.mkdtemp()
path = os.path.join(d, "trace.jsonl")
refpy.write_trace_jsonl(t, path)
size = os.path.getsize(path)
E = eng.Engine(0)
for r in range(reps):
    t0 = time.perf_counter()
    got = E.read_trace_jsonl(path)
    wall = time.perf_counter() - t0
    st = E.last_ingest
    print(json.dumps({"config": name, "records": n, "bytes": size, "wall_s": wall, **st,
                      "GBps_total": size / (st["ms_total"] / 1e3) / 1e9}), flush=True)
t0 = time.perf_counter()
ref = refpy.read_trace_jsonl(path, n + 1)
ref_wall = time.perf_counter() - t0
same = all(np.array_equal(np.asarray(got[k]).view(np.uint64), np.asarray(ref[k]).view(np.uint64))
           for k in ("arrival_s", "input_tokens", "output_tokens", "scores"))
print(json.dumps({"reference_read_s": ref["elapsed_s"], "reference_wall_s": ref_wall, "bit_identical": same}))
