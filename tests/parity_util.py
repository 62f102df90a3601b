"""Shared helpers for the parity tests: seeded workloads and exact comparison
of engine results against the reference oracle (oracle/refpy.py)."""
from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2506_04203_b200 import engine as eng  # noqa: E402
from paper_2506_04203_b200 import workloads as W  # noqa: E402


def bits(x: float) -> int:
    return int(np.float64(x).view(np.uint64))


def diff_json(a, b, path="$", out=None, limit=20):
    """Exact structural diff; floats compared bit-for-bit (0.0 == -0.0 excepted)."""
    if out is None:
        out = []
    if len(out) >= limit:
        return out
    if isinstance(a, dict) and isinstance(b, dict):
        if set(a) != set(b):
            out.append(f"{path}: keys {sorted(a)} != {sorted(b)}")
            return out
        for k in a:
            diff_json(a[k], b[k], f"{path}.{k}", out, limit)
    elif isinstance(a, list) and isinstance(b, list):
        if len(a) != len(b):
            out.append(f"{path}: len {len(a)} != {len(b)}")
            return out
        for i, (x, y) in enumerate(zip(a, b)):
            diff_json(x, y, f"{path}[{i}]", out, limit)
    elif isinstance(a, bool) or isinstance(b, bool):
        if a != b:
            out.append(f"{path}: {a} != {b}")
    elif isinstance(a, (int, float)) and isinstance(b, (int, float)):
        if isinstance(a, float) or isinstance(b, float):
            fa, fb = float(a), float(b)
            if fa != fb and not (math.isnan(fa) and math.isnan(fb)):
                out.append(f"{path}: {fa!r} != {fb!r}")
        elif a != b:
            out.append(f"{path}: {a} != {b}")
    elif a != b:
        out.append(f"{path}: {a!r} != {b!r}")
    return out


def small_trace(count=1500, rate=1.0, scores=((60, 20), (85, 10)), seed=3, hetero=False):
    spec = W.trace_spec(count, rate, list(scores),
                        W.HETERO_IN if hetero else None, W.HETERO_OUT if hetero else None)
    return eng.generate_trace(spec, seed), spec


def parity_cases():
    """(name, trace, config, total_gpus) small enough for the CPU reference."""
    cases = []
    # 2-stage reference fixture cluster (test_outerplan.cpp small_cluster)
    t, _ = small_trace(800, 0.4, ((70, 25), (95, 3)), seed=11)
    hw = W.hardware(8)
    hw["gpus_per_node"] = 4
    cfg = {"hardware": hw, "models": [W.model_spec("small-7b", 1), W.model_spec("mid-70b", 2)],
           "cost_model": dict(W.DEFAULT_COST_MODEL, queueing_sim_requests=300), "sweep": {}}
    cases.append(("fixture2_default_grid", t, cfg, 8))
    # C1 shape at reduced size, explicit 12-point grid
    t, _ = small_trace(3000, 1.0, ((60, 20), (92, 5)), seed=1)
    cfg, _ = W.planner_config("C1", t["scores"], grid=12)
    cases.append(("c1_small", t, cfg, 16))
    # 3-stage C2 cascade, N=16, 6x6 grid
    t, _ = small_trace(4000, 2.0, ((60, 20), (80, 12), (92, 5)), seed=5)
    cfg, _ = W.planner_config("C2", t["scores"], grid=6)
    cfg["hardware"]["gpu_count"] = 16
    cases.append(("c2_small_n16", t, cfg, 16))
    return cases


def golden_trace(case):
    """Trace of a golden case: inline arrays or (spec, seed) via our generator."""
    if case.get("trace") is not None:
        return {k: np.asarray(v, dtype=np.float64) for k, v in case["trace"].items()}
    return eng.generate_trace(case["trace_spec"], case["seed"])
