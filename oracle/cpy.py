"""TEST INFRASTRUCTURE ONLY: ctypes bindings to our plain-C restatement
(oracle/_ref/libcascade_oracle.so built from oracle/cascade_oracle.c), with
results converted to the reference's JSON schema so they compare directly
with oracle/refpy.py and the GPU engine."""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libcascade_oracle.so")
MAXS = 32
_lib = None


class CoHw(ctypes.Structure):
    _fields_ = [("gpu_count", ctypes.c_int), ("flops", ctypes.c_double), ("mem_bw", ctypes.c_double),
                ("mem_cap", ctypes.c_double), ("intra_bw", ctypes.c_double), ("inter_bw", ctypes.c_double),
                ("gpus_per_node", ctypes.c_int)]


class CoModel(ctypes.Structure):
    _fields_ = [("param_count", ctypes.c_double), ("bytes_per_param", ctypes.c_double),
                ("kv_bytes_per_token", ctypes.c_double), ("min_gpus", ctypes.c_int), ("stage_index", ctypes.c_int)]


class CoParams(ctypes.Structure):
    _fields_ = [("prefill_eff", ctypes.c_double), ("decode_eff", ctypes.c_double), ("bubble", ctypes.c_double),
                ("comm", ctypes.c_double), ("kv_frac", ctypes.c_double), ("n_req", ctypes.c_int),
                ("seed", ctypes.c_uint64)]


DEFAULTS = {"prefill_efficiency": 0.5, "decode_bw_efficiency": 0.7, "pipeline_bubble_factor": 0.1,
            "comm_overhead_per_stage": 0.002, "kv_memory_fraction": 0.9, "queueing_sim_requests": 2000,
            "queueing_sim_seed": 12345}


class OracleError(Exception):
    def __init__(self, code):
        super().__init__(f"oracle error code {code}")
        self.code = code


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(LIB_PATH)
    return _lib


def _hw(hw):
    return CoHw(int(hw["gpu_count"]), hw["flops_per_gpu"], hw["mem_bandwidth_per_gpu"], hw["mem_capacity_per_gpu"],
                hw["intra_node_bw"], hw["inter_node_bw"], int(hw["gpus_per_node"]))


def _model(m):
    return CoModel(m["param_count"], m["bytes_per_param"], m["kv_bytes_per_token"], int(m.get("min_gpus", 1)),
                   int(m["stage_index"]))


def _params(p):
    q = dict(DEFAULTS)
    q.update(p or {})
    return CoParams(q["prefill_efficiency"], q["decode_bw_efficiency"], q["pipeline_bubble_factor"],
                    q["comm_overhead_per_stage"], q["kv_memory_fraction"], int(q["queueing_sim_requests"]),
                    int(q["queueing_sim_seed"]))


def _P(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def legal_shapes(model, hw, params=None):
    """costmodel.cpp:92-116 (Python doubles are IEEE binary64: same arithmetic)."""
    q = dict(DEFAULTS)
    q.update(params or {})
    cands = []
    tp = 1
    while tp <= hw["gpus_per_node"]:
        for pp in range(1, 9):
            cands.append((tp, pp))
        tp *= 2
    cands.sort(key=lambda s: (-s[0] * s[1], -s[0]))
    out = []
    w = model["param_count"] * model["bytes_per_param"]
    for tp, pp in cands:
        g = float(tp * pp)
        if w / g > hw["mem_capacity_per_gpu"]:
            continue
        if q["kv_memory_fraction"] * (g * hw["mem_capacity_per_gpu"] - w) >= model["kv_bytes_per_token"] * 1.0:
            out.append((tp, pp))
    return out


def _plan_json(counts, shapes):
    if not any(counts):
        return None
    reps = []
    for s, c in enumerate(counts[: len(shapes)]):
        reps += [{"tp": shapes[s][0], "pp": shapes[s][1]}] * int(c)
    return {"replicas": reps, "gpus_used": sum(r["tp"] * r["pp"] for r in reps)}


def _trace(t):
    arr = np.ascontiguousarray(t["arrival_s"], dtype=np.float64)
    inp = np.ascontiguousarray(t["input_tokens"], dtype=np.float64)
    out = np.ascontiguousarray(t["output_tokens"], dtype=np.float64)
    sc = np.ascontiguousarray(t["scores"], dtype=np.float64)
    return arr, inp, out, sc, arr.shape[0], sc.shape[0]


def route(trace, thresholds, deployed):
    arr, inp, out, sc, n, c = _trace(trace)
    h = np.ascontiguousarray(list(thresholds) + [0.0], dtype=np.float64)
    dep = np.ascontiguousarray([1 if d else 0 for d in deployed], dtype=np.int32)
    ratios = np.zeros(c)
    wl = np.zeros(5 * c)
    q = ctypes.c_double()
    acc = np.zeros(max(n, 1), dtype=np.int32)
    L = lib()
    L.co_route.restype = ctypes.c_int
    rc = L.co_route(_P(arr), _P(inp), _P(out), _P(sc), ctypes.c_int64(n), c, _P(h), _P(dep), _P(ratios), _P(wl),
                    ctypes.byref(q), _P(acc))
    if rc != -1:
        raise OracleError(rc)
    keys = ["arrival_rate", "mean_input_tokens", "mean_output_tokens", "p95_input_tokens", "p95_output_tokens"]
    return {"ratios": ratios.tolist(), "quality": q.value,
            "stage_workloads": [dict(zip(keys, wl[5 * i: 5 * i + 5].tolist())) for i in range(c)],
            "per_request_accept_stage": acc[:n].tolist()}


def row(hw, params, model, workload, max_budget):
    w = np.array([workload[k] for k in ("arrival_rate", "mean_input_tokens", "mean_output_tokens",
                                        "p95_input_tokens", "p95_output_tokens")], dtype=np.float64)
    lat = np.zeros(max_budget + 1)
    plans = np.zeros((max_budget + 1) * MAXS, dtype=np.int32)
    ns = ctypes.c_int()
    shapes = np.zeros(2 * MAXS, dtype=np.int32)
    hwc, mc, pc = _hw(hw), _model(model), _params(params)
    L = lib()
    L.co_row.restype = ctypes.c_int
    rc = L.co_row(ctypes.byref(mc), _P(w), ctypes.byref(hwc), ctypes.byref(pc), int(max_budget), _P(lat),
                  _P(plans), ctypes.byref(ns), _P(shapes))
    if rc != -1:
        raise OracleError(rc)
    sh = [(int(shapes[2 * s]), int(shapes[2 * s + 1])) for s in range(ns.value)]
    return {"latency": [None if math.isinf(v) else float(v) for v in lat],
            "plan": [_plan_json(plans[f * MAXS:(f + 1) * MAXS].tolist(), sh) for f in range(max_budget + 1)]}


def row_shard(hw, params, model, workload, max_budget, plan_lo, plan_hi):
    """Per-budget best over plan indices [plan_lo, plan_hi): (lat_bits u64[N+1]
    with ~0 = none, plan_index u64[N+1] with ~0 = none, total_plans)."""
    w = np.array([workload[k] for k in ("arrival_rate", "mean_input_tokens", "mean_output_tokens",
                                        "p95_input_tokens", "p95_output_tokens")], dtype=np.float64)
    lat = np.zeros(max_budget + 1)
    idx = np.zeros(max_budget + 1, dtype=np.int64)
    total = ctypes.c_int64()
    hwc, mc, pc = _hw(hw), _model(model), _params(params)
    L = lib()
    L.co_row_shard.restype = ctypes.c_int
    rc = L.co_row_shard(ctypes.byref(mc), _P(w), ctypes.byref(hwc), ctypes.byref(pc), int(max_budget),
                        ctypes.c_int64(plan_lo), ctypes.c_int64(plan_hi), _P(lat), _P(idx), ctypes.byref(total))
    if rc != -1:
        raise OracleError(rc)
    bits = lat.view(np.uint64).copy()
    bits[idx < 0] = np.uint64(0xFFFFFFFFFFFFFFFF)
    pidx = idx.astype(np.uint64)
    pidx[idx < 0] = np.uint64(0xFFFFFFFFFFFFFFFF)
    return bits, pidx, total.value


def solve(table, total_gpus):
    n = int(table["gpu_budget"])
    ent = np.array([[math.inf if v is None else v for v in r] for r in table["entries"]], dtype=np.float64)
    c = ent.shape[0]
    al = np.zeros(max(c, 1), dtype=np.int32)
    L = ctypes.c_double()
    lib().co_solve.restype = ctypes.c_int
    rc = lib().co_solve(_P(np.ascontiguousarray(ent)), c, n, int(total_gpus), _P(al), ctypes.byref(L))
    if rc != -1:
        raise OracleError(rc)
    return {"allocations": al[:c].tolist(), "objective_L": L.value,
            "per_stage_latency": [float(ent[i, al[i]]) for i in range(c)]}


def sweep(trace, config, total_gpus):
    arr, inp, out, sc, n, c = _trace(trace)
    models = (CoModel * c)(*[_model(m) for m in config["models"]])
    hwc, pc = _hw(config["hardware"]), _params(config.get("cost_model"))
    sw = config.get("sweep") or {}
    grid = sw.get("threshold_grid") or []
    sizes = np.array([len(g) for g in grid] + [0], dtype=np.int64)
    vals = np.array([v for g in grid for v in g] + [0.0], dtype=np.float64)
    ncand = 1
    for g in grid:
        ncand *= len(g)
    if not grid:
        ncand = 11 ** max(c - 1, 0)
    W = int(sw.get("weight_count", 9))
    ecand = np.zeros(ncand, dtype=np.int64)
    eL = np.zeros(ncand)
    eQ = np.zeros(ncand)
    ealloc = np.zeros(ncand * c, dtype=np.int32)
    eplans = np.zeros(ncand * c * MAXS, dtype=np.int32)
    weights = np.zeros(2 * max(W, 1))
    sel = np.zeros(max(W, 1), dtype=np.int32)
    front = np.zeros(ncand, dtype=np.int64)
    skipped = np.zeros(ncand, dtype=np.int64)
    counts = np.zeros(4, dtype=np.int64)
    z = np.zeros(2)
    L = lib()
    L.co_sweep.restype = ctypes.c_int
    rc = L.co_sweep(_P(arr), _P(inp), _P(out), _P(sc), ctypes.c_int64(n), c, models, ctypes.byref(hwc),
                    ctypes.byref(pc), int(total_gpus), len(grid), _P(sizes), _P(vals),
                    ctypes.c_double(float(sw.get("weight_ratio_min", 0.1))),
                    ctypes.c_double(float(sw.get("weight_ratio_max", 10.0))), W, _P(ecand), _P(eL), _P(eQ),
                    _P(ealloc), _P(eplans), _P(weights), _P(sel), _P(front), _P(skipped), _P(counts), _P(z))
    if rc != -1:
        raise OracleError(rc)
    E, F, S, Wn = (int(v) for v in counts)
    if not grid:  # reconstruct the default grid the C code used
        grid = []
        for d in range(c - 1):
            s = np.sort(np.asarray(trace["scores"][d], dtype=np.float64))
            vals_d = {0.0, 101.0}
            for q in range(1, 10):
                r = min(max(int(math.ceil((q / 10.0) * float(n))), 1), n)
                vals_d.add(float(s[r - 1]))
            grid.append(sorted(vals_d))
    shapes = [legal_shapes(m, config["hardware"], config.get("cost_model")) for m in config["models"]]

    def thresholds_of(cand):
        rem = int(cand)
        h = [0.0] * (c - 1)
        for d in range(c - 2, -1, -1):
            h[d] = float(grid[d][rem % len(grid[d])])
            rem //= len(grid[d])
        return h

    # ratios via route (C oracle) per evaluation
    evals = []
    for e in range(E):
        h = thresholds_of(ecand[e])
        r = route(trace, h, [True] * c)
        plans = []
        for i in range(c):
            cnts = eplans[(e * c + i) * MAXS:(e * c + i + 1) * MAXS].tolist()
            plans.append(_plan_json(cnts, shapes[i]) if ealloc[e * c + i] > 0 else None)
        th = {"thresholds": h}
        evals.append({"latency_s": float(eL[e]), "quality": float(eQ[e]), "thresholds": th,
                      "plan_ref": {"allocations": ealloc[e * c:(e + 1) * c].tolist(), "plans": plans,
                                   "thresholds": th, "predicted_max_p95_s": float(eL[e]),
                                   "predicted_quality": float(eQ[e]), "processing_ratios": r["ratios"]}})
    return {"front": {"points": [evals[int(i)] for i in front[:F]]}, "evaluations": evals,
            "weights": [{"lambda1": float(weights[2 * k]), "lambda2": float(weights[2 * k + 1])} for k in range(Wn)],
            "weight_selection": sel[:Wn].tolist(), "utopia": {"z1_star": float(z[0]), "z2_star": float(z[1])},
            "skipped": [{"thresholds": thresholds_of(skipped[s])} for s in range(S)]}


CENSUS_BIN_LIMITS = [4, 8, 16, 32, 64, 128, 256, None]


def row_census(hw, params, model, workload, max_budget, threads=None):
    """Plans the reference enumerates for one row and how many pass its
    stability test (= the queueing simulations StageEvaluator::row runs,
    costmodel.cpp:366-376), binned by replica count.  No simulation."""
    w = np.array([workload[k] for k in ("arrival_rate", "mean_input_tokens", "mean_output_tokens",
                                        "p95_input_tokens", "p95_output_tokens")], dtype=np.float64)
    out = np.zeros(18, dtype=np.int64)
    hwc, mc, pc = _hw(hw), _model(model), _params(params)
    L = lib()
    L.co_row_census.restype = ctypes.c_int
    rc = L.co_row_census(ctypes.byref(mc), _P(w), ctypes.byref(hwc), ctypes.byref(pc), int(max_budget),
                         int(threads or os.cpu_count() or 1), _P(out))
    if rc != -1:
        raise OracleError(rc)
    bins = [{"dp_max": lim, "stable": int(out[2 + b]), "sum_dp": int(out[10 + b])}
            for b, lim in enumerate(CENSUS_BIN_LIMITS)]
    return {"plans": int(out[0]), "stable": int(out[1]), "bins": bins}
