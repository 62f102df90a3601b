"""Generates tests/golden/*.json from the UNMODIFIED reference planner
(oracle/_ref/libcascade_ref.so, built from /root/reference sources by
oracle/Makefile).  Traces are stored as generator specs + seeds (our
cg_generate_trace is bit-identical to the reference generator, which
tests/test_abi.py checks), so fixtures stay small.

    python tools/make_golden.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import refpy  # noqa: E402
from paper_2506_04203_b200 import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def trace_of(spec, seed):
    return refpy.generate_trace(spec, seed)


def sweep_case(name, spec, seed, cfg_fn, N, requirement=None, inline=None):
    t = trace_of(spec, seed) if inline is None else {k: __import__("numpy").asarray(v, dtype=float)
                                                     for k, v in inline.items()}
    cfg = cfg_fn(t)
    res = refpy.sweep_raw(t, cfg, N)
    case = {"name": name, "trace_spec": spec, "seed": seed, "config": cfg, "total_gpus": N}
    if inline is not None:
        case["trace"] = inline
    if res["ok"]:
        case["result"] = res["result"]
        if requirement:
            case["requirement"] = requirement
            case["files"] = refpy.plan_outputs(t, cfg, N, requirement)
    else:
        case["error"] = {"code": res["code"], "message": res["message"]}
    return case


def main():
    os.makedirs(OUT, exist_ok=True)
    cases = []
    hw8 = W.hardware(8)
    hw8["gpus_per_node"] = 4
    fast = dict(W.DEFAULT_COST_MODEL, queueing_sim_requests=300)
    two = [W.model_spec("small-7b", 1), W.model_spec("mid-70b", 2)]
    three = [W.model_spec("small-7b", 1), W.model_spec("mid-70b", 2), W.model_spec("large-671b-int4", 3)]

    s = W.trace_spec(800, 0.4, [(70, 25), (95, 3)])
    cases.append(sweep_case("fixture2_default_grid", s, 11,
                            lambda t: {"hardware": hw8, "models": two, "cost_model": fast, "sweep": {}}, 8,
                            {"min_quality": 80.0}))
    s = W.trace_spec(400, 0.4, [(75, 10)])
    cases.append(sweep_case("single_stage", s, 5,
                            lambda t: {"hardware": hw8, "models": [W.model_spec("small-7b", 1)],
                                       "cost_model": fast, "sweep": {}}, 8, {"max_latency": 100.0}))
    s = W.trace_spec(3000, 1.0, [(60, 20), (92, 5)])
    cases.append(sweep_case("c1_small_grid12", s, 1,
                            lambda t: W.planner_config("C1", t["scores"], grid=12)[0], 16,
                            {"min_quality": 85.0}))
    s = W.trace_spec(1500, 1.5, [(60, 20), (80, 12), (92, 5)])
    cases.append(sweep_case("three_stage_fixture_n16", s, 7,
                            lambda t: {"hardware": W.hardware(16), "models": three,
                                       "cost_model": dict(W.DEFAULT_COST_MODEL, queueing_sim_requests=500),
                                       "sweep": {"threshold_grid": W.explicit_grid(t["scores"], 5),
                                                 "weight_count": 5}}, 16))
    s = W.trace_spec(2000, 2.0, [(60, 20), (80, 12), (92, 5)], W.HETERO_IN, W.HETERO_OUT)
    cases.append(sweep_case("c3_hetero_small_default_grid", s, 3,
                            lambda t: {"hardware": W.hardware(16),
                                       "models": W.cascade(["llama-3-8b", "llama-3-70b", "llama-3.1-405b"]),
                                       "cost_model": dict(W.DEFAULT_COST_MODEL, queueing_sim_requests=800),
                                       "sweep": {}}, 16))
    # explicit grid with duplicates and unsorted values (kept in given order)
    s = W.trace_spec(1000, 0.8, [(60, 20), (92, 5)])
    cases.append(sweep_case("unsorted_duplicate_grid", s, 9,
                            lambda t: {"hardware": hw8, "models": two, "cost_model": fast,
                                       "sweep": {"threshold_grid": [[80.0, 0.0, 55.5, 80.0, 101.0, 30.0]],
                                                 "weight_count": 4, "weight_ratio_min": 0.5,
                                                 "weight_ratio_max": 4.0}}, 8))
    # every candidate infeasible -> INFEASIBLE_PROBLEM; smallest model unservable -> INFEASIBLE
    s = W.trace_spec(500, 50.0, [(60, 20), (92, 5)])
    cases.append(sweep_case("utopia_infeasible", s, 2,
                            lambda t: {"hardware": hw8, "models": two, "cost_model": fast, "sweep": {}}, 8))
    # every candidate infeasible (grid forces both stages live, N too small)
    hw2 = W.hardware(2)
    hw2["gpus_per_node"] = 2
    s = W.trace_spec(300, 0.2, [(60, 20), (92, 5)])
    cases.append(sweep_case("all_candidates_infeasible", s, 4,
                            lambda t: {"hardware": hw2, "models": two, "cost_model": fast,
                                       "sweep": {"threshold_grid": [[101.0]]}}, 2))
    # a live stage workload with p95 < mean (domain.cpp:190-193) aborts the sweep
    n = 40
    inline = {"arrival_s": [0.5 * i for i in range(n)],
              "input_tokens": [100.0] * 19 + [1000.0] + [0.0] * 20,
              "output_tokens": [[50.0] * n, [50.0] * n],
              "scores": [[90.0] * 19 + [10.0] * 21, [95.0] * n]}
    cases.append(sweep_case("invalid_stage_workload", None, 0,
                            lambda t: {"hardware": hw8, "models": two, "cost_model": fast,
                                       "sweep": {"threshold_grid": [[0.0, 50.0]]}}, 8, inline=inline))
    with open(os.path.join(OUT, "sweeps.json"), "w") as f:
        json.dump(cases, f)

    # rows (StageEvaluator::row) incl. zero-rate, tight KV, saturated
    rows = []
    hw = W.hardware(8)
    hw["gpus_per_node"] = 4
    for i, (model, w, N, p) in enumerate([
        ("small-7b", (0.8, 200, 80, 600, 240), 6, fast),
        ("small-7b", (0.5, 300, 120, 900, 360), 8, W.DEFAULT_COST_MODEL),
        ("mid-70b", (0.3, 400, 100, 1200, 300), 8, fast),
        ("small-7b", (0.0, 100, 100, 300, 300), 4, fast),
        ("small-7b", (1000.0, 300, 120, 900, 360), 4, fast),
        ("large-671b-int4", (0.2, 500, 200, 1500, 600), 16, fast),
        ("small-7b", (0.01, 500, 0, 1500, 0), 3, dict(fast, comm_overhead_per_stage=0.0)),
    ]):
        wl = dict(zip(["arrival_rate", "mean_input_tokens", "mean_output_tokens", "p95_input_tokens",
                       "p95_output_tokens"], [float(v) for v in w]))
        m = W.model_spec(model, 1)
        r = refpy.row(hw, p, m, wl, N)
        rows.append({"hw": hw, "params": p, "model": m, "workload": wl, "max_budget": N, "result": r["result"]})
    with open(os.path.join(OUT, "rows.json"), "w") as f:
        json.dump(rows, f)

    # routing known-answer cases (test_routing.cpp:63-120 shapes) + random
    routes = []
    import numpy as np
    rng = np.random.default_rng(123)
    for trial in range(12):
        c = int(rng.integers(2, 5))
        s = W.trace_spec(int(rng.integers(5, 300)), 1.0, [(50, 30)] * c)
        seed = int(rng.integers(1, 1 << 30))
        t = trace_of(s, seed)
        h = [101.0 if rng.random() < 0.1 else float(rng.uniform(0, 100)) for _ in range(c - 1)]
        dep = [True] + [bool(rng.random() > 0.2) for _ in range(c - 1)]
        r = refpy.route(t, h, dep)
        routes.append({"trace_spec": s, "seed": seed, "thresholds": h, "deployed": dep, "result": r["result"]})
    with open(os.path.join(OUT, "routes.json"), "w") as f:
        json.dump(routes, f)

    # min-max solves (test_innerplan.cpp random_table shape)
    solves = []
    for trial in range(60):
        c = int(rng.integers(1, 4))
        n = int(rng.integers(c, 17))
        entries = []
        for i in range(c):
            row = [None] * (n + 1)
            if rng.random() < 0.15:
                row = [0.0] * (n + 1)
            else:
                first = int(rng.integers(1, n + 1))
                v = float(rng.uniform(0.5, 10.0))
                for f in range(first, n + 1):
                    row[f] = v
                    if rng.random() < 0.6:
                        v *= float(rng.uniform(0.5, 1.0))
            entries.append(row)
        table = {"gpu_budget": n, "entries": entries, "best_plans": [[None] * (n + 1) for _ in range(c)]}
        res = refpy.lib().ref_solve
        out = refpy._call(res, json.dumps(table).encode(), n)
        solves.append({"table": table, "total_gpus": n, "result": out.get("result"),
                       "error": None if out["ok"] else {"code": out["code"], "message": out["message"]}})
    with open(os.path.join(OUT, "solves.json"), "w") as f:
        json.dump(solves, f)
    print("wrote", os.listdir(OUT))


if __name__ == "__main__":
    main()
