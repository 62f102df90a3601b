"""TEST INFRASTRUCTURE ONLY: the reference CPU planner's plan-search time on a
benchmark config, measured on a bounded sample and extrapolated to the full
sweep (bench.py's ``--impl reference`` arm and its ``cpu_baseline`` leg).

Nothing here touches the GPU engine's library: the trace comes from the
reference's own generator (``cli::generate_trace`` through oracle/_ref), the
sweep's unique rows from the reference's own ``route_trace`` over every grid
candidate, the per-row plan / stability counts from our C restatement
(``co_row_census``: enumeration + the stability test, no simulation), and
every timed call is an UNMODIFIED reference entry point (``route_trace``,
``StageEvaluator::row``) with CASCADE_PLANNER_THREADS = all host threads.

Why extrapolate: the full C3 sweep makes the reference materialise 3.9e8
plans (~25 GB) for its 8B row and run 4.8e8 queueing simulations -- about an
hour on 16 threads.  The reference's cost is

    sweep_s = sum over distinct plan sets (model, N) of  a * plans     (materialise + test)
            + sum over unique rows of                  b * stable    (one simulation per
                                                                      stable plan,
                                                                      costmodel.cpp:366-382)
            + (candidates + 3) * route_s                             (outerplan.cpp:206-231)

with the row census giving plans / stable exactly.  Per step (all timed by
the reference calls' own clocks):
  * route_s: one route_trace of the full trace (the all-accept candidate, the
    cheapest: fewest pushes into the per-stage lists);
  * a: a real row of the sweep with plans but no stable plan at its sampled
    budget (pure enumeration + stability tests);
  * b_floor: a calibration row -- the heaviest row's model, shapes, CRN stream
    and token statistics with arrival_rate = 1e-3, so every plan is stable and
    every arrival finds the first replica idle: the cheapest simulation the
    reference's dispatch loop can run (one replica check, one push per
    arrival), at a mean replica count below the sweep's;
  * b_est: the heaviest real row at budgets 32 and 36 (its per-simulation cost
    FALLS as the budget grows -- more capacity, shorter queues -- so this is an
    estimate, not a bound).
The headline is the strict LOWER BOUND  a*plans + b_floor*stable + (C+3)*route_s
("extrapolated_lower_bound": the reference is at least this slow); the
b_est-based estimate is reported next to it.
"""
from __future__ import annotations

import os
import time

from oracle import cpy, refpy

SAMPLE_BUDGETS = (32, 36)   # heavy-row budgets timed each step (36: dp > 32 plans present)
DIRECT_MAX_SIMULATIONS = 2_000_000   # below this the full sweep is timed directly (no extrapolation)


def _threads() -> int:
    return int(os.environ.get("CASCADE_PLANNER_THREADS", str(os.cpu_count() or 1)))


class ReferenceSample:
    """Setup (untimed): the sweep's rows and their census.  step(): one
    bounded sample of timed reference calls -> extrapolated sweep time."""

    def __init__(self, trace: dict, cfg: dict, total_gpus: int):
        os.environ.setdefault("CASCADE_PLANNER_THREADS", str(os.cpu_count() or 1))
        self.trace, self.cfg, self.N = trace, cfg, total_gpus
        t0 = time.perf_counter()
        u = refpy.unique_rows(trace, cfg, total_gpus)
        self.rows = u["rows"]
        self.candidates = int(u["candidates"])
        hw, params, models = cfg["hardware"], cfg["cost_model"], cfg["models"]
        self.census = [cpy.row_census(hw, params, models[r["stage"]], r["workload"], total_gpus)
                       for r in self.rows]
        # distinct plan sets (the reference caches plan_set per model and budget)
        sets = {}
        for r, c in zip(self.rows, self.census):
            sets[r["stage"]] = c["plans"]
        self.plans_per_set = sets
        self.plans = sum(c["plans"] for c in self.census)
        self.stable = sum(c["stable"] for c in self.census)
        self.sum_dp = sum(b["sum_dp"] for c in self.census for b in c["bins"])
        # samples: the heaviest row (most simulations) at small budgets, and a
        # row with plans but no stable plan at its sampled budget (pure
        # enumeration cost), both real rows of this sweep
        heavy = max(range(len(self.rows)), key=lambda i: self.census[i]["stable"])
        self.samples = []
        for nb in SAMPLE_BUDGETS:
            nb = min(nb, total_gpus)
            c = cpy.row_census(hw, params, models[self.rows[heavy]["stage"]], self.rows[heavy]["workload"], nb)
            if c["stable"] > 0 and all(s["budget"] != nb or s["row"] != heavy for s in self.samples):
                self.samples.append({"row": heavy, "budget": nb, "census": c, "kind": "simulation"})
        wl = dict(self.rows[heavy]["workload"], arrival_rate=1e-3)
        nb = min(32, total_gpus)
        c = cpy.row_census(hw, params, models[self.rows[heavy]["stage"]], wl, nb)
        self.samples.append({"row": heavy, "budget": nb, "census": c, "kind": "floor", "workload": wl})
        for i, r in enumerate(self.rows):
            nb = min(32, total_gpus)
            c = cpy.row_census(hw, params, models[r["stage"]], r["workload"], nb)
            if c["stable"] == 0 and c["plans"] >= 10_000:
                self.samples.append({"row": i, "budget": nb, "census": c, "kind": "enumeration"})
                break
        self.direct = self.stable <= DIRECT_MAX_SIMULATIONS
        self.setup_s = time.perf_counter() - t0

    def step(self) -> dict:
        """One bounded sample (timed by the reference calls' own clocks)."""
        if self.direct:  # small sweep: the reference's whole outerplan::sweep
            el = float(refpy.sweep(self.trace, self.cfg, self.N)["elapsed_s"])
            return {"kind": "measured", "sweep_s_lower_bound": el, "sweep_s_estimate": el, "sample_s": el}
        hw, params, models = self.cfg["hardware"], self.cfg["cost_model"], self.cfg["models"]
        C = int(self.trace["scores"].shape[0])
        r = refpy.route(self.trace, [0.0] * (C - 1), [True] * C)
        route_s = float(r["elapsed_s"])
        timed = []
        for s in self.samples:
            row = self.rows[s["row"]]
            res = refpy.row(hw, params, models[row["stage"]], s.get("workload", row["workload"]), s["budget"])
            timed.append(dict(s, seconds=float(res["elapsed_s"])))
        enum = [t["seconds"] / t["census"]["plans"] for t in timed if t["kind"] == "enumeration"]
        a = min(enum) if enum else 0.0
        def per_sim(kind):
            v = [(t["seconds"] - a * t["census"]["plans"]) / t["census"]["stable"]
                 for t in timed if t["kind"] == kind and t["census"]["stable"] > 0]
            return max(min(v), 0.0) if v else 0.0
        b_floor, b_est = per_sim("floor"), per_sim("simulation")
        fixed = a * sum(self.plans_per_set.values()) + (self.candidates + 3) * route_s
        sample_s = route_s + sum(t["seconds"] for t in timed)
        return {"kind": "extrapolated_lower_bound", "sweep_s_lower_bound": fixed + b_floor * self.stable,
                "sweep_s_estimate": fixed + max(b_est, b_floor) * self.stable,
                "sample_s": sample_s, "route_s": route_s, "a_s_per_plan": a,
                "b_floor_s_per_simulation": b_floor, "b_est_s_per_simulation": b_est,
                "samples": [{"stage": self.rows[t["row"]]["stage"], "budget": t["budget"], "kind": t["kind"],
                             "plans": t["census"]["plans"], "stable": t["census"]["stable"],
                             "mean_dp_stable": (sum(x["sum_dp"] for x in t["census"]["bins"]) /
                                                max(t["census"]["stable"], 1)),
                             "seconds": t["seconds"]} for t in timed]}

    def describe(self) -> dict:
        return {"unique_rows": len(self.rows), "candidates": self.candidates, "plans": self.plans,
                "stable_plans": self.stable, "mean_dp_stable": self.sum_dp / max(self.stable, 1),
                "plan_sets": {str(k): v for k, v in self.plans_per_set.items()},
                "threads": _threads(), "setup_s": self.setup_s}

    def sample_text(self) -> str:
        if self.direct:
            return ("reference CPU planner (oracle/_ref, unmodified sources), CASCADE_PLANNER_THREADS="
                    f"{_threads()}: the full outerplan::sweep ({len(self.rows)} rows, {self.plans} plans, "
                    f"{self.stable} simulations), measured")
        parts = ["route_trace on the full trace"]
        for s in self.samples:
            st = self.rows[s["row"]]["stage"]
            tag = " calibration, arrival_rate=1e-3" if s["kind"] == "floor" else ""
            parts.append(f"StageEvaluator::row(stage {st}{tag}, N={s['budget']}: {s['census']['plans']} plans, "
                         f"{s['census']['stable']} simulations)")
        return ("reference CPU planner (oracle/_ref, unmodified sources), CASCADE_PLANNER_THREADS="
                f"{_threads()}: " + "; ".join(parts) +
                f" -> extrapolated to the full sweep ({len(self.rows)} rows, {self.plans} plans, "
                f"{self.stable} simulations, {self.candidates}+3 route_trace calls) as a lower bound")
