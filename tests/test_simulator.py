"""GPU parity tests of the validation simulator:
cg_simulate vs the reference's cascade::sim::run / sim::compare
(proj/src/simulator.cpp:177-334), run live from oracle/_ref.

Bar: every per-request end-to-end latency, p95, throughput, attainment
fraction, SLO base and the unstable-stage list bit-identical (json(SimReport)
compared field by field); errors with the reference's code and message."""
import pytest

from parity_util import diff_json, small_trace
from paper_2506_04203_b200 import engine as eng
from paper_2506_04203_b200 import workloads as W

pytestmark = pytest.mark.gpu


def front_plans(engine, t, cfg, N, k=None):
    res = engine.sweep(t, cfg["models"], cfg["hardware"], cfg.get("cost_model"), N, cfg.get("sweep"))
    pts = res["front"]["points"]
    return [p["plan_ref"] for p in (pts if k is None else pts[:k])]


def setup_case(n=4000, rate=1.5, three=True, seed=5):
    if three:
        t, _ = small_trace(n, rate, ((60, 20), (80, 12), (92, 5)), seed=seed)
        cfg, _ = W.planner_config("C2", t["scores"], grid=4)
        cfg["hardware"]["gpu_count"] = 16
        cfg["cost_model"]["queueing_sim_requests"] = 400
        return t, cfg, 16
    t, _ = small_trace(n, rate, ((60, 20), (92, 5)), seed=seed)
    cfg, _ = W.planner_config("C1", t["scores"], grid=6)
    cfg["cost_model"]["queueing_sim_requests"] = 400
    return t, cfg, 16


@pytest.mark.parametrize("three", [True, False])
@pytest.mark.parametrize("simcfg", [{}, {"slo_base_s": 2.5, "warmup_fraction": 0.0},
                                    {"warmup_fraction": 0.35, "slo_scales": [0.5, 1, 3]}])
def test_run_matches_reference(engine, three, simcfg):
    from oracle import refpy
    t, cfg, N = setup_case(three=three)
    plans = front_plans(engine, t, cfg, N)
    for plan in plans[:: max(1, len(plans) // 4)]:
        ref = refpy.simulate(t, cfg, [plan], simcfg)["result"]
        got = engine.simulate(plan, t, cfg["models"], cfg["hardware"], cfg["cost_model"], simcfg)
        assert not diff_json(got, ref)


def test_compare_matches_reference(engine):
    from oracle import refpy
    t, cfg, N = setup_case(n=3000)
    plans = front_plans(engine, t, cfg, N)
    assert len(plans) >= 2
    ref = refpy.simulate(t, cfg, plans, {}, compare=True)["result"]
    got = engine.compare(plans, t, cfg["models"], cfg["hardware"], cfg["cost_model"], {})
    assert not diff_json(got, ref)


def test_overloaded_plan_unstable_stage(engine):
    """A heavy trace on a small plan: queues grow, the unstable-stage warning fires."""
    from oracle import refpy
    t, cfg, N = setup_case(n=3000, rate=40.0, three=False)
    plan = front_plans(engine, setup_case(n=3000, rate=1.0, three=False)[0], cfg, N, k=1)[0]
    ref = refpy.simulate(t, cfg, [plan], {})["result"]
    got = engine.simulate(plan, t, cfg["models"], cfg["hardware"], cfg["cost_model"], {})
    assert ref["unstable_stages"], ref["unstable_stages"]
    assert not diff_json(got, ref)


def test_simulator_errors_match_reference(engine):
    from oracle import refpy
    t, cfg, N = setup_case(n=500)
    good = front_plans(engine, t, cfg, N, k=1)[0]
    bad_budget = dict(good, allocations=[a + 1 for a in good["allocations"]])
    none = dict(good, allocations=[0] * len(good["allocations"]), plans=[None] * len(good["plans"]),
                processing_ratios=[0.0] * len(good["plans"]))
    cases = [([bad_budget], {}, False), ([good], {"warmup_fraction": 1.0}, False),
             ([good], {"slo_scales": [2, 1]}, False), ([good], {"slo_scales": [0, 1]}, False),
             ([good], {}, True), ([none], {}, False)]
    for plans, simcfg, cmp in cases:
        with pytest.raises(refpy.RefError) as re_:
            refpy.simulate(t, cfg, plans, simcfg, compare=cmp)
        with pytest.raises(eng.CascadeError) as ge:
            if cmp:
                engine.compare(plans, t, cfg["models"], cfg["hardware"], cfg["cost_model"], simcfg)
            else:
                engine.simulate(plans[0], t, cfg["models"], cfg["hardware"], cfg["cost_model"], simcfg)
        assert (ge.value.code, ge.value.message) == (re_.value.code, re_.value.message)
