"""GPU tests of the sharded (multi-rank) sweep path on one B200.

The driver's GPU box has one GPU, so the N>1 path runs here as several engines
on the same device: each engine evaluates its round-robin share of the plan
chunks, the ranks exchange p95 bounds after the pilot pass and after every
filter wave, and one all-gather feeds the device merge.  The all-gather is a
host-side exchange (torch copies between the engines' buffers) through the
cg_engine_set_collective callback, or NCCL inside the library at world 1
(cg_engine_create_multi / cg_engine_set_nccl: NCCL refuses two ranks on one
GPU).  Every sharded result must equal the single-engine result and the
reference bit for bit.
"""
import threading

import pytest

from parity_util import diff_json, golden_trace
from paper_2506_04203_b200 import engine as eng
from paper_2506_04203_b200 import workloads as W

pytestmark = pytest.mark.gpu


class DevPtr:
    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def run_sweep(E, t, cfg, N):
    return E.sweep(t, cfg["models"], cfg["hardware"], cfg.get("cost_model"), N, cfg.get("sweep"))


def sharded_sweep(world, t, cfg, N, options=()):
    """One sweep sharded over `world` engines on cuda:0 (threads + barrier)."""
    import torch
    engines = [eng.Engine(0) for _ in range(world)]
    bar = threading.Barrier(world)
    slots = {}
    calls = [0] * world

    def make_ag(rank):
        def ag(send, recv, nbytes):
            calls[rank] += 1
            slots[rank] = torch.as_tensor(DevPtr(send, nbytes), device="cuda").clone()
            bar.wait()
            r = torch.as_tensor(DevPtr(recv, world * nbytes), device="cuda")
            for k in range(world):
                r[k * nbytes:(k + 1) * nbytes].copy_(slots[k])
            torch.cuda.synchronize()
            bar.wait()
        return ag

    results, stats, errors = [None] * world, [None] * world, []

    def run(rank):
        try:
            E = engines[rank]
            for k, v in options:
                E.set_option(k, v)
            E.set_collective(rank, world, make_ag(rank))
            results[rank] = run_sweep(E, t, cfg, N)
            stats[rank] = E.last_stats
        except Exception as e:  # noqa: BLE001
            errors.append(e)
            bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for e in engines:
        e.close()
    assert not errors, errors
    return results, stats, calls


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_sweep_matches_golden(golden, world):
    for name in ("c1_small_grid12", "fixture2_default_grid"):
        cases = [c for c in golden["sweeps"] if c["name"] == name]
        if not cases:
            continue
        case = cases[0]
        t = golden_trace(case)
        results, _, _ = sharded_sweep(world, t, case["config"], case["total_gpus"])
        for r in range(world):
            assert not diff_json(results[r], case["result"]), (name, world, r)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_multi_wave_sweep_matches_reference(world):
    """A C2-model cascade whose plan lists span several filter waves
    (wave_plans=1: 2^20 plans per wave), so the per-wave bound exchanges run;
    the sharded result equals the single-engine result and the reference."""
    from oracle import refpy
    spec, seed = W.trace_specs("C2", 20000)[0]
    t = eng.generate_trace(spec, seed)
    cfg, N = W.planner_config("C2", t["scores"], grid=4)
    ref = refpy.sweep(t, cfg, N)["result"]
    E = eng.Engine(0)
    E.set_option("wave_plans", 1)
    single = run_sweep(E, t, cfg, N)
    st1 = E.last_stats
    E.close()
    assert not diff_json(single, ref)
    results, stats, calls = sharded_sweep(world, t, cfg, N, options=(("wave_plans", 1),))
    waves = -(-st1["plans_enumerated"] // (1 << 20))
    assert waves >= 2
    for r in range(world):
        assert not diff_json(results[r], ref), (world, r)
        assert stats[r]["num_ranks"] == world
        assert stats[r]["collectives"] >= 1  # the bound exchanges ran
    assert len(set(calls)) == 1  # every rank made the same collective calls
    # the shares add up: every stable plan decided exactly once over the ranks
    tot = {k: sum(s[k] for s in stats) for k in ("plans_stable", "plans_simulated_full", "plans_pruned",
                                                  "plans_bound_skipped")}
    assert tot["plans_stable"] == st1["plans_stable"]
    assert tot["plans_simulated_full"] + tot["plans_pruned"] + tot["plans_bound_skipped"] == tot["plans_stable"]


def test_multi_device_engine_nccl_one_device(golden):
    """cg_engine_create_multi over [0]: NCCL clique of one, the collective path
    (bound exchanges, all-gather, device merge) through the library's NCCL."""
    E = eng.Engine(devices=[0])
    assert E.device_count() == 1
    try:
        for case in golden["sweeps"]:
            if "error" in case:
                with pytest.raises(eng.CascadeError) as ei:
                    run_sweep(E, golden_trace(case), case["config"], case["total_gpus"])
                assert ei.value.code == case["error"]["code"]
                assert ei.value.message == case["error"]["message"]
                continue
            got = run_sweep(E, golden_trace(case), case["config"], case["total_gpus"])
            assert not diff_json(got, case["result"]), case["name"]
        assert E.last_stats["num_ranks"] == 1
        for case in golden["rows"]:
            got = E.row(case["hw"], case["params"], case["model"], case["workload"], case["max_budget"])
            assert not diff_json(got, case["result"]), case["workload"]
    finally:
        E.close()


def test_engine_set_nccl_world_one(golden):
    """cg_engine_set_nccl (one process per GPU) at world 1."""
    uid = eng.nccl_unique_id()
    assert len(uid) == 128
    E = eng.Engine(0)
    E.set_nccl(uid, 0, 1)
    try:
        case = [c for c in golden["sweeps"] if "error" not in c][0]
        got = run_sweep(E, golden_trace(case), case["config"], case["total_gpus"])
        assert not diff_json(got, case["result"])
        assert E.last_stats["collectives"] >= 0
        with pytest.raises(eng.CascadeError):
            E.set_collective(0, 2, lambda *a: None)
    finally:
        E.close()


def test_multi_device_engine_rejects_bad_device_lists():
    with pytest.raises(eng.CascadeError):
        eng.Engine(devices=[])
    with pytest.raises(eng.CascadeError):
        eng.Engine(devices=[0, 0])
