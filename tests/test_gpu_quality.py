"""K2 quality sums: the block-parallel exact form (quality_form 1: integer
units of the running sum's binade, sequential blocks at binade crossings,
ties, zero prefixes and negative / non-finite scores) against the one-chain
form (quality_form 0) and the reference's trace-order fold
(routing.cpp:79), on traces built to hit every branch."""
import numpy as np
import pytest

from parity_util import diff_json, small_trace
from paper_2506_04203_b200 import engine as eng

pytestmark = pytest.mark.gpu


def fold(t, th):
    """The reference's sequential fold (numpy cumsum is a left-to-right loop)."""
    sc = t["scores"]
    acc = sc[-1].copy()
    for d in range(len(th) - 1, -1, -1):
        acc = np.where(sc[d] >= th[d], sc[d], acc)
    return float(np.cumsum(acc)[-1]) if acc.size else 0.0


def make(kind, n, seed=3):
    t, _ = small_trace(n, 1.0, ((60, 20), (80, 12), (92, 5)), seed=seed)
    t = {k: np.array(v, dtype=np.float64, copy=True) for k, v in t.items()}
    rng = np.random.default_rng(seed)
    sc = t["scores"]
    if kind == "ties":
        # s near 2^20..2^22 has u = 2^-32..2^-30: these fractions sit exactly on
        # half units of several binades
        for j, e in enumerate((-31, -32, -33, -30, -29)):
            sc[:, j::7] = np.floor(sc[:, j::7]) + 2.0 ** e
    elif kind == "zero_prefix":
        sc[:, : n // 3] = 0.0
    elif kind == "neg_nan":
        idx = rng.choice(n, size=40, replace=False)
        sc[2, idx[:10]] = -1.0
        sc[2, idx[10:20]] = -0.0
        sc[0, idx[20:25]] = np.nan
        sc[2, idx[25:30]] = np.inf
        sc[1, idx[30:]] = -np.inf
    elif kind == "huge":
        sc[2, 5::97] = 1e300
        sc[2, 11::89] = 1.7e308
    elif kind == "tiny":
        sc[:] = rng.random(sc.shape) * 1e-300
        sc[:, ::13] = 5e-324
    elif kind == "binades":
        sc[:] = np.exp(rng.normal(0, 8, sc.shape))  # many magnitudes, many crossings
    return t


@pytest.mark.parametrize("kind,n,block", [("plain", 200_000, 0), ("plain", 1, 0), ("plain", 1023, 0),
                                          ("plain", 70_001, 4096), ("ties", 150_000, 0),
                                          ("zero_prefix", 50_000, 0), ("neg_nan", 60_000, 0),
                                          ("huge", 40_000, 0), ("tiny", 30_000, 0), ("binades", 90_000, 2048)])
def test_quality_forms_bit_exact(engine, kind, n, block):
    t = make(kind, n)
    cfg = {"threshold_grid": [[0.0, 50.0, 65.0, 80.0, 101.0], [0.0, 70.0, 90.0, 101.0]]}
    outs = []
    try:
        engine.set_option("quality_block", block)
        for form in (1, 0):
            engine.set_option("quality_form", form)
            outs.append(engine.route_grid(t, cfg))
    finally:
        engine.set_option("quality_form", 1)
        engine.set_option("quality_block", 0)
    q1 = [c["quality"] for c in outs[0]]
    q0 = [c["quality"] for c in outs[1]]
    assert np.array_equal(np.array(q1).view(np.uint64), np.array(q0).view(np.uint64)) or \
        all((a == b) or (a != a and b != b) for a, b in zip(q1, q0)), kind
    nn = float(n)
    for c in outs[0][::3]:
        want = fold(t, c["thresholds"]) / nn
        got = c["quality"]
        assert (got == want) or (got != got and want != want), (kind, c["thresholds"], got, want)


def test_quality_matches_reference_route(engine):
    from oracle import refpy
    t = make("ties", 20_000, seed=5)
    res = engine.route_grid(t, {})
    for c in res[::10]:
        ref = refpy.route(t, c["thresholds"], [True, True, True])["result"]
        assert c["quality"] == ref["quality"], c["thresholds"]


@pytest.mark.parametrize("kind", ["plain", "big_tokens", "nan_inf_neg", "fractional", "skewed"])
def test_p95_chunk_tables_match_direct_scan(engine, kind):
    """K3 chunk tables (traces >= 65536 requests) against the direct column
    scan and, sampled, the reference route."""
    from oracle import refpy
    n = 131_101
    t, _ = small_trace(n, 1.0, ((60, 20), (80, 12), (92, 5)), seed=21)
    t = {k: np.array(v, dtype=np.float64, copy=True) for k, v in t.items()}
    rng = np.random.default_rng(21)
    idx = rng.choice(n, size=n // 40, replace=False)
    if kind == "big_tokens":
        t["input_tokens"][idx] = rng.choice([65536.0, 1e6, 4294967295.0], size=idx.size)
    elif kind == "nan_inf_neg":
        t["scores"][0, idx[0::3]] = np.nan
        t["scores"][1, idx[1::3]] = -np.inf
        t["scores"][0, idx[2::3]] = 250.0
    elif kind == "fractional":
        t["output_tokens"][2, idx] += 0.5
    elif kind == "skewed":  # tokens correlated with the scores: deep scans for the small workloads
        t["output_tokens"][1] = np.floor(t["scores"][0] * 7.0)
        t["input_tokens"] = np.floor(1000.0 - t["scores"][1] * 3.0).clip(0)
    outs = []
    try:
        for tab in (1, 0):
            engine.set_option("p95_tables", tab)
            outs.append(engine.route_grid(t, {}))
    finally:
        engine.set_option("p95_tables", 1)
    assert not diff_json(outs[0], outs[1]), kind
    for c in outs[0][::17]:
        ref = refpy.route(t, c["thresholds"], [True, True, True])["result"]
        ref.pop("per_request_accept_stage")
        assert not diff_json({k: c[k] for k in ("ratios", "stage_workloads", "quality")}, ref), c["thresholds"]
