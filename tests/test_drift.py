"""GPU parity tests of drift detection: the windowing
and statistics of cli::cmd_drift and cli::compute_baseline vs the reference
(proj/src/cli.cpp:101-131, 216-334), run live from oracle/_ref.  Bar: the
windows of drift_report.json (starts, spans, counts, statistics, deviations,
drift flags) bit-identical; the whole-stream baseline likewise."""
import numpy as np
import pytest

from parity_util import diff_json, small_trace
from paper_2506_04203_b200 import engine as eng
from paper_2506_04203_b200 import workloads as W

pytestmark = pytest.mark.gpu


def bursty_stream(seed=3):
    parts = [eng.generate_trace(W.trace_spec(1500, rate, [(60, 20), (92, 5)]), seed + i)
             for i, rate in enumerate((1.0, 4.0, 0.5, 2.0))]
    return eng.concat_traces(parts)


@pytest.mark.parametrize("policy", [{"window_requests": 100, "window_interval_s": 300.0, "rel_tolerance": 0.2},
                                    {"window_requests": 7, "window_interval_s": 37.5, "rel_tolerance": 0.05},
                                    {"window_requests": 5000, "window_interval_s": 5000.0, "rel_tolerance": 0.5}])
@pytest.mark.parametrize("h1", [None, 70.0])
def test_drift_windows_match_reference(engine, tmp_path, policy, h1):
    from oracle import refpy
    stream = bursty_stream()
    t0, _ = small_trace(3000, 1.0, ((60, 20), (92, 5)), seed=1)
    base = engine.compute_baseline(t0, h1)
    cfg, _ = W.planner_config("C1", t0["scores"], grid=4)
    cfg["drift"] = policy
    ref = refpy.drift(stream, cfg, base, str(tmp_path / "ref"), h1)["result"]
    assert not diff_json(base, refpy.drift(t0, cfg, base, str(tmp_path / "b"), h1)["result"]["baseline_of_stream"])
    got = engine.drift_windows(stream, base, policy)
    assert not diff_json(got["windows"], ref["report"]["windows"])
    assert got["drift_detected"] == ref["report"]["drift_detected"]


def test_drift_zero_baseline_and_gaps(engine, tmp_path):
    """Zero baseline statistics (deviation null) and a stream with empty windows."""
    from oracle import refpy
    t, _ = small_trace(2000, 1.0, ((60, 20), (92, 5)), seed=4)
    t = {k: np.array(v, copy=True) for k, v in t.items()}
    t["arrival_s"][1000:] += 5000.0  # a long gap: empty windows in between
    base = {"arrival_rate": 0.0, "mean_input_tokens": 0.0, "mean_output_tokens": 300.0,
            "stage1_accept_rate": 0.0, "h1": 65.0}
    cfg, _ = W.planner_config("C1", t["scores"], grid=4)
    cfg["drift"] = {"window_requests": 50, "window_interval_s": 120.0, "rel_tolerance": 0.1}
    ref = refpy.drift(t, cfg, base, str(tmp_path / "ref"), 65.0)["result"]
    got = engine.drift_windows(t, base, cfg["drift"])
    assert not diff_json(got["windows"], ref["report"]["windows"])


def test_drift_empty_stream_error(engine):
    empty = {"arrival_s": np.zeros(0), "input_tokens": np.zeros(0), "output_tokens": np.zeros((2, 0)),
             "scores": np.zeros((2, 0))}
    with pytest.raises(eng.CascadeError) as ei:
        engine.drift_windows(empty, {"arrival_rate": 1, "mean_input_tokens": 1, "mean_output_tokens": 1,
                                     "stage1_accept_rate": 1, "h1": None})
    assert ei.value.code == 2 and ei.value.message == "drift stream is empty"
