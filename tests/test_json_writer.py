"""Output serialisation: sweep.json / front.json text
rendered on the GPU vs the reference's nlohmann dump(2) of the same result.

CPU: the number formatter (csrc/json_emit.cuh compiled as host code) against
nlohmann::json's serializer on millions of doubles.  GPU: full files against
the reference CLI payloads (ref_plan_outputs), byte for byte."""
import os
import subprocess

import pytest

from parity_util import ROOT, parity_cases, small_trace
from paper_2506_04203_b200 import build as B
from paper_2506_04203_b200 import workloads as W


def test_number_formatter_matches_nlohmann(tmp_path):
    B.build()
    exe = tmp_path / "dtoa_check"
    cmd = ["g++", "-std=c++17", "-O2", "-I", B._json_dir(), "-I", B.CSRC, "-I", os.path.join(B.LIBDIR, "gen"),
           os.path.join(ROOT, "tests", "native", "dtoa_check.cpp"), "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True)
    for seed in (1, 2, 3):
        r = subprocess.run([str(exe), "1000000", str(seed)], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr


@pytest.mark.gpu
def test_sweep_files_byte_identical(engine):
    from oracle import refpy
    for name, t, cfg, N in parity_cases():
        ref = refpy.plan_outputs(t, cfg, N, {"min_quality": 0.0})
        engine.sweep(t, cfg["models"], cfg["hardware"], cfg.get("cost_model"), N, cfg.get("sweep"), files=True)
        for f in ("sweep.json", "front.json"):
            assert engine.last_files[f] == ref[f], (name, f)


@pytest.mark.gpu
def test_sweep_files_with_skipped_candidates(engine):
    """A cascade where some candidates are infeasible (skipped[] non-empty)."""
    from oracle import refpy
    t, _ = small_trace(1500, 2.0, ((60, 20), (80, 12), (92, 5)), seed=4)
    cfg, _ = W.planner_config("C2", t["scores"], grid=4)
    cfg["hardware"]["gpu_count"] = 16
    cfg["cost_model"]["queueing_sim_requests"] = 300
    ref = refpy.plan_outputs(t, cfg, 16, {"min_quality": 0.0})
    engine.sweep(t, cfg["models"], cfg["hardware"], cfg.get("cost_model"), 16, cfg.get("sweep"), files=True)
    assert '"skipped": []' not in ref["sweep.json"]
    for f in ("sweep.json", "front.json"):
        assert engine.last_files[f] == ref[f], f
