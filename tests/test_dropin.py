"""GPU test of the reference-side binding (integration/outerplan_gpu.cpp):
the reference planner's own CLI pipeline (cli::cmd_plan) with its
outerplan::sweep served by the engine writes plan.json / front.json /
front.csv / sweep.json byte-identical to the reference's CPU sweep."""
import json
import os
import subprocess

import pytest

from parity_util import ROOT
from paper_2506_04203_b200 import workloads as W

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_check")


@pytest.mark.skipif(not os.path.exists(BIN), reason="drop-in binary not built (make -C oracle dropin)")
@pytest.mark.parametrize("gpus", ["", "all"])
@pytest.mark.parametrize("name", ["fixture2", "three_stage"])
def test_cli_outputs_byte_identical(tmp_path, name, gpus):
    """gpus="all": CASCADE_PLANNER_GPUS makes the binding create one engine over
    every visible GPU (cg_engine_create_multi, NCCL inside the library)."""
    if name == "fixture2":
        hw = W.hardware(8)
        hw["gpus_per_node"] = 4
        cfg = {"hardware": hw, "models": [W.model_spec("small-7b", 1), W.model_spec("mid-70b", 2)],
               "cost_model": dict(W.DEFAULT_COST_MODEL, queueing_sim_requests=300),
               "sweep": {"weight_count": 7}}
        spec = W.trace_spec(1500, 0.4, [(70, 25), (95, 3)])
        minq = 80.0
    else:
        cfg = {"hardware": W.hardware(16),
               "models": [W.model_spec("small-7b", 1), W.model_spec("mid-70b", 2),
                          W.model_spec("large-671b-int4", 3)],
               "cost_model": dict(W.DEFAULT_COST_MODEL, queueing_sim_requests=600), "sweep": {}}
        spec = W.trace_spec(2500, 1.5, [(60, 20), (80, 12), (92, 5)])
        minq = 60.0
    (tmp_path / "config.json").write_text(json.dumps(cfg))
    (tmp_path / "spec.json").write_text(json.dumps(spec))
    r = subprocess.run([BIN, str(tmp_path / "config.json"), str(tmp_path / "spec.json"), "7",
                        str(tmp_path / "out"), str(minq)], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, CASCADE_PLANNER_GPUS=gpus))
    assert r.returncode == 0, r.stdout + r.stderr
    rep = json.loads(r.stdout.strip().splitlines()[-1])
    assert rep["identical"], rep
    for f, info in rep["files"].items():
        assert info["identical"] and info["bytes"] > 0, f
