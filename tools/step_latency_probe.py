"""Lone-plan K4 latency: rows with exactly one plan (budget 1) and n requests;
the K4 time / n is the per-request-step latency of one plan with no other work
to hide it.  python tools/step_latency_probe.py"""
import json, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2506_04203_b200 import engine as eng, workloads as W

E = eng.Engine(0)
hw = W.hardware(1)
hw["gpus_per_node"] = 1
model = W.model_spec("small-7b", 1)
wl = {"arrival_rate": 0.3, "mean_input_tokens": 300.0, "mean_output_tokens": 150.0,
      "p95_input_tokens": 900.0, "p95_output_tokens": 450.0}
for n in (250, 2000, 16000):
    params = dict(W.DEFAULT_COST_MODEL, queueing_sim_requests=n)
    for pack in (3, 1):
        E.set_option("k4_pack", pack)
        for rep in range(3):
            E.row(hw, params, model, wl, 1)
        st = E.last_stats
        print(json.dumps({"n_req": n, "k4_pack": pack, "ms_k4": round(st["ms_k4"], 3),
                          "us_per_step": round(1000 * st["ms_k4"] / n, 3), "steps": st["request_steps"],
                          "stable": st["plans_stable"], "full": st["plans_simulated_full"], "seeded": st["plans_seeded"],
                          "launches": st["gpu_launches"]}), flush=True)
