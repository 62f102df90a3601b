#!/usr/bin/env python
"""Benchmark: candidate plans evaluated per second by one full plan search
(cascade::outerplan::sweep) on the B200 engine, vs the reference CPU planner.

A step = one complete sweep of the workload (routing of every threshold
candidate, every latency row over the allocation x TP/PP/DP space, the inner
min-max solve, Tchebycheff + Pareto).  The metric's numerator is the number of
(workload row, parallelism plan) pairs the sweep must decide -- the
reference's own count (sum over its row cache of |plan set|), identical for
both arms -- and the denominator the sweep time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C3]

The default workload is C3 (BASELINE.json configs[2], the north-star config:
3-model Llama 8B->70B->405B cascade, 1M-request bursty trace, 64-GPU pool).

N>1 runs under torchrun: every rank routes redundantly, the plan chunks are
dealt round-robin over the ranks, which exchange their p95 bounds after the
pilot pass and every filter wave and merge with one all-gather -- NCCL calls
made by the engine library itself on its stream (strong scaling).

--impl reference times the reference CPU planner (oracle/_ref, compiled from
the unmodified reference sources) on a bounded sample of the same workload and
extrapolates the full sweep's time as a lower bound (oracle/cpu_baseline.py);
its trace comes from the reference's own generator and it never loads the
engine library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "candidate plans evaluated/sec (plan-search sweep)"
UNIT = "plans/s"
WORKLOAD_DESC = {
    "C1": "C1: 2-model Llama-3 8B->70B, 10k-request trace, 16-GPU pool, 32-point grid",
    "C2": "C2: 3-model R1-Distill 8B->32B->671B, 100k-request trace, 32-GPU pool, 64x64 grid",
    "C3": "C3: 3-model Llama 8B->70B->405B, 1M-request heterogeneous bursty trace, 64-GPU pool, decile grid",
    "C4": "C4: C2 cascade, 100k requests, 256x256 grid, 32 Tchebycheff weights",
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def build_workload(name: str, generate=None):
    """The config's synthetic trace and planner config.  `generate` defaults
    to the engine's bit-identical generator; the reference arm passes the
    reference's own cli::generate_trace (oracle/_ref) so it never loads the
    engine library."""
    from paper_2506_04203_b200 import workloads as W
    if generate is None:
        from paper_2506_04203_b200 import engine as eng
        generate = eng.generate_trace
    trace = W.build_trace(name, generate)
    cfg, N = W.planner_config(name, trace["scores"])
    return trace, cfg, N


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        loaded = [v for v in sm if v > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.samples)}


def config_keys(name, trace, N, ref: dict) -> dict:
    """The `config` object both arms print (same keys, same values)."""
    return {"workload": WORKLOAD_DESC.get(name, name), "total_gpus_planned": N,
            "requests": int(trace["arrival_s"].shape[0]), "stages": int(trace["scores"].shape[0]),
            "candidates": ref["candidates"], "unique_rows": ref["unique_rows"], "plans_per_sweep": ref["plans"],
            "l2": "flushed (256 MiB write) before every timed step, outside the events"}


def run_reference(args):
    """The reference CPU planner (oracle/_ref: the unmodified reference
    sources) on this config: every step times a bounded sample of reference
    calls on all host threads and extrapolates the full sweep's time as a
    lower bound (oracle/cpu_baseline.py); value = the sweep's plans / that
    time.  Rank 0 only; the engine library is never loaded here."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    os.environ.setdefault("CASCADE_PLANNER_THREADS", str(os.cpu_count() or 1))
    from oracle import refpy
    if not refpy.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libcascade_ref.so not built"}))
        return 0
    from oracle import cpu_baseline
    trace, cfg, N = build_workload(args.config, refpy.generate_trace)
    ref = cpu_baseline.ReferenceSample(trace, cfg, N)
    for _ in range(args.warmup):
        ref.step()
    steps = [ref.step() for _ in range(args.steps)]
    sweep_s = float(np.mean([s["sweep_s_lower_bound"] for s in steps]))
    sample_s = float(np.mean([s["sample_s"] for s in steps]))
    d = ref.describe()
    value = d["plans"] / sweep_s
    cfg_keys = config_keys(args.config, trace, N, {"candidates": d["candidates"], "unique_rows": d["unique_rows"],
                                                   "plans": d["plans"]})
    cfg_keys["parallelism"] = f"CPU threads: {d['threads']}"
    kind = steps[-1]["kind"]
    base = {"value": value, "unit": UNIT, "cores": d["threads"], "kind": "reference",
            "sample": ref.sample_text(), "extrapolation": kind}
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": sweep_s * 1000.0,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": cfg_keys,
           "extrapolated": {"kind": kind, "sweep_s": sweep_s,
                            "sweep_s_estimate": float(np.mean([s["sweep_s_estimate"] for s in steps])),
                            "measured_sample_s_per_step": sample_s, "census": d,
                            "last_step": steps[-1]},
           "cpu_baseline": base,
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                   "kind": kind}}
    print(json.dumps(out), flush=True)
    return 0


def k1_at_scale(eng, torch, steps, warmup):
    """The routing/aggregation pass (K1) on the C5 trace (10M requests, 4
    stages, default decile grid) through cg_route_grid; K1's duration comes
    from the engine's CUDA events around that kernel on its own stream."""
    from paper_2506_04203_b200 import workloads as W
    spec, seed = W.trace_specs("C5")[0]
    t = eng.generate_trace(spec, seed)
    n, C = int(t["arrival_s"].shape[0]), int(t["scores"].shape[0])
    dev = {k: torch.from_numpy(np.ascontiguousarray(t[k])).cuda() for k in t}
    tb = eng.TraceBuffers(dev["arrival_s"].data_ptr(), dev["input_tokens"].data_ptr(),
                          dev["output_tokens"].data_ptr(), dev["scores"].data_ptr(), on_device=True,
                          keep={"n": n, "stages": C, "t": dev})
    E = eng.Engine(torch.cuda.current_device())
    for _ in range(warmup):
        E.route_grid(tb, {})
    ms, launches = [], 0
    for _ in range(steps):
        E.route_grid(tb, {})
        ms.append(E.last_stats["ms_k1"])
        launches += E.last_stats["gpu_launches"]
    bytes_per_launch = E.last_stats["k1_bytes"]
    E.close()
    del dev
    torch.cuda.empty_cache()
    return float(np.mean(ms)), bytes_per_launch, n, C, launches


def committed_k4_issue():
    """Time-weighted smsp__issue_active / warps_active of the K4 kernels from the
    committed ncu --set full capture summary (profiles/), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "k4_ncu_summary.json")) as f:
            d = json.load(f)
        return {"issue_active_pct": d["issue_active_pct_time_weighted"],
                "warps_active_pct": d["warps_active_pct_time_weighted"], "source": d["source"]}
    except Exception:
        return None


def committed_k1_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per K1 launch from the
    committed ncu --set full capture summary (profiles/), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "k1_ncu_summary.json")) as f:
            return float(json.load(f)["dram_bytes_per_launch"])
    except Exception:
        return None


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2506_04203_b200 import engine as eng

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    trace, cfg, N = build_workload(args.config)
    E = eng.Engine(local)
    if world > 1:
        # the sweep's collectives run inside the engine library on its own
        # NCCL communicator; torch.distributed only ships the unique id
        box = [eng.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        E.set_nccl(box[0], rank, world)
    stream = torch.cuda.ExternalStream(E.stream_handle())

    # HBM-resident trace (value) and pinned host trace (e2e)
    dev = {k: torch.from_numpy(np.ascontiguousarray(trace[k], dtype=np.float64)).cuda()
           for k in ("arrival_s", "input_tokens", "output_tokens", "scores")}
    pin = {k: torch.from_numpy(np.ascontiguousarray(trace[k], dtype=np.float64)).pin_memory()
           for k in ("arrival_s", "input_tokens", "output_tokens", "scores")}
    n = int(trace["arrival_s"].shape[0])
    C = int(trace["scores"].shape[0])
    tr_dev = eng.TraceBuffers(dev["arrival_s"].data_ptr(), dev["input_tokens"].data_ptr(),
                              dev["output_tokens"].data_ptr(), dev["scores"].data_ptr(), on_device=True,
                              keep={"n": n, "stages": C, "t": dev})
    tr_host = eng.TraceBuffers(pin["arrival_s"].numpy(), pin["input_tokens"].numpy(),
                               pin["output_tokens"].numpy(), pin["scores"].numpy())
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def one(tr):
        E.sweep(tr, cfg["models"], cfg["hardware"], cfg["cost_model"], N, cfg["sweep"], raw=True)
        return dict(E.last_stats)

    def timed(tr, steps):
        times, stats = [], []
        for _ in range(steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)  # L2 flush between timed iterations (outside the events)
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            st = one(tr)
            s1.record(stream)
            s1.synchronize()
            times.append(s0.elapsed_time(s1))
            stats.append(st)
        return times, stats

    for _ in range(args.warmup):
        one(tr_dev)
        one(tr_host)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_dev, st_dev = timed(tr_dev, args.steps)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_e2e, st_e2e = timed(tr_host, args.steps)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms_dev = float(np.sum(t_dev))
    ms_e2e = float(np.sum(t_e2e))
    if world > 1:
        tt = torch.tensor([ms_dev, ms_e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_dev, ms_e2e = float(tt[0]), float(tt[1])
    plans = st_dev[-1]["plans_enumerated"]
    value = plans * args.steps / (ms_dev / 1000.0)
    e2e = plans * args.steps / (ms_e2e / 1000.0)

    k1 = None
    if rank == 0 and not args.no_k1:
        k1 = k1_at_scale(eng, torch, args.steps, args.warmup)
    if rank == 0:
        peak, peak_kind = load_peaks()
        if k1:
            k1_ms, k1_bytes, k1_n, k1_C, k1_launches = k1
            k1_work = f"C5 routing pass: {k1_n} requests x {k1_C} stages, default decile grid (cg_route_grid)"
        else:
            k1_ms = float(np.mean([s["ms_k1"] for s in st_dev]))
            k1_bytes = st_dev[-1]["k1_bytes"]
            k1_work = "C2 sweep routing pass"
        k1_gbs = k1_bytes / (k1_ms / 1000.0) / 1e9 if k1_ms > 0 else 0.0
        k4_ms = float(np.mean([s["ms_k4"] for s in st_dev]))
        steps_k4 = st_dev[-1]["request_steps"]
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_dev / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(config_keys(args.config, trace, N, {"candidates": st_dev[-1]["candidates"],
                                                                "unique_rows": st_dev[-1]["unique_rows"],
                                                                "plans": plans}),
                           parallelism=(f"plan chunks dealt round-robin over {world} GPU(s); bound all-gather after the "
                                        "pilot and every wave, one merge all-gather (NCCL inside the engine library)"
                                        if world > 1 else "1 GPU")),
            "e2e": {"value": e2e, "unit": UNIT, "ms_per_step": ms_e2e / args.steps,
                    "h2d_bytes_per_step": st_e2e[-1]["h2d_bytes"], "d2h_bytes_per_step": st_e2e[-1]["d2h_bytes"]},
            "gpu_launches": int(sum(s["gpu_launches"] for s in st_dev) + sum(s["gpu_launches"] for s in st_e2e)),
            "roofline": {"bound": "hbm", "kernel": "k_route_tma (K1 routing/aggregation pass: cp.async.bulk ring + u32 smem histogram)",
                         "workload": k1_work, "achieved": k1_gbs, "peak": peak, "unit": "GB/s",
                         "frac": k1_gbs / peak if peak else None, "traffic": committed_k1_traffic(),
                         "peak_kind": peak_kind, "bytes_per_launch": k1_bytes, "ms_per_launch": k1_ms,
                         "bytes_per_request": "16*C+8 (scores of C-1 threshold stages, input, C outputs, 8 B ranks)"},
            "roofline_k4": {"bound": "issue", "kernel": "k_lane / k_sim (K4 JSQ simulation)", "ms_per_sweep": k4_ms,
                            "request_steps_per_s": steps_k4 / (k4_ms / 1000.0) if k4_ms > 0 else None,
                            "plans_simulated_full": st_dev[-1]["plans_simulated_full"],
                            "plans_pruned": st_dev[-1]["plans_pruned"],
                            "sm_issue_utilisation": committed_k4_issue()},
            "phases_ms": {k: float(np.mean([s[k] for s in st_dev])) for k in
                          ("ms_route", "ms_quality", "ms_rows", "ms_solve", "ms_total")},
            "clocks": clk.summary(),
        }
        if world == 1 and not args.no_cpu_baseline:
            os.environ.setdefault("CASCADE_PLANNER_THREADS", str(os.cpu_count() or 1))
            try:
                from oracle import cpu_baseline
                ref = cpu_baseline.ReferenceSample(trace, cfg, N)
                st = ref.step()
                d = ref.describe()
                out["cpu_baseline"] = {"value": d["plans"] / st["sweep_s_lower_bound"], "unit": UNIT,
                                       "cores": d["threads"], "kind": "reference", "sample": ref.sample_text(),
                                       "extrapolation": st["kind"], "sweep_s": st["sweep_s_lower_bound"],
                                       "sweep_s_estimate": st["sweep_s_estimate"],
                                       "measured_sample_s": st["sample_s"]}
            except Exception as ex:  # reported, never silently replaced
                out["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                                       "sample": f"unavailable: {ex}"}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(WORKLOAD_DESC))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-k1", action="store_true", help="skip the 10M-request K1 roofline pass")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
