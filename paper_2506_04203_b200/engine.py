"""Python mirror of the reference planner's plan-search entry points, bound to
the B200 engine's C ABI (include/cascade_gpu.h) through ctypes.

Names, argument meaning and error behaviour follow the reference C++ API:

    sweep(trace, models, hw, params, total_gpus, cfg)   cascade::outerplan::sweep
    route_trace(trace, thresholds, deployed)           cascade::routing::route_trace
    StageEvaluator(hw, params).row(model, w, budget)   cascade::costmodel::StageEvaluator::row
    solve_min_max(table, total_gpus)                   cascade::innerplan::solve_min_max
    generate_trace(spec, seed)                         cascade::cli::generate_trace
    read_trace_jsonl(path)                             cascade::read_trace_jsonl
    simulate(plan, ...) / compare(plans, ...)          cascade::sim::run / sim::compare

Results are returned in the reference's JSON schema (plain dicts, the
structure nlohmann::json(SweepResult) produces), errors raise CascadeError
carrying the reference's Errc code and message.  There is no CPU fallback:
if the CUDA library or a B200 is missing, every compute call raises.
"""
from __future__ import annotations

import ctypes
import json
import math
import os
from typing import Any, Optional, Sequence

import numpy as np

from . import build as _build

LIB_PATH = _build.LIB

ERRC_NAMES = {0: "INVALID_INPUT", 1: "IO_ERROR", 2: "EMPTY_TRACE", 3: "NO_DEPLOYED_STAGE",
              4: "INFEASIBLE", 5: "INFEASIBLE_PROBLEM", 6: "NO_FEASIBLE_POINT",
              100: "CUDA_ERROR", 101: "UNSUPPORTED"}


class CascadeError(Exception):
    """Mirror of cascade::CascadeError (errors.hpp:25-35)."""

    def __init__(self, code: int, message: str):
        super().__init__(f"{ERRC_NAMES.get(code, code)}: {message}")
        self.code = code
        self.code_name = ERRC_NAMES.get(code, str(code))
        self.message = message


# ---------------------------------------------------------------------------
# ctypes mirrors of include/cascade_gpu.h

class Status(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("message", ctypes.c_char * 512)]


class Hardware(ctypes.Structure):
    _fields_ = [("gpu_count", ctypes.c_int32), ("flops_per_gpu", ctypes.c_double),
                ("mem_bandwidth_per_gpu", ctypes.c_double), ("mem_capacity_per_gpu", ctypes.c_double),
                ("intra_node_bw", ctypes.c_double), ("inter_node_bw", ctypes.c_double),
                ("gpus_per_node", ctypes.c_int32)]


class Model(ctypes.Structure):
    _fields_ = [("id", ctypes.c_char_p), ("param_count", ctypes.c_double),
                ("bytes_per_param", ctypes.c_double), ("kv_bytes_per_token", ctypes.c_double),
                ("min_gpus", ctypes.c_int32), ("stage_index", ctypes.c_int32)]


class CostParams(ctypes.Structure):
    _fields_ = [("prefill_efficiency", ctypes.c_double), ("decode_bw_efficiency", ctypes.c_double),
                ("pipeline_bubble_factor", ctypes.c_double), ("comm_overhead_per_stage", ctypes.c_double),
                ("kv_memory_fraction", ctypes.c_double), ("queueing_sim_requests", ctypes.c_int32),
                ("queueing_sim_seed", ctypes.c_uint64)]


class Workload(ctypes.Structure):
    _fields_ = [("arrival_rate", ctypes.c_double), ("mean_input_tokens", ctypes.c_double),
                ("mean_output_tokens", ctypes.c_double), ("p95_input_tokens", ctypes.c_double),
                ("p95_output_tokens", ctypes.c_double)]


_DP = ctypes.POINTER(ctypes.c_double)


class Trace(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("stages", ctypes.c_int32), ("on_device", ctypes.c_int32),
                ("arrival_s", ctypes.c_void_p), ("input_tokens", ctypes.c_void_p),
                ("output_tokens", ctypes.c_void_p), ("scores", ctypes.c_void_p)]


class SweepConfigC(ctypes.Structure):
    _fields_ = [("grid_dims", ctypes.c_int32), ("grid_sizes", ctypes.POINTER(ctypes.c_int64)),
                ("grid_values", _DP), ("weight_ratio_min", ctypes.c_double),
                ("weight_ratio_max", ctypes.c_double), ("weight_count", ctypes.c_int32)]


class Replica(ctypes.Structure):
    _fields_ = [("tp", ctypes.c_int32), ("pp", ctypes.c_int32)]


class Plan(ctypes.Structure):
    _fields_ = [("gpus_used", ctypes.c_int32), ("dp", ctypes.c_int32), ("replica_offset", ctypes.c_int64)]


class SweepStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "candidates", "distinct_candidates", "stage_workloads", "unique_rows", "plans_enumerated",
        "plans_stable", "plans_simulated_full", "plans_pruned", "plans_bound_skipped", "plans_seeded", "plans_overflow", "request_steps",
        "h2d_bytes", "d2h_bytes")] + [("num_ranks", ctypes.c_int32), ("gpu_launches", ctypes.c_int32)] + \
        [(n, ctypes.c_double) for n in ("ms_total", "ms_route", "ms_quality", "ms_rows", "ms_solve",
                                        "ms_k1", "k1_bytes", "ms_k4")] + [("collectives", ctypes.c_int64), ("quality_blocks", ctypes.c_int64),
                                                           ("quality_blocks_seq", ctypes.c_int64),
                                                           ("waves_total", ctypes.c_int64), ("waves_run", ctypes.c_int64),
                                                           ("plans_in_waves", ctypes.c_int64)]


class SweepResultC(ctypes.Structure):
    _fields_ = [("stages", ctypes.c_int32), ("z1_star", ctypes.c_double), ("z2_star", ctypes.c_double),
                ("num_evaluations", ctypes.c_int64), ("eval_candidate", ctypes.POINTER(ctypes.c_int64)),
                ("eval_thresholds", _DP), ("eval_latency", _DP), ("eval_quality", _DP),
                ("eval_ratios", _DP), ("eval_allocations", ctypes.POINTER(ctypes.c_int32)),
                ("eval_plan", ctypes.POINTER(ctypes.c_int64)), ("num_plans", ctypes.c_int64),
                ("plans", ctypes.POINTER(Plan)), ("num_replicas", ctypes.c_int64),
                ("replicas", ctypes.POINTER(Replica)), ("num_weights", ctypes.c_int32),
                ("weights", _DP), ("weight_selection", ctypes.POINTER(ctypes.c_int32)),
                ("front_size", ctypes.c_int64), ("front", ctypes.POINTER(ctypes.c_int64)),
                ("num_skipped", ctypes.c_int64), ("skipped_candidate", ctypes.POINTER(ctypes.c_int64)),
                ("skipped_thresholds", _DP), ("stats", SweepStats)]


class RouteResultC(ctypes.Structure):
    _fields_ = [("stages", ctypes.c_int32), ("ratios", ctypes.c_double * 8),
                ("stage_workloads", Workload * 8), ("quality", ctypes.c_double)]


class RouteGridResultC(ctypes.Structure):
    _fields_ = [("stages", ctypes.c_int32), ("num_candidates", ctypes.c_int64), ("thresholds", _DP),
                ("ratios", _DP), ("workloads", ctypes.POINTER(Workload)), ("quality", _DP),
                ("stats", SweepStats)]


class RowResultC(ctypes.Structure):
    _fields_ = [("max_budget", ctypes.c_int32), ("latency", _DP),
                ("plan_index", ctypes.POINTER(ctypes.c_int64)), ("num_plans", ctypes.c_int64),
                ("plans", ctypes.POINTER(Plan)), ("num_replicas", ctypes.c_int64),
                ("replicas", ctypes.POINTER(Replica)), ("stats", SweepStats)]


# The reference's JSON files are written by its nlohmann build; the one in this
# image (and therefore the compiled oracle) prints integer arrays on one line.
JSON_FLAGS = int(os.environ.get("CASCADE_JSON_FLAGS", "1"))


class IngestStats(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_int64), ("lines", ctypes.c_int64), ("records", ctypes.c_int64),
                ("host_lines", ctypes.c_int64), ("gpu_launches", ctypes.c_int32), ("ms_total", ctypes.c_double),
                ("ms_read", ctypes.c_double)]


class TraceBufferC(ctypes.Structure):
    _fields_ = [("host", Trace), ("device", Trace), ("stats", IngestStats)]


class SimConfigC(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("slo_base_s", ctypes.c_double), ("slo_scales", _DP),
                ("num_scales", ctypes.c_int32), ("warmup_fraction", ctypes.c_double)]


class CascadePlanC(ctypes.Structure):
    _fields_ = [("allocations", ctypes.POINTER(ctypes.c_int32)), ("processing_ratios", _DP), ("thresholds", _DP),
                ("has_plan", ctypes.POINTER(ctypes.c_int32)), ("gpus_used", ctypes.POINTER(ctypes.c_int32)),
                ("dp", ctypes.POINTER(ctypes.c_int32)), ("replicas", ctypes.POINTER(Replica))]


class SimReportC(ctypes.Structure):
    _fields_ = [("end_to_end_s", _DP), ("accept_stage", ctypes.POINTER(ctypes.c_int32)), ("p95_s", ctypes.c_double),
                ("throughput_rps", ctypes.c_double), ("num_scales", ctypes.c_int32), ("attainment_scale", _DP),
                ("attainment_fraction", _DP), ("has_min_scale_95", ctypes.c_int32), ("min_scale_95", ctypes.c_double),
                ("slo_base_s", ctypes.c_double), ("num_unstable", ctypes.c_int32),
                ("unstable_stages", ctypes.c_int32 * 8)]


class SimResultC(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("num_reports", ctypes.c_int32), ("reports", ctypes.POINTER(SimReportC)),
                ("gpu_launches", ctypes.c_int32), ("ms_total", ctypes.c_double)]


class DriftPolicyC(ctypes.Structure):
    _fields_ = [("window_requests", ctypes.c_int32), ("window_interval_s", ctypes.c_double),
                ("rel_tolerance", ctypes.c_double)]


class DriftStatsC(ctypes.Structure):
    _fields_ = [("arrival_rate", ctypes.c_double), ("mean_input_tokens", ctypes.c_double),
                ("mean_output_tokens", ctypes.c_double), ("stage1_accept_rate", ctypes.c_double),
                ("has_h1", ctypes.c_int32), ("h1", ctypes.c_double)]


class DriftWindowC(ctypes.Structure):
    _fields_ = [("start_s", ctypes.c_double), ("span_s", ctypes.c_double), ("requests", ctypes.c_int32),
                ("sampled", ctypes.c_int32), ("first_record", ctypes.c_int64), ("stats", DriftStatsC),
                ("deviation", ctypes.c_double * 4), ("deviation_is_null", ctypes.c_int32 * 4),
                ("drifted", ctypes.c_int32 * 4), ("any_drift", ctypes.c_int32)]


class DriftResultC(ctypes.Structure):
    _fields_ = [("num_windows", ctypes.c_int64), ("windows", ctypes.POINTER(DriftWindowC)),
                ("drift_detected", ctypes.c_int32)]


DRIFT_STATS = ["arrival_rate", "mean_input_tokens", "mean_output_tokens", "stage1_accept_rate"]


def _drift_stats_json(s: DriftStatsC) -> dict:
    return {"arrival_rate": s.arrival_rate, "mean_input_tokens": s.mean_input_tokens,
            "mean_output_tokens": s.mean_output_tokens, "stage1_accept_rate": s.stage1_accept_rate,
            "h1": s.h1 if s.has_h1 else None}


SIM_DEFAULT_SCALES = [1, 1.5, 2, 2.5, 3, 4, 5, 6, 8, 10, 12, 14, 16, 20]


def sim_config_c(cfg: Optional[dict]):
    cfg = cfg or {}
    scales = [float(v) for v in cfg.get("slo_scales", SIM_DEFAULT_SCALES)]
    arr = (ctypes.c_double * max(1, len(scales)))(*scales)
    return SimConfigC(int(cfg.get("seed", 0)), float(cfg.get("slo_base_s", 0.0)), arr, len(scales),
                      float(cfg.get("warmup_fraction", 0.1))), arr


def cascade_plan_c(plan: dict):
    """CascadePlan JSON (domain.cpp:317-342 schema) -> cg_cascade_plan."""
    C = len(plan["allocations"])
    I32 = ctypes.c_int32
    alloc = (I32 * C)(*[int(v) for v in plan["allocations"]])
    ratios = (ctypes.c_double * C)(*[float(v) for v in plan["processing_ratios"]])
    h = plan["thresholds"]["thresholds"]
    thr = (ctypes.c_double * max(1, len(h)))(*[float(v) for v in h])
    has = (I32 * C)(*[0 if p is None else 1 for p in plan["plans"]])
    used = (I32 * C)(*[0 if p is None else int(p["gpus_used"]) for p in plan["plans"]])
    dps = (I32 * C)(*[0 if p is None else len(p["replicas"]) for p in plan["plans"]])
    reps = [r for p in plan["plans"] if p is not None for r in p["replicas"]]
    rarr = (Replica * max(1, len(reps)))(*[Replica(int(r["tp"]), int(r["pp"])) for r in reps])
    keep = (alloc, ratios, thr, has, used, dps, rarr)
    return CascadePlanC(alloc, ratios, thr, has, used, dps, rarr), keep


def _sim_report_json(r: SimReportC, n: int) -> dict:
    e2e = np.ctypeslib.as_array(r.end_to_end_s, shape=(n,)) if n else np.zeros(0)
    st = np.ctypeslib.as_array(r.accept_stage, shape=(n,)) if n else np.zeros(0, dtype=np.int32)
    return {"per_request": [{"end_to_end_s": float(e2e[i]), "accept_stage": int(st[i])} for i in range(n)],
            "p95_s": float(r.p95_s), "throughput_rps": float(r.throughput_rps),
            "attainment": [{"scale": float(r.attainment_scale[k]), "fraction": float(r.attainment_fraction[k])}
                           for k in range(r.num_scales)],
            "min_scale_95": float(r.min_scale_95) if r.has_min_scale_95 else None,
            "slo_base_s": float(r.slo_base_s),
            "unstable_stages": [int(r.unstable_stages[k]) for k in range(r.num_unstable)]}


ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                ctypes.c_void_p)

EXPORTED = ["cg_engine_create", "cg_engine_destroy", "cg_engine_stream", "cg_engine_set_collective", "cg_engine_set_option",
            "cg_sweep", "cg_sweep_result_free", "cg_route", "cg_stage_row", "cg_row_result_free",
            "cg_solve_min_max", "cg_generate_trace", "cg_version", "cg_route_grid", "cg_route_grid_result_free",
            "cg_merge_row_shards", "cg_shard_row_plans", "cg_merge_budget_bests", "cg_read_trace_jsonl", "cg_parse_trace_jsonl",
            "cg_trace_buffer_free", "cg_sweep_result_json", "cg_text_free", "cg_simulate",
            "cg_sim_result_free", "cg_drift_windows", "cg_drift_result_free", "cg_trace_baseline",
            "cg_engine_create_multi", "cg_engine_device_count", "cg_nccl_unique_id_bytes", "cg_nccl_unique_id",
            "cg_engine_set_nccl"]

_lib = None


def library():
    """Loads the in-tree engine library (never a CPU substitute)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"engine library missing: {LIB_PATH} (run __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        L.cg_engine_create.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]
        L.cg_engine_create.restype = Status
        L.cg_engine_destroy.argtypes = [ctypes.c_void_p]
        L.cg_engine_destroy.restype = None
        L.cg_engine_set_collective.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                               ALLGATHER_FN, ctypes.c_void_p]
        L.cg_engine_set_collective.restype = Status
        L.cg_engine_create_multi.argtypes = [ctypes.POINTER(ctypes.c_int32), ctypes.c_int32,
                                             ctypes.POINTER(ctypes.c_void_p)]
        L.cg_engine_create_multi.restype = Status
        L.cg_engine_device_count.argtypes = [ctypes.c_void_p]
        L.cg_engine_device_count.restype = ctypes.c_int32
        L.cg_nccl_unique_id_bytes.argtypes = []
        L.cg_nccl_unique_id_bytes.restype = ctypes.c_int32
        L.cg_nccl_unique_id.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        L.cg_nccl_unique_id.restype = Status
        L.cg_engine_set_nccl.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int32, ctypes.c_int32]
        L.cg_engine_set_nccl.restype = Status
        L.cg_engine_set_option.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int64]
        L.cg_engine_set_option.restype = Status
        L.cg_sweep.argtypes = [ctypes.c_void_p, ctypes.POINTER(Trace), ctypes.POINTER(Model), ctypes.c_int32,
                               ctypes.POINTER(Hardware), ctypes.POINTER(CostParams), ctypes.c_int32,
                               ctypes.POINTER(SweepConfigC), ctypes.POINTER(ctypes.POINTER(SweepResultC))]
        L.cg_sweep.restype = Status
        L.cg_sweep_result_free.argtypes = [ctypes.POINTER(SweepResultC)]
        L.cg_sweep_result_free.restype = None
        L.cg_route.argtypes = [ctypes.c_void_p, ctypes.POINTER(Trace), _DP, ctypes.POINTER(ctypes.c_int32),
                               ctypes.POINTER(RouteResultC), ctypes.POINTER(ctypes.c_int32)]
        L.cg_route.restype = Status
        L.cg_route_grid.argtypes = [ctypes.c_void_p, ctypes.POINTER(Trace), ctypes.POINTER(SweepConfigC),
                                    ctypes.POINTER(ctypes.POINTER(RouteGridResultC))]
        L.cg_route_grid.restype = Status
        L.cg_route_grid_result_free.argtypes = [ctypes.POINTER(RouteGridResultC)]
        L.cg_route_grid_result_free.restype = None
        L.cg_merge_row_shards.argtypes = [ctypes.POINTER(Model), ctypes.POINTER(Hardware), ctypes.POINTER(CostParams),
                                          ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_uint64),
                                          ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.POINTER(RowResultC))]
        L.cg_merge_row_shards.restype = Status
        L.cg_shard_row_plans.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int64]
        L.cg_shard_row_plans.restype = ctypes.c_int64
        L.cg_merge_budget_bests.argtypes = [ctypes.POINTER(Model), ctypes.POINTER(Hardware), ctypes.POINTER(CostParams),
                                            ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_uint64),
                                            ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64),
                                            ctypes.POINTER(ctypes.c_uint64)]
        L.cg_merge_budget_bests.restype = Status
        L.cg_stage_row.argtypes = [ctypes.c_void_p, ctypes.POINTER(Model), ctypes.POINTER(Workload),
                                   ctypes.POINTER(Hardware), ctypes.POINTER(CostParams), ctypes.c_int32,
                                   ctypes.POINTER(ctypes.POINTER(RowResultC))]
        L.cg_stage_row.restype = Status
        L.cg_row_result_free.argtypes = [ctypes.POINTER(RowResultC)]
        L.cg_row_result_free.restype = None
        L.cg_solve_min_max.argtypes = [ctypes.c_void_p, _DP, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.POINTER(ctypes.c_int32), _DP, _DP]
        L.cg_solve_min_max.restype = Status
        L.cg_generate_trace.argtypes = [ctypes.c_char_p, ctypes.c_uint64, _DP, _DP, _DP, _DP, ctypes.c_int64,
                                        ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int32)]
        L.cg_generate_trace.restype = Status
        L.cg_version.restype = ctypes.c_char_p
        L.cg_read_trace_jsonl.argtypes = [ctypes.c_void_p, ctypes.c_char_p,
                                          ctypes.POINTER(ctypes.POINTER(TraceBufferC))]
        L.cg_read_trace_jsonl.restype = Status
        L.cg_parse_trace_jsonl.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int64, ctypes.c_char_p,
                                           ctypes.POINTER(ctypes.POINTER(TraceBufferC))]
        L.cg_parse_trace_jsonl.restype = Status
        L.cg_sweep_result_json.argtypes = [ctypes.c_void_p, ctypes.POINTER(SweepResultC), ctypes.c_int32,
                                           ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p),
                                           ctypes.POINTER(ctypes.c_int64)]
        L.cg_sweep_result_json.restype = Status
        L.cg_text_free.argtypes = [ctypes.c_void_p]
        L.cg_text_free.restype = None
        L.cg_simulate.argtypes = [ctypes.c_void_p, ctypes.POINTER(Trace), ctypes.POINTER(Model), ctypes.c_int32,
                                  ctypes.POINTER(Hardware), ctypes.POINTER(CostParams), ctypes.POINTER(SimConfigC),
                                  ctypes.POINTER(CascadePlanC), ctypes.c_int32, ctypes.c_int32,
                                  ctypes.POINTER(ctypes.POINTER(SimResultC))]
        L.cg_simulate.restype = Status
        L.cg_drift_windows.argtypes = [ctypes.c_void_p, ctypes.POINTER(Trace), ctypes.POINTER(DriftStatsC),
                                       ctypes.POINTER(DriftPolicyC), ctypes.POINTER(ctypes.POINTER(DriftResultC))]
        L.cg_drift_windows.restype = Status
        L.cg_drift_result_free.argtypes = [ctypes.POINTER(DriftResultC)]
        L.cg_drift_result_free.restype = None
        L.cg_trace_baseline.argtypes = [ctypes.c_void_p, ctypes.POINTER(Trace), ctypes.c_int32, ctypes.c_double,
                                        ctypes.POINTER(DriftStatsC)]
        L.cg_trace_baseline.restype = Status
        L.cg_sim_result_free.argtypes = [ctypes.POINTER(SimResultC)]
        L.cg_sim_result_free.restype = None
        L.cg_trace_buffer_free.argtypes = [ctypes.POINTER(TraceBufferC)]
        L.cg_trace_buffer_free.restype = None
        L.cg_engine_stream.argtypes = [ctypes.c_void_p]
        L.cg_engine_stream.restype = ctypes.c_void_p
        _lib = L
    return _lib


def _check(st: Status):
    if st.code != -1:
        raise CascadeError(int(st.code), st.message.decode(errors="replace"))


# ---------------------------------------------------------------------------
# conversions


def hardware_c(hw: dict) -> Hardware:
    return Hardware(int(hw["gpu_count"]), float(hw["flops_per_gpu"]), float(hw["mem_bandwidth_per_gpu"]),
                    float(hw["mem_capacity_per_gpu"]), float(hw["intra_node_bw"]), float(hw["inter_node_bw"]),
                    int(hw["gpus_per_node"]))


DEFAULT_PARAMS = {"prefill_efficiency": 0.5, "decode_bw_efficiency": 0.7, "pipeline_bubble_factor": 0.1,
                  "comm_overhead_per_stage": 0.002, "kv_memory_fraction": 0.9,
                  "queueing_sim_requests": 2000, "queueing_sim_seed": 12345}


def params_c(p: Optional[dict]) -> CostParams:
    q = dict(DEFAULT_PARAMS)
    q.update(p or {})
    return CostParams(float(q["prefill_efficiency"]), float(q["decode_bw_efficiency"]),
                      float(q["pipeline_bubble_factor"]), float(q["comm_overhead_per_stage"]),
                      float(q["kv_memory_fraction"]), int(q["queueing_sim_requests"]),
                      int(q["queueing_sim_seed"]))


def models_c(models: Sequence[dict]):
    arr = (Model * max(1, len(models)))()
    keep = []
    for i, m in enumerate(models):
        mid = str(m["id"]).encode()
        keep.append(mid)
        arr[i] = Model(mid, float(m["param_count"]), float(m["bytes_per_param"]),
                       float(m["kv_bytes_per_token"]), int(m.get("min_gpus", 1)), int(m["stage_index"]))
    return arr, keep


class TraceBuffers:
    """SoA trace columns (host numpy, or device pointers when on_device)."""

    def __init__(self, arrival_s, input_tokens, output_tokens, scores, on_device=False, keep=None):
        self.on_device = on_device
        self.keep = keep
        if on_device:
            self.ptrs = (arrival_s, input_tokens, output_tokens, scores)
            self.n = int(keep["n"])
            self.stages = int(keep["stages"])
        else:
            self.arrival_s = np.ascontiguousarray(arrival_s, dtype=np.float64)
            self.input_tokens = np.ascontiguousarray(input_tokens, dtype=np.float64)
            self.output_tokens = np.ascontiguousarray(output_tokens, dtype=np.float64)
            self.scores = np.ascontiguousarray(scores, dtype=np.float64)
            self.n = int(self.arrival_s.shape[0])
            self.stages = int(self.scores.shape[0]) if self.scores.ndim == 2 else 0

    @staticmethod
    def from_dict(t: dict) -> "TraceBuffers":
        return TraceBuffers(t["arrival_s"], t["input_tokens"], t["output_tokens"], t["scores"])

    def c(self) -> Trace:
        if self.on_device:
            a, i, o, s = self.ptrs
            return Trace(self.n, self.stages, 1, a, i, o, s)
        return Trace(self.n, self.stages, 0, self.arrival_s.ctypes.data, self.input_tokens.ctypes.data,
                     self.output_tokens.ctypes.data, self.scores.ctypes.data)


def _as_trace(trace) -> TraceBuffers:
    if isinstance(trace, TraceBuffers):
        return trace
    return TraceBuffers.from_dict(trace)


def _plan_json(res, idx: int) -> Optional[dict]:
    if idx < 0:
        return None
    p = res.plans[idx]
    reps = [{"tp": int(res.replicas[p.replica_offset + k].tp), "pp": int(res.replicas[p.replica_offset + k].pp)}
            for k in range(p.dp)]
    return {"replicas": reps, "gpus_used": int(p.gpus_used)}


def _sweep_to_json(r: SweepResultC) -> dict:
    C = r.stages
    D = C - 1
    E = r.num_evaluations
    thr = np.ctypeslib.as_array(r.eval_thresholds, shape=(max(1, E * D),))[: E * D].reshape(E, D) \
        if E * D > 0 else np.zeros((E, 0))
    lat = np.ctypeslib.as_array(r.eval_latency, shape=(E,)).copy()
    qual = np.ctypeslib.as_array(r.eval_quality, shape=(E,)).copy()
    ratios = np.ctypeslib.as_array(r.eval_ratios, shape=(E * C,)).reshape(E, C)
    alloc = np.ctypeslib.as_array(r.eval_allocations, shape=(E * C,)).reshape(E, C)
    eplan = np.ctypeslib.as_array(r.eval_plan, shape=(E * C,)).reshape(E, C)
    plan_cache = {}

    def plan_of(i):
        if i not in plan_cache:
            plan_cache[i] = _plan_json(r, int(i))
        return plan_cache[i]

    evals = []
    for e in range(E):
        h = {"thresholds": [float(v) for v in thr[e]]}
        plan = {"allocations": [int(v) for v in alloc[e]],
                "plans": [plan_of(eplan[e, i]) for i in range(C)],
                "thresholds": h,
                "predicted_max_p95_s": float(lat[e]),
                "predicted_quality": float(qual[e]),
                "processing_ratios": [float(v) for v in ratios[e]]}
        evals.append({"latency_s": float(lat[e]), "quality": float(qual[e]), "thresholds": h, "plan_ref": plan})
    W = r.num_weights
    weights = [{"lambda1": float(r.weights[2 * k]), "lambda2": float(r.weights[2 * k + 1])} for k in range(W)]
    sel = [int(r.weight_selection[k]) for k in range(W)]
    front = [evals[int(r.front[k])] for k in range(r.front_size)]
    S = r.num_skipped
    skipped = [{"thresholds": [float(r.skipped_thresholds[s * D + d]) for d in range(D)]} for s in range(S)]
    return {"front": {"points": front}, "evaluations": evals, "weights": weights,
            "weight_selection": sel, "utopia": {"z1_star": float(r.z1_star), "z2_star": float(r.z2_star)},
            "skipped": skipped}


def _stats_dict(s: SweepStats) -> dict:
    return {name: getattr(s, name) for name, _ in SweepStats._fields_}


def _sweep_config_c(cfg: Optional[dict]):
    cfg = cfg or {}
    grid = cfg.get("threshold_grid") or []
    sizes = (ctypes.c_int64 * max(1, len(grid)))(*[len(g) for g in grid])
    flat = [float(v) for g in grid for v in g]
    vals = (ctypes.c_double * max(1, len(flat)))(*flat)
    c = SweepConfigC(len(grid), sizes, vals, float(cfg.get("weight_ratio_min", 0.1)),
                     float(cfg.get("weight_ratio_max", 10.0)), int(cfg.get("weight_count", 9)))
    return c, (sizes, vals)


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the engine library (rank 0 of a multi-process sweep)."""
    L = library()
    n = L.cg_nccl_unique_id_bytes()
    buf = ctypes.create_string_buffer(n)
    _check(L.cg_nccl_unique_id(buf, n))
    return buf.raw


class Engine:
    """One engine per GPU (cg_engine), or with `devices` one engine over
    several GPUs of this process (cg_engine_create_multi: NCCL clique, sharded
    sweeps)."""

    def __init__(self, device: int = 0, devices: Optional[Sequence[int]] = None):
        self._lib = library()
        h = ctypes.c_void_p()
        if devices is not None:
            arr = (ctypes.c_int32 * len(devices))(*[int(d) for d in devices])
            _check(self._lib.cg_engine_create_multi(arr, len(devices), ctypes.byref(h)))
        else:
            _check(self._lib.cg_engine_create(int(device), ctypes.byref(h)))
        self._h = h
        self._ag_keep = None
        self.last_stats: dict = {}

    def close(self):
        if getattr(self, "_h", None):
            self._lib.cg_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stream_handle(self) -> int:
        """cudaStream_t of the engine (all work of a call runs on it)."""
        return int(self._lib.cg_engine_stream(self._h) or 0)

    def set_option(self, key: str, value: int):
        _check(self._lib.cg_engine_set_option(self._h, key.encode(), int(value)))

    def device_count(self) -> int:
        return int(self._lib.cg_engine_device_count(self._h))

    def set_nccl(self, unique_id: bytes, rank: int, world: int) -> None:
        """Joins an NCCL communicator (one process per GPU); the library then
        runs the sweep's all-gathers itself on the engine's stream."""
        _check(self._lib.cg_engine_set_nccl(self._h, unique_id, int(rank), int(world)))

    def set_collective(self, rank: int, world: int, allgather) -> None:
        """allgather(send_ptr, recv_ptr, nbytes) -> None, device pointers."""
        def _cb(send, recv, nbytes, user):
            try:
                allgather(int(send), int(recv), int(nbytes))
                return 0
            except Exception:  # reported as a CUDA error by the engine
                import traceback
                traceback.print_exc()
                return 1
        fn = ALLGATHER_FN(_cb)
        self._ag_keep = fn
        _check(self._lib.cg_engine_set_collective(self._h, int(rank), int(world), fn, None))

    # -- cascade::outerplan::sweep
    def sweep(self, trace, models, hw: dict, params: Optional[dict], total_gpus: int,
              cfg: Optional[dict] = None, raw: bool = False, files: bool = False):
        """files=True also renders sweep.json / front.json on the GPU exactly as
        cmd_plan writes them (dump(2) + "\\n") into self.last_files."""
        tb = _as_trace(trace)
        tc = tb.c()
        marr, keep = models_c(models)
        hwc = hardware_c(hw)
        pc = params_c(params)
        cc, keep2 = _sweep_config_c(cfg)
        out = ctypes.POINTER(SweepResultC)()
        st = self._lib.cg_sweep(self._h, ctypes.byref(tc), marr, len(models), ctypes.byref(hwc),
                                ctypes.byref(pc), int(total_gpus), ctypes.byref(cc), ctypes.byref(out))
        _check(st)
        try:
            r = out.contents
            self.last_stats = _stats_dict(r.stats)
            if files:
                self.last_files = {"sweep.json": self._result_text(out, 2, 0) + "\n",
                                   "front.json": self._result_text(out, 2, 1) + "\n"}
            if raw:
                return None
            return _sweep_to_json(r)
        finally:
            self._lib.cg_sweep_result_free(out)

    def _result_text(self, res_ptr, indent: int, what: int) -> str:
        p = ctypes.c_void_p()
        n = ctypes.c_int64()
        _check(self._lib.cg_sweep_result_json(self._h, res_ptr, int(indent), int(what), JSON_FLAGS,
                                              ctypes.byref(p), ctypes.byref(n)))
        try:
            return ctypes.string_at(p, n.value).decode()
        finally:
            self._lib.cg_text_free(p)

    # -- cascade::read_trace_jsonl (trace ingest on the GPU)
    def read_trace_jsonl(self, path: str) -> dict:
        """SoA trace dict (arrival_s, input_tokens, output_tokens[C][n], scores[C][n])."""
        out = ctypes.POINTER(TraceBufferC)()
        _check(self._lib.cg_read_trace_jsonl(self._h, os.fsencode(path), ctypes.byref(out)))
        return self._take_trace(out)

    def ingest_to_device(self, path: str) -> "TraceBuffers":
        """Ingest into HBM and return the device-resident columns (engine-owned,
        valid until the next ingest on this engine) for sweep()/route_grid()."""
        out = ctypes.POINTER(TraceBufferC)()
        _check(self._lib.cg_read_trace_jsonl(self._h, os.fsencode(path), ctypes.byref(out)))
        try:
            b = out.contents
            d = b.device
            self.last_ingest = {name: getattr(b.stats, name) for name, _ in IngestStats._fields_}
            return TraceBuffers(d.arrival_s, d.input_tokens, d.output_tokens, d.scores, on_device=True,
                                keep={"n": int(d.n), "stages": int(d.stages)})
        finally:
            self._lib.cg_trace_buffer_free(out)

    def parse_trace_jsonl(self, data: bytes, path: str = "<memory>") -> dict:
        out = ctypes.POINTER(TraceBufferC)()
        _check(self._lib.cg_parse_trace_jsonl(self._h, data, len(data), path.encode(), ctypes.byref(out)))
        return self._take_trace(out)

    def _take_trace(self, out) -> dict:
        try:
            b = out.contents
            n, C = int(b.host.n), int(b.host.stages)

            def col(ptr, count):
                if count == 0:
                    return np.zeros(0)
                return np.ctypeslib.as_array(ctypes.cast(ptr, _DP), shape=(count,)).copy()
            self.last_ingest = {name: getattr(b.stats, name) for name, _ in IngestStats._fields_}
            return {"arrival_s": col(b.host.arrival_s, n), "input_tokens": col(b.host.input_tokens, n),
                    "output_tokens": col(b.host.output_tokens, C * n).reshape(C, n),
                    "scores": col(b.host.scores, C * n).reshape(C, n)}
        finally:
            self._lib.cg_trace_buffer_free(out)

    # -- cascade::sim::run / sim::compare (validation simulator)
    def _simulate(self, trace, plans, models, hw, params, cfg, compare):
        tb = _as_trace(trace)
        tc = tb.c()
        marr, keep = models_c(models)
        hwc = hardware_c(hw)
        pc = params_c(params)
        sc, keep_s = sim_config_c(cfg)
        conv = [cascade_plan_c(p) for p in plans]
        parr = (CascadePlanC * max(1, len(conv)))(*[c for c, _ in conv])
        out = ctypes.POINTER(SimResultC)()
        _check(self._lib.cg_simulate(self._h, ctypes.byref(tc), marr, len(models), ctypes.byref(hwc),
                                     ctypes.byref(pc), ctypes.byref(sc), parr, len(conv), 1 if compare else 0,
                                     ctypes.byref(out)))
        try:
            r = out.contents
            self.last_sim = {"gpu_launches": int(r.gpu_launches), "ms_total": float(r.ms_total)}
            return [_sim_report_json(r.reports[i], int(r.n)) for i in range(r.num_reports)]
        finally:
            self._lib.cg_sim_result_free(out)

    def simulate(self, plan: dict, trace, models, hw: dict, params: Optional[dict] = None,
                 cfg: Optional[dict] = None) -> dict:
        """sim::run -> json(SimReport)."""
        return self._simulate(trace, [plan], models, hw, params, cfg, False)[0]

    def simulate_many(self, plans, trace, models, hw: dict, params: Optional[dict] = None,
                      cfg: Optional[dict] = None) -> list:
        """sim::run of every plan (independent runs, one GPU batch)."""
        return self._simulate(trace, plans, models, hw, params, cfg, False)

    def compare(self, plans, trace, models, hw: dict, params: Optional[dict] = None,
                cfg: Optional[dict] = None) -> dict:
        """sim::compare -> json(CompareResult)."""
        reps = self._simulate(trace, plans, models, hw, params, cfg, True)
        return {"rows": [{"p95_s": r["p95_s"], "throughput_rps": r["throughput_rps"],
                          "min_scale_95": r["min_scale_95"]} for r in reps], "reports": reps}

    # -- cli::cmd_drift windowing (drift detection) and compute_baseline
    def drift_windows(self, stream, baseline: dict, policy: Optional[dict] = None) -> dict:
        """{"windows": [...], "drift_detected": bool} in drift_report.json's schema."""
        policy = dict({"window_requests": 100, "window_interval_s": 600.0, "rel_tolerance": 0.2}, **(policy or {}))
        tb = _as_trace(stream)
        tc = tb.c()
        h1 = baseline.get("h1")
        bc = DriftStatsC(float(baseline["arrival_rate"]), float(baseline["mean_input_tokens"]),
                         float(baseline["mean_output_tokens"]), float(baseline["stage1_accept_rate"]),
                         0 if h1 is None else 1, 0.0 if h1 is None else float(h1))
        pc = DriftPolicyC(int(policy["window_requests"]), float(policy["window_interval_s"]),
                          float(policy["rel_tolerance"]))
        out = ctypes.POINTER(DriftResultC)()
        _check(self._lib.cg_drift_windows(self._h, ctypes.byref(tc), ctypes.byref(bc), ctypes.byref(pc),
                                          ctypes.byref(out)))
        try:
            r = out.contents
            wins = []
            for i in range(r.num_windows):
                w = r.windows[i]
                wins.append({"start_s": w.start_s, "span_s": w.span_s, "requests": int(w.requests),
                             "sampled": int(w.sampled), "stats": _drift_stats_json(w.stats),
                             "deviations": {DRIFT_STATS[q]: (None if w.deviation_is_null[q] else w.deviation[q])
                                            for q in range(4)},
                             "drifted_stats": [DRIFT_STATS[q] for q in range(4) if w.drifted[q]],
                             "any_drift": bool(w.any_drift)})
            return {"windows": wins, "drift_detected": bool(r.drift_detected)}
        finally:
            self._lib.cg_drift_result_free(out)

    def compute_baseline(self, trace, h1: Optional[float] = None) -> dict:
        tb = _as_trace(trace)
        tc = tb.c()
        out = DriftStatsC()
        _check(self._lib.cg_trace_baseline(self._h, ctypes.byref(tc), 0 if h1 is None else 1,
                                           0.0 if h1 is None else float(h1), ctypes.byref(out)))
        return _drift_stats_json(out)

    # -- cascade::routing::route_trace
    def route_trace(self, trace, thresholds: Sequence[float], deployed: Sequence[bool],
                    with_accept: bool = False) -> dict:
        tb = _as_trace(trace)
        tc = tb.c()
        C = tb.stages
        h = (ctypes.c_double * max(1, C))(*[float(v) for v in thresholds])
        dep = (ctypes.c_int32 * max(1, C))(*[1 if d else 0 for d in deployed])
        out = RouteResultC()
        acc = (ctypes.c_int32 * tb.n)() if with_accept else None
        _check(self._lib.cg_route(self._h, ctypes.byref(tc), h, dep, ctypes.byref(out), acc))
        res = {"ratios": [out.ratios[i] for i in range(C)],
               "stage_workloads": [{"arrival_rate": out.stage_workloads[i].arrival_rate,
                                    "mean_input_tokens": out.stage_workloads[i].mean_input_tokens,
                                    "mean_output_tokens": out.stage_workloads[i].mean_output_tokens,
                                    "p95_input_tokens": out.stage_workloads[i].p95_input_tokens,
                                    "p95_output_tokens": out.stage_workloads[i].p95_output_tokens}
                                   for i in range(C)],
               "quality": out.quality}
        if with_accept:
            res["per_request_accept_stage"] = list(acc)
        return res

    # -- batched route_trace over a threshold grid (the sweep's routing phase)
    def route_grid(self, trace, cfg: Optional[dict] = None) -> list:
        tb = _as_trace(trace)
        tc = tb.c()
        cc, keep2 = _sweep_config_c(cfg)
        out = ctypes.POINTER(RouteGridResultC)()
        _check(self._lib.cg_route_grid(self._h, ctypes.byref(tc), ctypes.byref(cc), ctypes.byref(out)))
        try:
            r = out.contents
            self.last_stats = _stats_dict(r.stats)
            C, K, D = r.stages, r.num_candidates, r.stages - 1
            keys = ["arrival_rate", "mean_input_tokens", "mean_output_tokens", "p95_input_tokens",
                    "p95_output_tokens"]
            res = []
            for c in range(K):
                res.append({"thresholds": [r.thresholds[c * D + d] for d in range(D)],
                            "ratios": [r.ratios[c * C + i] for i in range(C)],
                            "stage_workloads": [{k: getattr(r.workloads[c * C + i], k) for k in keys}
                                                for i in range(C)],
                            "quality": r.quality[c]})
            return res
        finally:
            self._lib.cg_route_grid_result_free(out)

    # -- cascade::costmodel::StageEvaluator::row
    def row(self, hw: dict, params: Optional[dict], model: dict, workload: dict, max_budget: int) -> dict:
        marr, keep = models_c([model])
        w = Workload(float(workload["arrival_rate"]), float(workload["mean_input_tokens"]),
                     float(workload["mean_output_tokens"]), float(workload["p95_input_tokens"]),
                     float(workload["p95_output_tokens"]))
        hwc = hardware_c(hw)
        pc = params_c(params)
        out = ctypes.POINTER(RowResultC)()
        _check(self._lib.cg_stage_row(self._h, marr, ctypes.byref(w), ctypes.byref(hwc), ctypes.byref(pc),
                                      int(max_budget), ctypes.byref(out)))
        try:
            r = out.contents
            self.last_stats = _stats_dict(r.stats)
            lat = [r.latency[f] for f in range(r.max_budget + 1)]
            plans = [_plan_json(r, int(r.plan_index[f])) for f in range(r.max_budget + 1)]
            return {"latency": [None if math.isinf(v) else v for v in lat], "plan": plans}
        finally:
            self._lib.cg_row_result_free(out)

    # -- cascade::innerplan::solve_min_max
    def solve_min_max(self, table: dict, total_gpus: int) -> dict:
        n = int(table["gpu_budget"])
        rows = table["entries"]
        C = len(rows)
        flat = [math.inf if v is None else float(v) for row in rows for v in row]
        if any(len(row) != n + 1 for row in rows):
            raise CascadeError(0, "latency table: row length != N+1")
        ent = (ctypes.c_double * max(1, len(flat)))(*flat)
        alloc = (ctypes.c_int32 * max(1, C))()
        per = (ctypes.c_double * max(1, C))()
        L = ctypes.c_double()
        _check(self._lib.cg_solve_min_max(self._h, ent, C, n, int(total_gpus), alloc, per, ctypes.byref(L)))
        return {"allocations": [alloc[i] for i in range(C)], "objective_L": L.value,
                "per_stage_latency": [per[i] for i in range(C)]}


def generate_trace(spec: dict, seed: int) -> dict:
    """cascade::cli::generate_trace with bit-identical output (host code)."""
    L = library()
    n = int(spec["count"])
    c = len(spec["stages"])
    arr = np.zeros(max(n, 1))
    inp = np.zeros(max(n, 1))
    out = np.zeros(max(n * c, 1))
    sc = np.zeros(max(n * c, 1))
    no = ctypes.c_int64()
    so = ctypes.c_int32()
    P = lambda a: a.ctypes.data_as(_DP)  # noqa: E731
    _check(L.cg_generate_trace(json.dumps(spec).encode(), int(seed), P(arr), P(inp), P(out), P(sc),
                               max(n, 0), ctypes.byref(no), ctypes.byref(so)))
    return {"arrival_s": arr[:n], "input_tokens": inp[:n], "output_tokens": out[: n * c].reshape(c, n),
            "scores": sc[: n * c].reshape(c, n)}


def shard_row_plans(num_plans, row: int, rank: int, world: int):
    """Plan ranges [(lo, hi), ...] of row `row` that `rank` evaluates in a
    sharded call over rows with `num_plans` plans (the device filter's chunk
    mapping, cg_shard_row_plans)."""
    L = library()
    U64 = ctypes.POINTER(ctypes.c_uint64)
    npl = np.ascontiguousarray(num_plans, dtype=np.uint64)
    n = L.cg_shard_row_plans(npl.ctypes.data_as(U64), len(npl), int(row), int(rank), int(world), None, 0)
    if n < 0:
        raise CascadeError(0, "invalid shard arguments")
    out = np.zeros(max(1, 2 * n), dtype=np.uint64)
    L.cg_shard_row_plans(npl.ctypes.data_as(U64), len(npl), int(row), int(rank), int(world),
                         out.ctypes.data_as(U64), n)
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(n)]


def merge_budget_bests(hw: dict, params: Optional[dict], model: dict, max_budget: int, lat_bits, plan_index):
    """Per-budget best over partial results (merge rule only, no prefix min)."""
    L = library()
    lat = np.ascontiguousarray(lat_bits, dtype=np.uint64).reshape(-1)
    idx = np.ascontiguousarray(plan_index, dtype=np.uint64).reshape(-1)
    shards = lat.size // (max_budget + 1)
    marr, keep = models_c([model])
    hwc, pc = hardware_c(hw), params_c(params)
    lo = np.zeros(max_budget + 1, dtype=np.uint64)
    po = np.zeros(max_budget + 1, dtype=np.uint64)
    U64 = ctypes.POINTER(ctypes.c_uint64)
    _check(L.cg_merge_budget_bests(marr, ctypes.byref(hwc), ctypes.byref(pc), int(max_budget), int(shards),
                                   lat.ctypes.data_as(U64), idx.ctypes.data_as(U64), lo.ctypes.data_as(U64),
                                   po.ctypes.data_as(U64)))
    return lo, po


def merge_row_shards(hw: dict, params: Optional[dict], model: dict, max_budget: int, lat_bits, plan_index) -> dict:
    """Host-side merge of per-shard per-budget bests (no GPU), the rule the
    multi-GPU path applies after its all-gather, then the prefix minimum."""
    L = library()
    lat = np.ascontiguousarray(lat_bits, dtype=np.uint64).reshape(-1)
    idx = np.ascontiguousarray(plan_index, dtype=np.uint64).reshape(-1)
    shards = lat.size // (max_budget + 1)
    marr, keep = models_c([model])
    hwc, pc = hardware_c(hw), params_c(params)
    out = ctypes.POINTER(RowResultC)()
    U64 = ctypes.POINTER(ctypes.c_uint64)
    _check(L.cg_merge_row_shards(marr, ctypes.byref(hwc), ctypes.byref(pc), int(max_budget), int(shards),
                                 lat.ctypes.data_as(U64), idx.ctypes.data_as(U64), ctypes.byref(out)))
    try:
        r = out.contents
        lats = [r.latency[f] for f in range(r.max_budget + 1)]
        return {"latency": [None if math.isinf(v) else v for v in lats],
                "plan": [_plan_json(r, int(r.plan_index[f])) for f in range(r.max_budget + 1)]}
    finally:
        L.cg_row_result_free(out)


def concat_traces(parts: Sequence[dict]) -> dict:
    """Concatenates trace segments with time offsets (bursty traces, C3)."""
    from . import workloads
    return workloads.concat_traces(parts)


_default_engine: Optional[Engine] = None


def default_engine() -> Engine:
    global _default_engine
    if _default_engine is None:
        _default_engine = Engine(0)
    return _default_engine


def sweep(trace, models, hw, params, total_gpus, cfg=None) -> dict:
    return default_engine().sweep(trace, models, hw, params, total_gpus, cfg)


def route_trace(trace, thresholds, deployed) -> dict:
    return default_engine().route_trace(trace, thresholds, deployed)


def read_trace_jsonl(path: str) -> dict:
    return default_engine().read_trace_jsonl(path)


def solve_min_max(table: dict, total_gpus: int) -> dict:
    return default_engine().solve_min_max(table, total_gpus)


class StageEvaluator:
    def __init__(self, hw: dict, params: Optional[dict] = None, engine: Optional[Engine] = None):
        self.hw = hw
        self.params = params
        self.engine = engine or default_engine()

    def row(self, model: dict, w: dict, max_budget: int) -> dict:
        return self.engine.row(self.hw, self.params, model, w, max_budget)
