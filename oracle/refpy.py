"""TEST INFRASTRUCTURE ONLY: ctypes bindings to oracle/_ref/libcascade_ref.so.

The library is the UNMODIFIED reference planner (compiled from
/root/reference/proj/src by oracle/Makefile) plus oracle/ref_harness.cpp.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module; it is the checker and the timed CPU baseline, never the
product path.
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Any

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libcascade_ref.so")
_lib = None

_D = ctypes.POINTER(ctypes.c_double)


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        L = ctypes.CDLL(LIB_PATH)
        L.ref_free.argtypes = [ctypes.c_void_p]
        L.ref_free.restype = None
        for name, args in {
            "ref_sweep": [_D, _D, _D, _D, ctypes.c_int64, ctypes.c_int, ctypes.c_char_p, ctypes.c_int],
            "ref_plan_outputs": [_D, _D, _D, _D, ctypes.c_int64, ctypes.c_int, ctypes.c_char_p,
                                 ctypes.c_int, ctypes.c_char_p],
            "ref_route": [_D, _D, _D, _D, ctypes.c_int64, ctypes.c_int, _D, ctypes.POINTER(ctypes.c_int)],
            "ref_row": [ctypes.c_char_p] * 4 + [ctypes.c_int],
            "ref_solve": [ctypes.c_char_p, ctypes.c_int],
            "ref_export_milp": [ctypes.c_char_p, ctypes.c_int],
            "ref_generate_trace": [ctypes.c_char_p, ctypes.c_uint64, _D, _D, _D, _D, ctypes.c_int64],
            "ref_weight_ladder": [ctypes.c_double, ctypes.c_double, ctypes.c_int],
            "ref_pareto": [_D, _D, ctypes.c_int64],
            "ref_plan_count": [_D, _D, _D, _D, ctypes.c_int64, ctypes.c_int, ctypes.c_char_p, ctypes.c_int],
            "ref_dump_sweep": [ctypes.c_char_p],
            "ref_unique_rows": [_D, _D, _D, _D, ctypes.c_int64, ctypes.c_int, ctypes.c_char_p, ctypes.c_int,
                                ctypes.c_int],
            "ref_drift": [_D, _D, _D, _D, ctypes.c_int64, ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p,
                          ctypes.c_char_p, ctypes.c_int, ctypes.c_double],
            "ref_simulate": [_D, _D, _D, _D, ctypes.c_int64, ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p,
                             ctypes.c_char_p, ctypes.c_int],
            "ref_write_trace_jsonl": [_D, _D, _D, _D, ctypes.c_int64, ctypes.c_int, ctypes.c_char_p],
            "ref_read_trace_jsonl": [ctypes.c_char_p, _D, _D, _D, _D, ctypes.c_int64, ctypes.c_int],
        }.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_void_p
        L.ref_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _call(fn, *args) -> dict:
    p = fn(*args)
    try:
        s = ctypes.string_at(p).decode()
    finally:
        lib().ref_free(p)
    return json.loads(s)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_D)


class RefError(Exception):
    def __init__(self, code: int, code_name: str, message: str):
        super().__init__(f"{code_name}: {message}")
        self.code = code
        self.code_name = code_name
        self.message = message


def _unwrap(res: dict) -> Any:
    if not res["ok"]:
        raise RefError(res["code"], res["code_name"], res["message"])
    return res


def generate_trace(spec: dict, seed: int) -> dict:
    n = int(spec["count"])
    c = len(spec["stages"])
    arr = np.zeros(max(n, 1))
    inp = np.zeros(max(n, 1))
    out = np.zeros(max(n * c, 1))
    sc = np.zeros(max(n * c, 1))
    _unwrap(_call(lib().ref_generate_trace, json.dumps(spec).encode(), seed,
                  _ptr(arr), _ptr(inp), _ptr(out), _ptr(sc), n))
    return {"arrival_s": arr[:n], "input_tokens": inp[:n],
            "output_tokens": out[: n * c].reshape(c, n), "scores": sc[: n * c].reshape(c, n)}


def _trace_args(trace: dict):
    arr = np.ascontiguousarray(trace["arrival_s"], dtype=np.float64)
    inp = np.ascontiguousarray(trace["input_tokens"], dtype=np.float64)
    out = np.ascontiguousarray(trace["output_tokens"], dtype=np.float64)
    sc = np.ascontiguousarray(trace["scores"], dtype=np.float64)
    c = sc.shape[0]
    n = arr.shape[0]
    return (arr, inp, out, sc), n, c


def sweep(trace: dict, config: dict, total_gpus: int) -> dict:
    """Returns {"ok":..., "result": SweepResult JSON, "elapsed_s": t} or raises RefError."""
    keep, n, c = _trace_args(trace)
    return _unwrap(_call(lib().ref_sweep, *map(_ptr, keep), n, c,
                         json.dumps(config).encode(), total_gpus))


def sweep_raw(trace: dict, config: dict, total_gpus: int) -> dict:
    keep, n, c = _trace_args(trace)
    return _call(lib().ref_sweep, *map(_ptr, keep), n, c, json.dumps(config).encode(), total_gpus)


def plan_outputs(trace: dict, config: dict, total_gpus: int, requirement: dict) -> dict:
    keep, n, c = _trace_args(trace)
    return _unwrap(_call(lib().ref_plan_outputs, *map(_ptr, keep), n, c,
                         json.dumps(config).encode(), total_gpus,
                         json.dumps(requirement).encode()))["result"]


def plan_count(trace: dict, config: dict, total_gpus: int) -> dict:
    keep, n, c = _trace_args(trace)
    return _unwrap(_call(lib().ref_plan_count, *map(_ptr, keep), n, c, json.dumps(config).encode(),
                         total_gpus))["result"]


def unique_rows(trace: dict, config: dict, total_gpus: int, threads: int = 0) -> dict:
    """The sweep's unique (stage, WorkloadStats) rows, by the reference's own
    route_trace over every candidate (routed on `threads` threads)."""
    keep, n, c = _trace_args(trace)
    return _unwrap(_call(lib().ref_unique_rows, *map(_ptr, keep), n, c, json.dumps(config).encode(),
                         int(total_gpus), int(threads or os.cpu_count() or 1)))["result"]


def route(trace: dict, thresholds, deployed) -> dict:
    keep, n, c = _trace_args(trace)
    h = np.ascontiguousarray(np.asarray(thresholds, dtype=np.float64).reshape(-1))
    if h.size == 0:
        h = np.zeros(1)
    dep = (ctypes.c_int * c)(*[1 if d else 0 for d in deployed])
    return _unwrap(_call(lib().ref_route, *map(_ptr, keep), n, c, _ptr(h), dep))


def row(hw: dict, params: dict, model: dict, workload: dict, max_budget: int) -> dict:
    return _unwrap(_call(lib().ref_row, json.dumps(hw).encode(), json.dumps(params).encode(),
                         json.dumps(model).encode(), json.dumps(workload).encode(), max_budget))


def solve(table: dict, total_gpus: int) -> dict:
    return _unwrap(_call(lib().ref_solve, json.dumps(table).encode(), total_gpus))


def weight_ladder(rmin: float, rmax: float, count: int) -> list:
    return _unwrap(_call(lib().ref_weight_ladder, rmin, rmax, count))["result"]


def pareto(latency, quality) -> list:
    lat = np.ascontiguousarray(latency, dtype=np.float64)
    q = np.ascontiguousarray(quality, dtype=np.float64)
    return _unwrap(_call(lib().ref_pareto, _ptr(lat), _ptr(q), lat.shape[0]))["result"]


def max_threads() -> int:
    return int(lib().ref_max_threads())


def write_trace_jsonl(trace: dict, path: str) -> None:
    """The reference writer (nlohmann dump of each TraceRecord + '\\n')."""
    keep, n, c = _trace_args(trace)
    _unwrap(_call(lib().ref_write_trace_jsonl, *map(_ptr, keep), n, c, path.encode()))


def read_trace_jsonl(path: str, capacity: int, max_stages: int = 16) -> dict:
    """The reference reader; raises RefError with the reference's code/message."""
    cap = max(1, capacity)
    arr, inp = np.zeros(cap), np.zeros(cap)
    out, sc = np.zeros(cap * max_stages), np.zeros(cap * max_stages)
    res = _unwrap(_call(lib().ref_read_trace_jsonl, path.encode(), _ptr(arr), _ptr(inp), _ptr(out), _ptr(sc),
                        capacity, max_stages))
    n, c = res["result"]["n"], res["result"]["stages"]
    return {"arrival_s": arr[:n], "input_tokens": inp[:n], "output_tokens": out[: n * c].reshape(c, n),
            "scores": sc[: n * c].reshape(c, n), "elapsed_s": res["elapsed_s"]}


def dump_sweep(result: dict) -> dict:
    """The reference's sweep.json / front.json text of a SweepResult (JSON dict),
    plus the time json(res).dump(2) took ("elapsed_s")."""
    res = _unwrap(_call(lib().ref_dump_sweep, json.dumps(result).encode()))
    out = dict(res["result"])
    out["elapsed_s"] = res["elapsed_s"]
    return out


def simulate(trace: dict, config: dict, plans: list, sim_cfg: dict, compare: bool = False) -> dict:
    """sim::run(plans[0]) or sim::compare(plans): {"result": json(report), "elapsed_s": t}."""
    keep, n, c = _trace_args(trace)
    return _unwrap(_call(lib().ref_simulate, *map(_ptr, keep), n, c, json.dumps(config).encode(),
                         json.dumps(plans).encode(), json.dumps(sim_cfg).encode(), 1 if compare else 0))


def drift(trace: dict, config: dict, baseline: dict, work_dir: str, h1=None) -> dict:
    """cmd_drift's drift_report.json ("report") and compute_baseline ("baseline_of_stream")."""
    keep, n, c = _trace_args(trace)
    return _unwrap(_call(lib().ref_drift, *map(_ptr, keep), n, c, json.dumps(config).encode(),
                         json.dumps(baseline).encode(), work_dir.encode(), 0 if h1 is None else 1,
                         0.0 if h1 is None else float(h1)))
