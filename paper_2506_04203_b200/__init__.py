"""B200-native batched candidate-plan evaluation for the Cascade Planner's
bi-level scheduler (arXiv 2506.04203): the body of cascade::outerplan::sweep
as sm_100a CUDA kernels behind a C ABI (include/cascade_gpu.h)."""
from .engine import (CascadeError, Engine, StageEvaluator, concat_traces, generate_trace, route_trace,
                     solve_min_max, sweep)

__all__ = ["CascadeError", "Engine", "StageEvaluator", "concat_traces", "generate_trace", "route_trace",
           "solve_min_max", "sweep"]
