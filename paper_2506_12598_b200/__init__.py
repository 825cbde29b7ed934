"""B200-native ECLIP resource-allocation planner (arXiv 2506.12598, §IV-B).

The hot path lives in libeclip.so (CUDA for sm_100a behind the C-ABI of include/eclip.h);
this package is its thin Python binding (eclip.py) plus the multi-GPU protocol
(parallel.py).  Build with `python -m paper_2506_12598_b200.build`.
"""
from .eclip import (EclipError, Profiles, Plan, Session, Planner, Comm, plan, plan_batch, plan_problem, alloc_batch_out, lib,
                    baseline_plan, lookup_table_json, simulate, level_table, BASELINES, MODES, OBJECTIVES, EXPORTS)

__all__ = ["EclipError", "Profiles", "Plan", "Session", "Planner", "Comm", "plan", "plan_batch", "plan_problem", "alloc_batch_out",
           "baseline_plan", "lookup_table_json", "simulate", "level_table", "BASELINES", "lib", "MODES", "OBJECTIVES", "EXPORTS"]
