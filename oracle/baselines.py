"""ORACLE for the comparison planners and the lookup table — TEST
INFRASTRUCTURE ONLY (see oracle/__init__).  Plain Python, exact integers / Fractions.

  min_cu_threshold     SPEC S:80-88: smallest size c with t(c) <= (1 + tol) t(max)
                       ("minimum number of CUs needed without experiencing noticeable slowdown",
                        PAPER §IV-B)
  model_wise_rightsize SPEC S:90-98: smallest size c with sum_k t_k(c) <= factor sum_k t_k(max)
                       (Model-Wise right-sizing, PAPER §V; factor 3 = "3x the tail latency
                        when running in isolation")
  baseline plans       Baseline: every kernel at the largest size ("default stream that
                       uses all 60 CUs"); Model-Wise; Kernel-Wise (every kernel at its threshold,
                       KW^IOCTL / KW^Prealloc differ only at run time)
  lookup table         SPEC S:225-233: JSON {meta: {hash, mode, switch_max},
                       workers: [{worker_id, configs}]}; hash = 64-bit FNV-1a over the canonical
                       serialization without the hash field.
Tolerances / factors are the rationals round(x 1e9) / 1e9 so the predicates are exact.
"""
from __future__ import annotations

import json
from fractions import Fraction
from typing import List, Optional, Sequence

from . import brute

FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3


def fnv1a64(data: bytes) -> int:
    h = FNV_OFFSET
    for b in data:
        h ^= b
        h = (h * FNV_PRIME) & 0xFFFFFFFFFFFFFFFF
    return h


def _rat(x: float) -> Fraction:
    return Fraction(int(round(x * 1e9)), 10**9)


def min_cu_threshold(times: Sequence[int], allowed: Sequence[int], tol: float) -> int:
    """index (into the size columns) of the smallest allowed size meeting the threshold"""
    jmax = max(allowed)
    lim = (1 + _rat(tol)) * times[jmax]
    for j in sorted(allowed):
        if times[j] <= lim:
            return j
    return jmax


def model_wise_rightsize(group_times: Sequence[Sequence[int]], allowed: Sequence[int], factor: float) -> int:
    jmax = max(allowed)
    tot = lambda j: sum(t[j] for t in group_times)
    lim = _rat(factor) * tot(jmax)
    for j in sorted(allowed):
        if tot(j) <= lim:
            return j
    return jmax


KINDS = {"all_max": 0, "model_wise": 1, "kernel_wise": 2}


def baseline_columns(problem, kind: str, param: float) -> List[List[int]]:
    """per worker, the size column chosen for every kernel group"""
    p = problem
    C = len(p.sizes)
    cols = []
    for w in range(p.W):
        m = p.models[p.model_ids[w]]
        gb = p.group_bounds[w] if p.group_bounds is not None and p.group_bounds[w] is not None else \
            list(range(m.n_kernels + 1))
        G = len(gb) - 1
        beta = [[int(m.exec_ns[gb[g]:gb[g + 1], j].sum()) for j in range(C)] for g in range(G)]
        mask = p.allowed_mask[w] if p.allowed_mask is not None else (1 << C) - 1
        allowed = [j for j in range(C) if (mask >> j) & 1]
        if kind == "all_max":
            cols.append([max(allowed)] * G)
        elif kind == "model_wise":
            cols.append([model_wise_rightsize(beta, allowed, param)] * G)
        else:
            cols.append([min_cu_threshold(beta[g], allowed, param) for g in range(G)])
    return cols


def evaluate_columns(problem, cols):
    """exact evaluation (oracle.brute.evaluate) of a fixed plan; returns dict"""
    p = problem
    choice = []
    for w in range(p.W):
        m = p.models[p.model_ids[w]]
        gb = p.group_bounds[w] if p.group_bounds is not None and p.group_bounds[w] is not None else \
            list(range(m.n_kernels + 1))
        S = sum((gb[g + 1] - gb[g]) * p.sizes[cols[w][g]] for g in range(len(gb) - 1))
        B = sum(int(m.exec_ns[k, cols[w][g]]) for g in range(len(gb) - 1) for k in range(gb[g], gb[g + 1]))
        choice.append((tuple(cols[w]), S, B))
    feas, key, L, pw, al = brute.evaluate(p, choice)
    return dict(feasible=feas, key=key, L=L, power=pw, alpha=al,
                switches=[brute.switch_count(c) for c in cols],
                group_sm=[[p.sizes[j] for j in c] for c in cols])


def lookup_table(problem, group_sm: Sequence[Sequence[int]], mode: Optional[str] = None):
    """(canonical bytes, JSON text, hash) of the lookup table: every kernel of every worker ->
    its pool size (a group's size for each of its kernels)."""
    p = problem
    workers = []
    for w in range(p.W):
        m = p.models[p.model_ids[w]]
        gb = p.group_bounds[w] if p.group_bounds is not None and p.group_bounds[w] is not None else \
            list(range(m.n_kernels + 1))
        cfg = []
        for g in range(len(gb) - 1):
            cfg.extend([int(group_sm[w][g])] * (gb[g + 1] - gb[g]))
        workers.append({"worker_id": w, "configs": cfg})
    mode = mode or p.mode
    canon = json.dumps({"meta": {"mode": mode, "switch_max": p.switch_max}, "workers": workers},
                       separators=(",", ":")).encode()
    h = fnv1a64(canon)
    text = json.dumps({"meta": {"hash": f"0x{h:016x}", "mode": mode, "switch_max": p.switch_max},
                       "workers": workers}, separators=(",", ":"))
    return canon, text, h
