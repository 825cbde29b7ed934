"""O-A: the literal definition, by brute force over every raw joint plan, in exact
rational arithmetic (fractions.Fraction).  TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Follows PAPER.md §IV-B term by term, for tiny instances:
  x_{k,c}: one configuration per kernel group
  switchTotal_w = sum_k sum_c |x_{k,c} - x_{k-1,c}| / 2 <= switchMax
  beta_k = profile[c_k]
  CUAverage_w = sum_k c_k / #kernels_w
  CUOverlap_w = per slowdown mode (P:314 and readings c3-O / c3-M)
  alpha_w = CUOverlap_w / total#CUs ;  e_k = beta_k (1 + alpha_w)
  objective: SUM_w omega_w sum_{k in w} e_k (equal weights omega = 1; SPEC S:130 per-worker
  weights, reading R20), or MAX_w omega_w sum_k e_k, or ENERGY =
  power x makespan, power = p_idle + (p_max - p_idle) min(1, sum_w CUAverage_w / N)
  (SPEC power_at S:406-409 applied to the paper's CUAverage abstraction).
  QoS (optional): sum_{k in w} e_k <= Q_w.
Selection: candidates are joint plans whose every worker plan is the
canonical witness of its level (min B at its CU-sum, lexicographically smallest among
those); ordered lexicographically (worker 0, group 0 most significant); m = exact min;
winner = first candidate with key <= m (1 + tau).
"""
from __future__ import annotations

import itertools
from fractions import Fraction
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np


def switch_count(configs: Sequence[int]) -> int:
    """Number of adjacent pairs with differing configs."""
    if len(configs) == 0:
        raise ValueError("empty list")
    return sum(1 for k in range(1, len(configs)) if configs[k] != configs[k - 1])


def switch_count_indicator(configs: Sequence[int], allowed: Sequence[int]) -> int:
    """sum_k sum_c |x_{k,c} - x_{k-1,c}| / 2 (indicator-matrix form)."""
    x = [[1 if cfg == c else 0 for c in allowed] for cfg in configs]
    tot = sum(abs(x[k][i] - x[k - 1][i]) for k in range(1, len(x)) for i in range(len(allowed)))
    assert tot % 2 == 0
    return tot // 2


def estimate_exec(beta, alpha):
    """e = beta (1 + alpha)."""
    return beta * (1 + alpha)


def cu_overlap(averages: Sequence, w: int, mode: str, total: int, M=None):
    """CUOverlap_w (S:162-173 modes; c3-M matrix)."""
    if mode == "paper":
        return averages[w] + sum(a for v, a in enumerate(averages) if v != w)
    if mode == "exclude_self":
        return sum(a for v, a in enumerate(averages) if v != w)
    if mode == "excess":
        return max(Fraction(0), sum(averages) - total)
    if mode == "matrix":
        return sum(Fraction(float(M[w][v])) * a for v, a in enumerate(averages) if v != w)
    raise ValueError(mode)


def alpha(overlap, total):
    """alpha = overlap / total CUs."""
    return Fraction(overlap) / total


def weight_values(weights, W):
    """omega_w as exact rationals round-half-up(omega_w x 1e6 in binary64) / 1e6 (reading R20;
    SPEC S:130: strictly positive, default all 1)."""
    from decimal import Decimal, ROUND_HALF_UP
    if weights is None:
        return [Fraction(1)] * W
    return [Fraction(int(Decimal(float(x) * 1e6).quantize(Decimal(1), rounding=ROUND_HALF_UP)), 10**6)
            for x in weights]


def busy_energy(group_sm, group_lat, total, p_idle, p_max):
    """Busy-SM energy integral of a plan's predicted co-located run (SPEC integrate_energy S:416-419,
    power_at S:406-409; reading R21): every worker starts at t = 0 and runs its groups back to back,
    group g of worker w occupying group_sm[w][g] SMs for group_lat[w][g]; busy(t) = min(N, sum of the
    running groups' SMs); E = integral over [0, makespan] of p_idle + (p_max - p_idle) busy(t) / N.
    Exact when the inputs are Fractions.  Returns joules per ns-unit (the caller scales)."""
    W = len(group_sm)
    ends = []                           # per worker: group end times
    for w in range(W):
        t, e = 0, []
        for d in group_lat[w]:
            t = t + d
            e.append(t)
        ends.append(e)
    cuts = sorted({0} | {x for e in ends for x in e})
    E = 0
    for a, b in zip(cuts, cuts[1:]):
        busy = 0
        for w in range(W):
            start = 0
            for g, end in enumerate(ends[w]):
                if start <= a and b <= end and end > start:
                    busy += group_sm[w][g]
                    break
                start = end
        E += (p_idle + (p_max - p_idle) * Fraction(min(busy, total), total)) * (b - a)
    return E


def power_at(busy, total, p_idle, p_max):
    """p_idle + (p_max - p_idle) * min(1, busy / total) (capped per c3-E)."""
    frac = min(Fraction(1), Fraction(busy) / total)
    return Fraction(p_idle) + (Fraction(p_max) - Fraction(p_idle)) * frac


def _worker_plans(exec_ns: np.ndarray, bounds, sizes, mask, R):
    K = exec_ns.shape[0]
    if bounds is None:
        bounds = list(range(K + 1))
    G = len(bounds) - 1
    allowed = [j for j in range(len(sizes)) if (mask >> j) & 1]
    plans = []
    for sig in itertools.product(allowed, repeat=G):   # lexicographic order
        if switch_count(sig) > R:
            continue
        S = sum((bounds[g + 1] - bounds[g]) * sizes[sig[g]] for g in range(G))
        B = sum(int(exec_ns[k, sig[g]]) for g in range(G) for k in range(bounds[g], bounds[g + 1]))
        plans.append((sig, S, B))
    return plans, K, bounds


def canonical(plans):
    """level S -> (B*, witness): min B, then lexicographically smallest sigma."""
    best: Dict[int, Tuple[int, tuple]] = {}
    for sig, S, B in plans:
        if S not in best or (B, sig) < best[S]:
            best[S] = (B, sig)
    return best


def evaluate(problem, choice):
    """Exact evaluation of a joint plan: choice[w] = (sigma, S, B).  Returns
    (feasible, key, L list, power, alpha list)."""
    p = problem
    W = p.W
    Ks = []
    for w in range(W):
        m = p.models[p.model_ids[w]]
        Ks.append(m.n_kernels)
    avg = [Fraction(choice[w][1], Ks[w]) for w in range(W)]
    L, al = [], []
    feas = True
    for w in range(W):
        ov = cu_overlap(avg, w, p.mode, p.total_sms, p.slowdown_matrix)
        a = alpha(ov, p.total_sms)
        Lw = estimate_exec(Fraction(choice[w][2]), a)
        L.append(Lw); al.append(a)
        if p.qos_ns is not None and p.qos_ns[w] != float("inf") and Lw > Fraction(p.qos_ns[w]):
            feas = False
    pw = power_at(sum(avg), p.total_sms, Fraction(float(np.float32(p.p_idle_w))), Fraction(float(np.float32(p.p_max_w))))
    om = weight_values(getattr(p, "weights", None), W)
    if p.objective == "sum":
        key = sum(o * x for o, x in zip(om, L))
    elif p.objective == "max":
        key = max(o * x for o, x in zip(om, L))
    else:
        key = pw * max(L)
    return feas, key, L, pw, al


def brute_force(problem, tol: float = 1e-5, level_efficient: bool = True, max_joint: int = 2_000_000):
    """Returns None if infeasible, else dict(sigmas, key, min_key, L, power, alpha, rank)."""
    p = problem
    W = p.W
    C = len(p.sizes)
    per = []
    for w in range(W):
        m = p.models[p.model_ids[w]]
        gb = p.group_bounds[w] if p.group_bounds is not None else None
        mask = p.allowed_mask[w] if p.allowed_mask is not None else (1 << C) - 1
        plans, K, bounds = _worker_plans(m.exec_ns, gb, p.sizes, mask, p.switch_max)
        if level_efficient:
            can = canonical(plans)
            plans = sorted([(sig, S, B) for S, (B, sig) in can.items()])
        per.append(plans)
    total = 1
    for pl in per:
        total *= len(pl)
    if total > max_joint:
        raise ValueError(f"instance too large for brute force: {total}")
    cands = []
    for choice in itertools.product(*per):   # lexicographic in the concatenated sigmas
        feas, key, L, pw, al = evaluate(p, choice)
        if feas:
            cands.append((choice, key, L, pw, al))
    if not cands:
        return None
    m = min(c[1] for c in cands)
    tau = Fraction(int(round(tol * 1e9)), 10**9)
    for rank, (choice, key, L, pw, al) in enumerate(cands):
        if key <= m * (1 + tau):
            return dict(sigmas=[list(c[0]) for c in choice], key=key, min_key=m, L=L, power=pw,
                        alpha=al, S=[c[1] for c in choice], B=[c[2] for c in choice])
    raise AssertionError("unreachable")
