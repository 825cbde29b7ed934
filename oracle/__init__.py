"""ORACLE for the ECLIP resource-allocation optimizer — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  The product (paper_2506_12598_b200/) never imports it, and it
imports nothing from the product; the only shared module is synth/ (seeded inputs).

  oracle.brute   O-A: the literal definition — every raw joint plan, exact Fractions
                 (tiny instances only).  PAPER.md §IV-B; SPEC brute_force_solve
                 S:205-213.
  liboracle.so   O-B: the exact reduced oracle in plain C (oracle/eclip_oracle.c): level
                 tables by memoised recursion, exhaustive level-tuple enumeration, and the
                 T'-slice DP + lexicographic walk; exact integer keys.
  this module    SPEC-format profile parsing, group aggregation,
                 marshalling into O-B, FP64 evaluation of the winner.

Parity status: every function here is pinned by tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
from dataclasses import dataclass, field
from decimal import Decimal, ROUND_HALF_EVEN, ROUND_HALF_UP, InvalidOperation
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "eclip_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

MODES = {"exclude_self": 0, "paper": 1, "excess": 2, "matrix": 3}
OBJECTIVES = {"sum": 0, "max": 1, "energy": 2}
MAXW = 16


def build(force: bool = False) -> str:
    """Compile O-B with gcc (plain C; -ffp-contract=off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-shared", "-fPIC",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Problem(C.Structure):
    _fields_ = [("W", C.c_int32), ("N", C.c_int32), ("mode", C.c_int32), ("objective", C.c_int32),
                ("L", C.POINTER(C.c_int32)), ("S", C.POINTER(C.c_int64)), ("B", C.POINTER(C.c_int64)),
                ("K", C.POINTER(C.c_int64)), ("Q", C.POINTER(C.c_double)), ("M", C.POINTER(C.c_float)),
                ("p_idle", C.c_float), ("p_max", C.c_float), ("tol_num", C.c_int64), ("tol_den", C.c_int64),
                ("wt", C.POINTER(C.c_int64)), ("wval", C.POINTER(C.c_double))]


class _Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("levels", C.c_int32 * MAXW), ("index", C.c_uint64),
                ("key", C.c_uint64 * 4), ("min_key", C.c_uint64 * 4), ("scored", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P, R = C.POINTER(_Problem), C.POINTER(_Result)
        _lib.or_levels.restype = C.c_int
        _lib.or_levels.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                   C.POINTER(C.c_int32), C.c_uint32, C.c_int, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int64), C.POINTER(C.c_uint8), C.c_int]
        for name in ("or_enum", "or_slice"):
            getattr(_lib, name).argtypes = [P, R]
        _lib.or_enum_range.argtypes = [P, C.c_uint64, C.c_uint64, R]
        _lib.or_enum_min_range.argtypes = [P, C.c_uint64, C.c_uint64, R]
        _lib.or_enum_first_within.argtypes = [P, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64), R]
        _lib.or_key_of.argtypes = [P, C.POINTER(C.c_int32), C.POINTER(C.c_uint64)]
        _lib.or_eval_f64.argtypes = [P, C.POINTER(C.c_int32), C.POINTER(C.c_double)]
    return _lib


# ----------------------------------------------------------------------------------------
# Profile files (SPEC "External Interfaces" of [MODULE] profiles; errors S:64)
# ----------------------------------------------------------------------------------------
class ProfileError(ValueError):
    pass


def us_to_ns(text: str) -> int:
    """Exact decimal microseconds -> integer ns, round half to even (must not lose
    precision beyond 1 ns)."""
    try:
        d = Decimal(text.strip())
    except InvalidOperation:
        raise ProfileError(f"parse failure: not a decimal: {text!r}")
    if not d.is_finite():
        raise ProfileError(f"parse failure: not finite: {text!r}")
    return int((d * 1000).quantize(Decimal(1), rounding=ROUND_HALF_EVEN))


@dataclass
class ModelProfile:
    name: str
    sizes: List[int]
    exec_ns: np.ndarray  # int64 [K, C]


def parse_profiles(text: str) -> List[ModelProfile]:
    lines = [ln for ln in text.splitlines() if ln.strip()]
    out: List[ModelProfile] = []
    i = 0
    while i < len(lines):
        try:
            hdr = json.loads(lines[i])
        except json.JSONDecodeError:
            raise ProfileError(f"parse failure: line {i + 1} is not a JSON header")
        if not isinstance(hdr, dict) or "model" not in hdr or "kernels" not in hdr or "configs" not in hdr:
            raise ProfileError(f"parse failure: header on line {i + 1} lacks model/kernels/configs")
        name, nk, cfg = str(hdr["model"]), int(hdr["kernels"]), [int(c) for c in hdr["configs"]]
        if nk < 1 or not cfg:
            raise ProfileError(f"parse failure: model {name}: empty kernels or configs")
        rows = lines[i + 1:i + 1 + nk]
        if len(rows) < nk:
            raise ProfileError(f"parse failure: model {name}: expected {nk} kernel rows")
        ex = np.zeros((nk, len(cfg)), dtype=np.int64)
        for k, row in enumerate(rows):
            cells = [c for c in row.split(",")]
            if len(cells) != len(cfg) + 1:
                raise ProfileError(f"missing config column: model {name}, kernel {k}")
            for j, cell in enumerate(cells[1:]):
                v = us_to_ns(cell)
                if v <= 0:
                    raise ProfileError(f"non-positive exec_time: model {name}, kernel {k}")
                ex[k, j] = v
            for j in range(len(cfg) - 1):
                if ex[k, j] < ex[k, j + 1]:
                    raise ProfileError(f"non-monotone exec_time: model {name}, kernel {k}")
        out.append(ModelProfile(name, cfg, ex))
        i += 1 + nk
    if not out:
        raise ProfileError("parse failure: empty profile file")
    return out


# ----------------------------------------------------------------------------------------
# Groups: beta_group = sum of member kernels; n_g = member count.
# ----------------------------------------------------------------------------------------
def group_tables(exec_ns: np.ndarray, bounds: Optional[Sequence[int]]):
    K = exec_ns.shape[0]
    if bounds is None:
        bounds = list(range(K + 1))
    G = len(bounds) - 1
    beta = np.zeros((G, exec_ns.shape[1]), dtype=np.int64)
    n = np.zeros(G, dtype=np.int32)
    for g in range(G):
        beta[g] = exec_ns[bounds[g]:bounds[g + 1]].sum(axis=0)
        n[g] = bounds[g + 1] - bounds[g]
    return beta, n


def levels(beta: np.ndarray, n: np.ndarray, sizes: Sequence[int], mask: int, R: int):
    """O-B level table: (S[L], B[L], wit[L, G]) in canonical rank order."""
    G, Cn = beta.shape
    beta = np.ascontiguousarray(beta, dtype=np.int64)
    n = np.ascontiguousarray(n, dtype=np.int32)
    sz = np.ascontiguousarray(sizes, dtype=np.int32)
    cap = int(n.sum()) * (max(sizes) // 1) + 1
    cap = min(cap, 1 << 22)
    S = np.zeros(cap, dtype=np.int64)
    B = np.zeros(cap, dtype=np.int64)
    wit = np.zeros(cap * G, dtype=np.uint8)
    L = lib().or_levels(G, Cn, beta.ctypes.data_as(C.POINTER(C.c_int64)), n.ctypes.data_as(C.POINTER(C.c_int32)),
                        sz.ctypes.data_as(C.POINTER(C.c_int32)), mask, R,
                        S.ctypes.data_as(C.POINTER(C.c_int64)), B.ctypes.data_as(C.POINTER(C.c_int64)),
                        wit.ctypes.data_as(C.POINTER(C.c_uint8)), cap)
    if L < 0:
        raise RuntimeError(f"or_levels failed: {L}")
    return S[:L].copy(), B[:L].copy(), wit[:L * G].reshape(L, G).copy()


def weight_ints(weights, W: int):
    """Per-worker objective weights ("weights: per-worker scalar (default all 1)",
    invariant "weights all strictly positive"; reading R20).  Each weight is taken as
    the integer n_w = round-half-up(omega_w x 1e6), omega_w x 1e6 computed in binary64, so the
    objective uses omega_w = n_w / 1e6 exactly; the exact keys use n_w / gcd_w(n_w) (a common
    positive factor changes neither the arg-min nor the relative tolerance).  Valid: finite,
    0 < omega_w <= 1000 and n_w >= 1.  Returns (ints, values) or raises ValueError."""
    import math
    if weights is None:
        return [1] * W, [1.0] * W
    if len(weights) != W:
        raise ValueError("weights must have one entry per worker")
    n = []
    for x in weights:
        x = float(x)
        if not (math.isfinite(x) and 0.0 < x <= 1000.0):
            raise ValueError(f"weight {x} outside (0, 1000]")
        v = int(Decimal(x * 1e6).quantize(Decimal(1), rounding=ROUND_HALF_UP))
        if v < 1:
            raise ValueError(f"weight {x} rounds to 0 at 1e-6 resolution")
        n.append(v)
    g = 0
    for v in n:
        g = math.gcd(g, v)
    return [v // g for v in n], [v / 1e6 for v in n]


def tol_rational(tol: float):
    """tau as the rational round(tol * 1e9) / 1e9."""
    return int(round(tol * 1e9)), 1_000_000_000


def _key_int(words) -> int:
    return sum(int(words[i]) << (64 * i) for i in range(4))


@dataclass
class OracleResult:
    status: str
    levels: List[int] = field(default_factory=list)
    index: int = 0
    key: int = 0
    min_key: int = 0
    group_cols: List[List[int]] = field(default_factory=list)   # size column per group
    group_sm: List[List[int]] = field(default_factory=list)
    switches: List[int] = field(default_factory=list)
    latency_ns: List[float] = field(default_factory=list)
    alpha: List[float] = field(default_factory=list)
    objective: float = float("nan")
    makespan_ns: float = float("nan")
    power_w: float = float("nan")
    energy_j: float = float("nan")
    throughput_rps: float = float("nan")
    energy_busy_j: float = float("nan")
    group_latency_ns: List[List[float]] = field(default_factory=list)
    tables: list = field(default_factory=list)


class Prepared:
    """A problem marshalled for O-B: per-worker level tables + the C struct."""

    def __init__(self, problem, tol: float = 1e-5):
        p = problem
        self.problem = p
        W = p.W
        self.W = W
        self.tables = []
        Ls, Ss, Bs, Ks = [], [], [], []
        C_ = len(p.sizes)
        for w in range(W):
            m = p.models[p.model_ids[w]]
            gb = p.group_bounds[w] if p.group_bounds is not None else None
            beta, n = group_tables(m.exec_ns, gb)
            mask = p.allowed_mask[w] if p.allowed_mask is not None else (1 << C_) - 1
            S, B, wit = levels(beta, n, p.sizes, mask, p.switch_max)
            self.tables.append((S, B, wit, beta, n))
            Ls.append(len(S)); Ss.append(S); Bs.append(B); Ks.append(int(n.sum()))
        self.L = np.array(Ls, dtype=np.int32)
        self.S = np.ascontiguousarray(np.concatenate(Ss) if Ss else np.zeros(0), dtype=np.int64)
        self.B = np.ascontiguousarray(np.concatenate(Bs) if Bs else np.zeros(0), dtype=np.int64)
        self.K = np.array(Ks, dtype=np.int64)
        q = p.qos_ns if p.qos_ns is not None else [float("inf")] * W
        self.Q = np.array(q, dtype=np.float64)
        M = p.slowdown_matrix if p.slowdown_matrix is not None else np.zeros((W, W), np.float32)
        self.M = np.ascontiguousarray(M, dtype=np.float32).reshape(-1)
        tn, td = tol_rational(tol)
        wi, wv = weight_ints(getattr(p, "weights", None), W)
        self.weighted = getattr(p, "weights", None) is not None
        self.wt = np.array(wi, dtype=np.int64)
        self.wval = np.array(wv, dtype=np.float64)
        self.c = _Problem(W, p.total_sms, MODES[p.mode], OBJECTIVES[p.objective],
                          self.L.ctypes.data_as(C.POINTER(C.c_int32)), self.S.ctypes.data_as(C.POINTER(C.c_int64)),
                          self.B.ctypes.data_as(C.POINTER(C.c_int64)), self.K.ctypes.data_as(C.POINTER(C.c_int64)),
                          self.Q.ctypes.data_as(C.POINTER(C.c_double)), self.M.ctypes.data_as(C.POINTER(C.c_float)),
                          p.p_idle_w, p.p_max_w, tn, td, self.wt.ctypes.data_as(C.POINTER(C.c_int64)),
                          self.wval.ctypes.data_as(C.POINTER(C.c_double)))

    @property
    def n_tuples(self) -> int:
        return int(np.prod([int(x) for x in self.L], dtype=object)) if self.W else 0

    def finish(self, r: _Result) -> OracleResult:
        if r.status < 0:
            raise RuntimeError(f"oracle error {r.status}")
        if r.status == 1:
            return OracleResult("infeasible", tables=self.tables)
        W = self.W
        lv = [int(r.levels[w]) for w in range(W)]
        out = OracleResult("ok", levels=lv, index=int(r.index), key=_key_int(r.key),
                           min_key=_key_int(r.min_key), tables=self.tables)
        vals = (C.c_double * (2 * W + 5))()
        arr = (C.c_int32 * W)(*lv)
        lib().or_eval_f64(C.byref(self.c), arr, vals)
        out.latency_ns = [vals[w] for w in range(W)]
        out.objective, out.makespan_ns, out.power_w, out.energy_j, out.throughput_rps = (
            vals[W], vals[W + 1], vals[W + 2], vals[W + 3], vals[W + 4])
        out.alpha = [vals[W + 5 + w] for w in range(W)]
        sizes = self.problem.sizes
        for w in range(W):
            S, B, wit, beta, n = self.tables[w]
            cols = [int(x) for x in wit[lv[w]]]
            out.group_cols.append(cols)
            out.group_sm.append([sizes[j] for j in cols])
            out.switches.append(sum(1 for g in range(1, len(cols)) if cols[g] != cols[g - 1]))
            out.group_latency_ns.append([float(beta[g, cols[g]]) * (1.0 + out.alpha[w]) for g in range(len(cols))])
        p = self.problem
        out.energy_busy_j = busy_energy_sweep(out.group_sm, out.group_latency_ns, p.total_sms,
                                              float(np.float32(p.p_idle_w)), float(np.float32(p.p_max_w))) * 1e-9
        return out


def busy_energy_sweep(group_sm, group_lat, total: int, p_idle: float, p_max: float) -> float:
    """Busy-SM energy of a plan's predicted run (SPEC integrate_energy S:416-419 with power_at
    S:406-409; reading R21), in W x ns: all workers start at 0 and run their groups back
    to back (group g of worker w on group_sm[w][g] SMs for group_lat[w][g] ns); between consecutive
    group boundaries the power is p_idle + (p_max - p_idle) min(N, sum of running groups' SMs) / N.
    An event loop: repeatedly advance to the earliest current-group end over the workers."""
    W = len(group_sm)
    g = [0] * W                                   # current group of each worker
    end = [group_lat[w][0] if group_lat[w] else 0.0 for w in range(W)]
    t, E = 0.0, 0.0
    while True:
        live = [w for w in range(W) if g[w] < len(group_lat[w])]
        if not live:
            return E
        nxt = min(end[w] for w in live)
        busy = sum(group_sm[w][g[w]] for w in live)
        E += (p_idle + (p_max - p_idle) * min(busy, total) / total) * (nxt - t)
        t = nxt
        for w in live:
            if end[w] == nxt:                     # this worker's group ends now: start its next one
                g[w] += 1
                if g[w] < len(group_lat[w]):
                    end[w] = end[w] + group_lat[w][g[w]]


def solve(problem, engine: str = "enum", tol: float = 1e-5) -> OracleResult:
    """O-B exact answer for a synth.Problem (engine 'enum' or 'slice')."""
    pp = Prepared(problem, tol)
    r = _Result()
    fn = lib().or_enum if engine == "enum" else lib().or_slice
    fn(C.byref(pp.c), C.byref(r))
    if r.status == -1:
        raise ValueError("oracle rejected the problem (invalid argument)")
    return pp.finish(r)


def key_of(pp: Prepared, lv: Sequence[int]):
    """Exact key of one level tuple, or None if a QoS bound fails."""
    arr = (C.c_int32 * pp.W)(*[int(x) for x in lv])
    out = (C.c_uint64 * 4)()
    rc = lib().or_key_of(C.byref(pp.c), arr, out)
    return None if rc == 1 else _key_int(out)
