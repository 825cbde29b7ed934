"""Thin Python binding of the C-ABI planner (include/eclip.h) — argument marshalling only.

Every step of planning runs in libeclip.so's CUDA kernels.  There is no CPU fallback: if
the library is missing, importing this module raises; if no GPU is visible, planning calls
raise EclipError(ECLIP_E_CUDA).  numpy arrays and torch tensors (host or CUDA) are accepted
wherever an array is expected; PyTorch is only used for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ECLIP_LIB") or os.path.join(_HERE, "libeclip.so")   # ECLIP_LIB: A/B builds only

OK, INFEASIBLE = 0, 1
E_PARSE, E_MISSING_CONFIG, E_NONMONOTONE, E_INVALID_ARG, E_TOO_LARGE, E_CUDA, E_OOM, E_IO = range(-1, -9, -1)
MODES = {"exclude_self": 0, "paper": 1, "paper_as_written": 1, "excess": 2, "excess_over_capacity": 2, "matrix": 3}
OBJECTIVES = {"sum": 0, "max": 1, "energy": 2}
ENGINES = {"auto": 0, "enum": 1, "slice": 2}
ENGINE_NAMES = {1: "enum", 2: "slice", 3: "baseline"}


class EclipError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[eclip {code}] {msg}")
        self.code = code


P = C.POINTER


class Problem(C.Structure):
    _fields_ = [("n_models", C.c_int32), ("model_ids", P(C.c_int32)), ("group_bounds", P(C.c_int32)),
                ("total_sms", C.c_int32), ("allowed_mask", P(C.c_uint32)), ("qos_ns", P(C.c_double)),
                ("switch_max", C.c_int32), ("slowdown", C.c_int32), ("slowdown_matrix", P(C.c_float)),
                ("objective", C.c_int32), ("p_idle_w", C.c_float), ("p_max_w", C.c_float),
                ("weights", P(C.c_double))]


class Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("engine_used", C.c_int32), ("group_sm", P(C.c_int32)),
                ("group_latency_ns", P(C.c_double)), ("model_latency_ns", P(C.c_double)),
                ("model_switches", P(C.c_int32)), ("winner_levels", P(C.c_int32)), ("objective", C.c_double),
                ("makespan_ns", C.c_double), ("power_w", C.c_double), ("energy_j", C.c_double),
                ("throughput_rps", C.c_double), ("winner_index", C.c_uint64), ("candidates", C.c_uint64),
                ("units_scored", C.c_uint64), ("candidates_evaluated", C.c_uint64), ("exact_key", C.c_uint64 * 4),
                ("energy_busy_j", C.c_double)]


class Options(C.Structure):
    _fields_ = [("engine", C.c_int32), ("device", C.c_int32), ("cuda_stream", C.c_void_p), ("tie_tol", C.c_double),
                ("shard", C.c_int32), ("n_shards", C.c_int32), ("no_prune", C.c_int32), ("timing", C.c_int32),
                ("comm", C.c_void_p)]


class Batch(C.Structure):
    _fields_ = [("n_problems", C.c_int32), ("n_models", C.c_int32), ("model_ids", C.c_void_p),
                ("qos_ns", C.c_void_p), ("allowed_mask", P(C.c_uint32)), ("slowdown_matrix", C.c_void_p),
                ("total_sms", C.c_int32), ("switch_max", C.c_int32), ("slowdown", C.c_int32),
                ("objective", C.c_int32), ("p_idle_w", C.c_float), ("p_max_w", C.c_float), ("on_device", C.c_int32),
                ("weights", C.c_void_p)]


class BatchOut(C.Structure):
    _fields_ = [("status", C.c_void_p), ("winner_levels", C.c_void_p), ("winner_index", C.c_void_p),
                ("objective", C.c_void_p), ("makespan_ns", C.c_void_p), ("power_w", C.c_void_p),
                ("energy_j", C.c_void_p), ("throughput_rps", C.c_void_p), ("model_latency_ns", C.c_void_p),
                ("model_switches", C.c_void_p), ("group_sm", C.c_void_p), ("group_stride", C.c_int32),
                ("energy_busy_j", C.c_void_p)]


_lib = None

EXPORTS = ["eclip_load_profiles", "eclip_load_profiles_mem", "eclip_profiles_from_arrays", "eclip_free_profiles",
           "eclip_profiles_info", "eclip_last_error", "eclip_version", "eclip_default_options", "eclip_plan",
           "eclip_plan_batch", "eclip_session_create", "eclip_session_pass1", "eclip_session_pass2_min",
           "eclip_session_pass2_first", "eclip_session_finish", "eclip_session_free",
           "eclip_session_create_problem", "eclip_session_finish_problem", "eclip_session_stats",
           "eclip_session_counters",
           "eclip_baseline_plan", "eclip_lookup_table_json", "eclip_simulate", "eclip_level_table",
           "eclip_planner_create", "eclip_planner_plan", "eclip_planner_phase_ms", "eclip_planner_counters",
           "eclip_planner_free", "eclip_comm_unique_id", "eclip_comm_create", "eclip_comm_create_local",
           "eclip_comm_info", "eclip_comm_free"]


def lib():
    """Load libeclip.so (raises if it has not been built — there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2506_12598_b200.build`")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.eclip_last_error.restype = C.c_char_p
        L.eclip_version.restype = C.c_char_p
        L.eclip_load_profiles.argtypes = [C.c_char_p, P(vp)]
        L.eclip_load_profiles_mem.argtypes = [C.c_char_p, C.c_size_t, P(vp)]
        L.eclip_profiles_from_arrays.argtypes = [C.c_int32, P(C.c_int32), C.c_int32, P(C.c_int32), P(C.c_int64), P(vp)]
        L.eclip_free_profiles.argtypes = [vp]
        L.eclip_free_profiles.restype = None
        L.eclip_profiles_info.argtypes = [vp, P(C.c_int32), P(C.c_int32), P(C.c_int32), P(C.c_int32), P(C.c_int64),
                                          C.c_char_p, C.c_size_t]
        L.eclip_default_options.argtypes = [P(Options)]
        L.eclip_default_options.restype = None
        L.eclip_plan.argtypes = [vp, P(Problem), P(Options), P(Result)]
        L.eclip_plan_batch.argtypes = [vp, P(Batch), P(Options), P(BatchOut)]
        L.eclip_session_create.argtypes = [vp, P(Batch), P(Options), P(vp)]
        L.eclip_session_create_problem.argtypes = [vp, P(Problem), P(Options), P(vp)]
        L.eclip_session_pass1.argtypes = [vp, P(C.c_float)]
        L.eclip_session_pass2_min.argtypes = [vp, P(C.c_float), P(C.c_uint64)]
        L.eclip_session_pass2_first.argtypes = [vp, P(C.c_uint64), P(C.c_uint64)]
        L.eclip_session_finish.argtypes = [vp, P(C.c_uint64), P(BatchOut)]
        L.eclip_session_finish_problem.argtypes = [vp, P(C.c_uint64), P(Result)]
        L.eclip_session_stats.argtypes = [vp, P(C.c_uint64)]
        L.eclip_session_counters.argtypes = [vp, P(C.c_uint64), C.c_int32]
        L.eclip_session_free.argtypes = [vp]
        L.eclip_session_free.restype = None
        L.eclip_baseline_plan.argtypes = [vp, P(Problem), C.c_int32, C.c_double, P(Options), P(Result)]
        L.eclip_lookup_table_json.argtypes = [vp, P(Problem), P(C.c_int32), C.c_char_p, C.c_size_t,
                                              P(C.c_size_t), P(C.c_uint64)]
        L.eclip_planner_create.argtypes = [vp, P(Batch), C.c_int32, P(Options), P(vp)]
        L.eclip_planner_plan.argtypes = [vp, P(Batch), P(BatchOut)]
        L.eclip_planner_phase_ms.argtypes = [vp, P(C.c_float), C.c_int32]
        L.eclip_planner_counters.argtypes = [vp, P(C.c_uint64), C.c_int32]
        L.eclip_planner_free.argtypes = [vp]
        L.eclip_planner_free.restype = None
        L.eclip_comm_unique_id.argtypes = [C.c_char_p]
        L.eclip_comm_create.argtypes = [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, P(vp)]
        L.eclip_comm_create_local.argtypes = [C.c_int32, C.c_int32, P(vp)]
        L.eclip_comm_info.argtypes = [vp, P(C.c_int32), P(C.c_int32), P(C.c_int32)]
        L.eclip_comm_free.argtypes = [vp]
        L.eclip_comm_free.restype = None
        L.eclip_level_table.argtypes = [vp, C.c_int32, P(C.c_int32), C.c_uint32, C.c_int32, P(Options), C.c_int32,
                                        P(C.c_int64), P(C.c_int64), P(C.c_uint8), P(C.c_int32), P(C.c_int32)]
        _lib = L
    return _lib


def _check(rc: int):
    if rc < 0:
        raise EclipError(rc, lib().eclip_last_error().decode(errors="replace"))
    return rc


def _np(a, dtype):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


def _ptr(a, ctype):
    return a.ctypes.data_as(P(ctype)) if a is not None else None


def _addr(x):
    """address of a numpy array or torch tensor"""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return x.ctypes.data


# ------------------------------------------------------------------------------------------
class Profiles:
    """Library-owned, immutable profile tables (eclip_profiles)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        self._nk = None

    def n_kernels(self) -> List[int]:
        """kernels per model (cached: profiles are immutable after loading)"""
        if self._nk is None:
            n, c = C.c_int32(), C.c_int32()
            _check(lib().eclip_profiles_info(self._h, C.byref(n), C.byref(c), None, None, None, None, 0))
            nk = np.zeros(n.value, np.int32)
            _check(lib().eclip_profiles_info(self._h, None, None, None, _ptr(nk, C.c_int32), None, None, 0))
            self._nk = nk.tolist()
        return self._nk

    @classmethod
    def from_text(cls, text: str) -> "Profiles":
        h = C.c_void_p()
        b = text.encode()
        _check(lib().eclip_load_profiles_mem(b, len(b), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_file(cls, path: str) -> "Profiles":
        h = C.c_void_p()
        _check(lib().eclip_load_profiles(path.encode(), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_arrays(cls, sizes: Sequence[int], exec_ns_per_model: Sequence[np.ndarray]) -> "Profiles":
        nk = _np([len(e) for e in exec_ns_per_model], np.int32)
        sz = _np(sizes, np.int32)
        ex = _np(np.concatenate([np.asarray(e, dtype=np.int64).reshape(-1, len(sizes)) for e in exec_ns_per_model]),
                 np.int64)
        h = C.c_void_p()
        _check(lib().eclip_profiles_from_arrays(len(nk), _ptr(nk, C.c_int32), len(sz), _ptr(sz, C.c_int32),
                                                _ptr(ex, C.c_int64), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_models(cls, models) -> "Profiles":
        """from objects with .sizes and .exec_ns (e.g. synth.Model)"""
        return cls.from_arrays(models[0].sizes, [m.exec_ns for m in models])

    def info(self):
        n, c = C.c_int32(), C.c_int32()
        _check(lib().eclip_profiles_info(self._h, C.byref(n), C.byref(c), None, None, None, None, 0))
        sizes = np.zeros(c.value, np.int32)
        nk = np.zeros(n.value, np.int32)
        _check(lib().eclip_profiles_info(self._h, None, None, _ptr(sizes, C.c_int32), _ptr(nk, C.c_int32), None, None, 0))
        ex = np.zeros((int(nk.sum()), c.value), np.int64)
        names = C.create_string_buffer(1 << 16)
        _check(lib().eclip_profiles_info(self._h, None, None, None, None, _ptr(ex, C.c_int64), names, len(names)))
        return dict(n_models=n.value, sizes=sizes.tolist(), n_kernels=nk.tolist(), exec_ns=ex,
                    names=names.value.decode().split("\n")[:-1])

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value and _lib is not None:
            _lib.eclip_free_profiles(self._h)
            self._h = None


# ------------------------------------------------------------------------------------------
@dataclass
class Plan:
    status: str
    engine: str
    group_sm: List[List[int]]
    group_latency_ns: List[List[float]]
    model_latency_ns: List[float]
    model_switches: List[int]
    winner_levels: List[int]
    objective: float
    makespan_ns: float
    power_w: float
    energy_j: float
    throughput_rps: float
    winner_index: int
    candidates: int
    units_scored: int
    exact_key: int
    candidates_evaluated: int = 0
    energy_busy_j: float = 0.0


def _options(engine="auto", device=0, stream=None, tie_tol=1e-5, shard=0, n_shards=1, prune=True,
             timing=False, comm=None) -> Options:
    o = Options()
    lib().eclip_default_options(C.byref(o))
    o.engine = ENGINES[engine]
    o.device = device
    o.cuda_stream = stream if isinstance(stream, int) or stream is None else getattr(stream, "cuda_stream", stream)
    o.tie_tol = tie_tol
    o.shard, o.n_shards = shard, n_shards
    o.no_prune = 0 if prune else 1
    o.timing = 1 if timing else 0
    o.comm = comm.handle.value if comm is not None else None
    return o


class Comm:
    """eclip_comm: the in-library exchange of a sharded plan (NCCL, one process per GPU), or one of
    a local group of communicators in one process (tests).  Pass as comm= to plan / plan_batch."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)

    @staticmethod
    def unique_id() -> bytes:
        b = C.create_string_buffer(128)
        _check(lib().eclip_comm_unique_id(b))
        return b.raw

    @classmethod
    def create(cls, uid: bytes, n_ranks: int, rank: int, device: int) -> "Comm":
        h = C.c_void_p()
        _check(lib().eclip_comm_create(uid, n_ranks, rank, device, C.byref(h)))
        return cls(h.value)

    @classmethod
    def local_group(cls, n_ranks: int, device: int = 0):
        hs = (C.c_void_p * n_ranks)()
        _check(lib().eclip_comm_create_local(n_ranks, device, hs))
        return [cls(h) for h in hs]

    @property
    def handle(self):
        return self._h

    def info(self):
        r, n, d = C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().eclip_comm_info(self._h, C.byref(r), C.byref(n), C.byref(d)))
        return dict(rank=r.value, size=n.value, device=d.value)

    def close(self):
        if self._h is not None and self._h.value and _lib is not None:
            _lib.eclip_comm_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _ProblemArgs:
    """keeps the numpy buffers alive while the C struct points at them"""

    def _nk(self, nk, w):
        m = int(self.ids[w])
        return nk[m] if 0 <= m < len(nk) else 0  # invalid ids are rejected by the library

    def __init__(self, profiles, model_ids, total_sms, switch_max, slowdown, objective, allowed_mask, qos_ns,
                 slowdown_matrix, group_bounds, p_idle_w, p_max_w, weights=None):
        self.ids = _np(model_ids, np.int32)
        W = len(self.ids)
        self.W = W
        self.gb = None
        self.G = []
        nk = profiles.n_kernels()
        if group_bounds is not None:
            flat = []
            for w in range(W):
                b = group_bounds[w] if group_bounds[w] is not None else list(range(self._nk(nk, w) + 1))
                flat.extend(int(x) for x in b)
                self.G.append(len(b) - 1)
            self.gb = _np(flat, np.int32)
        else:
            self.G = [self._nk(nk, w) for w in range(W)]
        self.mask = _np(allowed_mask, np.uint32) if allowed_mask is not None else None
        self.qos = _np(qos_ns, np.float64) if qos_ns is not None else None
        self.M = _np(slowdown_matrix, np.float32).reshape(-1) if slowdown_matrix is not None else None
        self.wt = _np(weights, np.float64) if weights is not None else None
        self.c = Problem(W, _ptr(self.ids, C.c_int32), _ptr(self.gb, C.c_int32), total_sms, _ptr(self.mask, C.c_uint32),
                         _ptr(self.qos, C.c_double), switch_max, MODES[slowdown], _ptr(self.M, C.c_float),
                         OBJECTIVES[objective], p_idle_w, p_max_w, _ptr(self.wt, C.c_double))


def _result_buffers(W, G):
    tot = int(sum(G))
    bufs = dict(gsm=np.zeros(tot, np.int32), glat=np.zeros(tot, np.float64), lat=np.zeros(W, np.float64),
                sw=np.zeros(W, np.int32), lv=np.zeros(W, np.int32))
    r = Result()
    r.group_sm = _ptr(bufs["gsm"], C.c_int32)
    r.group_latency_ns = _ptr(bufs["glat"], C.c_double)
    r.model_latency_ns = _ptr(bufs["lat"], C.c_double)
    r.model_switches = _ptr(bufs["sw"], C.c_int32)
    r.winner_levels = _ptr(bufs["lv"], C.c_int32)
    return r, bufs


def _to_plan(r: Result, bufs, G) -> Plan:
    gsm, glat, off = [], [], 0
    for g in G:
        gsm.append(bufs["gsm"][off:off + g].tolist())
        glat.append(bufs["glat"][off:off + g].tolist())
        off += g
    key = sum(int(r.exact_key[i]) << (64 * i) for i in range(4))
    return Plan("ok" if r.status == OK else "infeasible", ENGINE_NAMES.get(r.engine_used, "?"), gsm, glat,
                bufs["lat"].tolist(), bufs["sw"].tolist(), bufs["lv"].tolist(), r.objective, r.makespan_ns, r.power_w,
                r.energy_j, r.throughput_rps, int(r.winner_index), int(r.candidates), int(r.units_scored), key,
                int(r.candidates_evaluated), float(r.energy_busy_j))


def plan(profiles: Profiles, model_ids, *, total_sms: int, switch_max: int = 14, slowdown: str = "exclude_self",
         objective: str = "sum", allowed_mask=None, qos_ns=None, slowdown_matrix=None, group_bounds=None,
         p_idle_w: float = 75.0, p_max_w: float = 225.0, engine: str = "auto", tie_tol: float = 1e-5,
         device: int = 0, stream=None, prune: bool = True, comm: "Comm" = None, weights=None) -> Plan:
    """eclip_plan: the exact optimum of one co-location problem (§IV-B); with comm, sharded
    over the communicator's ranks (every rank returns the same plan).  weights: per-worker objective
    weights, None = all 1."""
    a = _ProblemArgs(profiles, model_ids, total_sms, switch_max, slowdown, objective, allowed_mask, qos_ns,
                     slowdown_matrix, group_bounds, p_idle_w, p_max_w, weights)
    o = _options(engine, device, stream, tie_tol, prune=prune, comm=comm)
    r, bufs = _result_buffers(a.W, a.G)
    _check(lib().eclip_plan(profiles.handle, C.byref(a.c), C.byref(o), C.byref(r)))
    return _to_plan(r, bufs, a.G)


def plan_problem(profiles: Profiles, p, **kw) -> Plan:
    """eclip_plan for a synth.Problem-like object"""
    return plan(profiles, p.model_ids, total_sms=p.total_sms, switch_max=p.switch_max, slowdown=p.mode,
                objective=p.objective, allowed_mask=p.allowed_mask, qos_ns=p.qos_ns,
                slowdown_matrix=p.slowdown_matrix, group_bounds=p.group_bounds, p_idle_w=p.p_idle_w,
                p_max_w=p.p_max_w, weights=getattr(p, "weights", None), **kw)


def level_table(profiles: Profiles, model: int, *, switch_max: int = 14, group_bounds=None, allowed_mask: int = 0,
                device: int = 0):
    """eclip_level_table: the K1 level table of one worker, built on the GPU -> (S [L] int64 SMs,
    B [L] int64 ns, witness [L, G] uint8 size columns), levels in canonical rank order."""
    gb = _np(group_bounds, np.int32) if group_bounds is not None else None
    o = _options("auto", device)
    L, G = C.c_int32(), C.c_int32()
    _check(lib().eclip_level_table(profiles.handle, model, _ptr(gb, C.c_int32), allowed_mask, switch_max, C.byref(o),
                                   0, None, None, None, C.byref(L), C.byref(G)))
    S = np.zeros(L.value, np.int64)
    B = np.zeros(L.value, np.int64)
    wit = np.zeros((L.value, G.value), np.uint8)
    _check(lib().eclip_level_table(profiles.handle, model, _ptr(gb, C.c_int32), allowed_mask, switch_max, C.byref(o),
                                   L.value, _ptr(S, C.c_int64), _ptr(B, C.c_int64), _ptr(wit, C.c_uint8), C.byref(L),
                                   C.byref(G)))
    return S, B, wit


BASELINES = {"all_max": 0, "model_wise": 1, "kernel_wise": 2}


def baseline_plan(profiles: Profiles, model_ids, *, kind: str, param: float = 0.0, total_sms: int,
                  switch_max: int = 14, slowdown: str = "exclude_self", objective: str = "sum", allowed_mask=None,
                  qos_ns=None, slowdown_matrix=None, group_bounds=None, p_idle_w: float = 75.0,
                  p_max_w: float = 225.0, device: int = 0, stream=None, weights=None) -> Plan:
    """eclip_baseline_plan: the paper's comparison plans (Baseline / Model-Wise / Kernel-Wise,
    PAPER.md §V) evaluated on the GPU under the same model as plan()."""
    a = _ProblemArgs(profiles, model_ids, total_sms, switch_max, slowdown, objective, allowed_mask, qos_ns,
                     slowdown_matrix, group_bounds, p_idle_w, p_max_w, weights)
    o = _options("auto", device, stream)
    r, bufs = _result_buffers(a.W, a.G)
    _check(lib().eclip_baseline_plan(profiles.handle, C.byref(a.c), BASELINES[kind], float(param), C.byref(o),
                                     C.byref(r)))
    return _to_plan(r, bufs, a.G)


def lookup_table_json(profiles: Profiles, model_ids, group_sm, *, total_sms: int, switch_max: int = 14,
                      slowdown: str = "exclude_self", group_bounds=None, slowdown_matrix=None):
    """eclip_lookup_table_json: (JSON text, FNV-1a 64 hash) of a plan's lookup table."""
    if slowdown == "matrix" and slowdown_matrix is None:
        slowdown_matrix = np.zeros((len(model_ids), len(model_ids)), np.float32)
    a = _ProblemArgs(profiles, model_ids, total_sms, switch_max, slowdown, "sum", None, None, slowdown_matrix,
                     group_bounds, 75.0, 225.0)
    g = _np([c for row in group_sm for c in row], np.int32)
    n, h = C.c_size_t(), C.c_uint64()
    _check(lib().eclip_lookup_table_json(profiles.handle, C.byref(a.c), _ptr(g, C.c_int32), None, 0, C.byref(n),
                                         C.byref(h)))
    buf = C.create_string_buffer(n.value + 1)
    _check(lib().eclip_lookup_table_json(profiles.handle, C.byref(a.c), _ptr(g, C.c_int32), buf, len(buf),
                                         C.byref(n), C.byref(h)))
    return buf.value.decode(), int(h.value)


# ------------------------------------------------------------------------------------------
class _BatchArgs:
    def __init__(self, model_ids, qos_ns, slowdown_matrix, allowed_mask, total_sms, switch_max, slowdown, objective,
                 p_idle_w, p_max_w, on_device, weights=None):
        if on_device:
            self.ids, self.qos, self.M, self.wt = model_ids, qos_ns, slowdown_matrix, weights
            n, W = int(model_ids.shape[0]), int(model_ids.shape[1])
        else:
            self.ids = _np(model_ids, np.int32)
            n, W = self.ids.shape
            self.qos = _np(qos_ns, np.float64) if qos_ns is not None else None
            self.M = _np(slowdown_matrix, np.float32) if slowdown_matrix is not None else None
            self.wt = _np(weights, np.float64) if weights is not None else None
        self.mask = _np(allowed_mask, np.uint32) if allowed_mask is not None else None
        self.n, self.W = n, W
        self.c = Batch(n, W, _addr(self.ids), _addr(self.qos), _ptr(self.mask, C.c_uint32), _addr(self.M), total_sms,
                       switch_max, MODES[slowdown], OBJECTIVES[objective], p_idle_w, p_max_w, 1 if on_device else 0,
                       _addr(self.wt))


def alloc_batch_out(n: int, W: int, gmax: int = 0, device=None, pinned: bool = False):
    """result buffers for plan_batch: numpy (host; page-locked when pinned) or torch tensors on `device`"""
    if device is None:
        if pinned:
            import torch
            tdt = {np.int32: torch.int32, np.uint64: torch.int64, np.float64: torch.float64}
            mk = lambda shape, dt: torch.zeros(shape, dtype=tdt[dt]).pin_memory().numpy().view(dt)
        else:
            mk = lambda shape, dt: np.zeros(shape, dt)
        i32, u64, f64 = np.int32, np.uint64, np.float64
    else:
        import torch
        mk = lambda shape, dt: torch.zeros(shape, dtype=dt, device=device)
        i32, u64, f64 = torch.int32, torch.int64, torch.float64
    out = dict(status=mk((n,), i32), winner_levels=mk((n, W), i32), winner_index=mk((n,), u64),
               objective=mk((n,), f64), makespan_ns=mk((n,), f64), power_w=mk((n,), f64), energy_j=mk((n,), f64),
               throughput_rps=mk((n,), f64), model_latency_ns=mk((n, W), f64), model_switches=mk((n, W), i32),
               energy_busy_j=mk((n,), f64))
    if gmax:
        out["group_sm"] = mk((n, W, gmax), i32)
    out["_gmax"] = gmax
    return out


def _batch_out_struct(out) -> BatchOut:
    b = BatchOut()
    for k in ("status", "winner_levels", "winner_index", "objective", "makespan_ns", "power_w", "energy_j",
              "throughput_rps", "model_latency_ns", "model_switches"):
        setattr(b, k, _addr(out[k]))
    b.group_sm = _addr(out.get("group_sm"))
    b.group_stride = int(out.get("_gmax", 0))
    b.energy_busy_j = _addr(out.get("energy_busy_j"))
    return b


def plan_batch(profiles: Profiles, model_ids, *, total_sms: int, switch_max: int = 14, slowdown: str = "exclude_self",
               objective: str = "sum", qos_ns=None, slowdown_matrix=None, allowed_mask=None, p_idle_w: float = 75.0,
               p_max_w: float = 225.0, tie_tol: float = 1e-5, device: int = 0, stream=None, out=None, gmax: int = 0,
               prune: bool = True, comm: "Comm" = None, weights=None):
    """eclip_plan_batch: many independent mixes per launch (BASELINE config 5).

    With torch CUDA tensors for model_ids / qos_ns / slowdown_matrix (and `out` from
    alloc_batch_out(..., device=...)), everything stays in device memory (on_device=1)."""
    on_device = hasattr(model_ids, "is_cuda") and model_ids.is_cuda
    a = _BatchArgs(model_ids, qos_ns, slowdown_matrix, allowed_mask, total_sms, switch_max, slowdown, objective,
                   p_idle_w, p_max_w, on_device, weights)
    if out is None:
        out = alloc_batch_out(a.n, a.W, gmax, device=(model_ids.device if on_device else None))
    b = _batch_out_struct(out)
    o = _options("enum", device, stream, tie_tol, prune=prune, comm=comm)
    _check(lib().eclip_plan_batch(profiles.handle, C.byref(a.c), C.byref(o), C.byref(b)))
    return out


# ------------------------------------------------------------------------------------------
PHASES = ("h2d", "prep", "pass1", "pass2", "materialize")


class Planner:
    """eclip_planner_*: a persistent batch planner over one profile library (serving-loop
    replanning).  The level tables are built once at construction; plan() runs the per-mix work
    only.  Host (numpy) inputs and outputs are copied on the planner's stream; torch CUDA inputs
    with device outputs (alloc_batch_out(..., device=...)) stay on the device."""

    def __init__(self, profiles: Profiles, *, n_models: int, max_problems: int, total_sms: int, switch_max: int = 14,
                 slowdown: str = "exclude_self", objective: str = "sum", qos: bool = True, allowed_mask=None,
                 p_idle_w: float = 75.0, p_max_w: float = 225.0, tie_tol: float = 1e-5, device: int = 0,
                 stream=None, prune: bool = True, timing: bool = False, weights: bool = False):
        self.profiles = profiles
        self.W, self.n_max = n_models, max_problems
        self.mask = _np(allowed_mask, np.uint32) if allowed_mask is not None else None
        self.kw = (total_sms, switch_max, MODES[slowdown], OBJECTIVES[objective], p_idle_w, p_max_w)
        self.qos = qos
        self._h = C.c_void_p()
        shape = Batch(1, n_models, None, 1 if qos else None, _ptr(self.mask, C.c_uint32), None, total_sms, switch_max,
                      MODES[slowdown], OBJECTIVES[objective], p_idle_w, p_max_w, 0, 1 if weights else None)
        o = _options("enum", device, stream, tie_tol, prune=prune, timing=timing)
        _check(lib().eclip_planner_create(profiles.handle, C.byref(shape), max_problems, C.byref(o), C.byref(self._h)))
        self._cache = {}

    def _structs(self, model_ids, qos_ns, slowdown_matrix, out, weights=None):
        key = (_addr(model_ids), _addr(qos_ns), _addr(slowdown_matrix), id(out), _addr(weights))
        hit = self._cache.get(key)
        if hit is None:
            on_device = hasattr(model_ids, "is_cuda") and model_ids.is_cuda
            n = int(model_ids.shape[0])
            b = Batch(n, self.W, _addr(model_ids), _addr(qos_ns), _ptr(self.mask, C.c_uint32), _addr(slowdown_matrix),
                      *self.kw, 1 if on_device else 0, _addr(weights))
            hit = (b, _batch_out_struct(out), (model_ids, qos_ns, slowdown_matrix, out, weights))
            if len(self._cache) > 64:
                self._cache.clear()
            self._cache[key] = hit
        return hit

    def plan(self, model_ids, qos_ns=None, slowdown_matrix=None, out=None, gmax: int = 0, weights=None):
        """plan one batch: model_ids [n, W] int32 (numpy / pinned numpy / torch CUDA), qos_ns [n, W]
        float64 when the planner has QoS.  Returns `out` (allocated if None)."""
        if not (hasattr(model_ids, "is_cuda") and model_ids.is_cuda):
            model_ids = np.ascontiguousarray(model_ids, dtype=np.int32)
            qos_ns = None if qos_ns is None else np.ascontiguousarray(qos_ns, dtype=np.float64)
            weights = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
        if out is None:
            dev = model_ids.device if hasattr(model_ids, "is_cuda") and model_ids.is_cuda else None
            out = alloc_batch_out(int(model_ids.shape[0]), self.W, gmax, device=dev)
        b, bo, _ = self._structs(model_ids, qos_ns, slowdown_matrix, out, weights)
        _check(lib().eclip_planner_plan(self._h, C.byref(b), C.byref(bo)))
        return out

    def phase_ms(self) -> dict:
        """CUDA-event split of the last plan (needs timing=True)"""
        ms = (C.c_float * 5)()
        _check(lib().eclip_planner_phase_ms(self._h, ms, 5))
        return {k: float(ms[i]) for i, k in enumerate(PHASES)}

    def counters(self) -> dict:
        v = (C.c_uint64 * 8)()
        _check(lib().eclip_planner_counters(self._h, v, 8))
        return {"evaluated_candidates": int(v[0]), "units_processed": int(v[1]), "kernel_ms": int(v[2]) * 1e-6,
                "units_with_swept_entries": int(v[3]), "entries_swept": int(v[4]), "units_past_unit_bound": int(v[5]),
                "units_with_kept_chunks": int(v[6]), "chunks_kept": int(v[7])}

    def close(self):
        if self._h is not None and self._h.value:
            lib().eclip_planner_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------------------------------
class Session:
    """The split API (eclip_session_*): one shard of a problem or batch; the caller combines
    the per-step values across shards (see parallel.py)."""

    def __init__(self, profiles: Profiles, *, problem=None, batch=None, shard=0, n_shards=1, engine="auto",
                 tie_tol=1e-5, device=0, stream=None, prune=True, **problem_kw):
        self.profiles = profiles
        self._h = C.c_void_p()
        o = _options(engine, device, stream, tie_tol, shard, n_shards, prune)
        if problem is not None:
            self.args = _ProblemArgs(profiles, problem.model_ids, problem.total_sms, problem.switch_max, problem.mode,
                                     problem.objective, problem.allowed_mask, problem.qos_ns,
                                     problem.slowdown_matrix, problem.group_bounds, problem.p_idle_w,
                                     problem.p_max_w, getattr(problem, "weights", None))
            self.n, self.W, self.single = 1, self.args.W, True
            _check(lib().eclip_session_create_problem(profiles.handle, C.byref(self.args.c), C.byref(o),
                                                      C.byref(self._h)))
        else:
            self.args = _BatchArgs(batch["model_ids"], batch.get("qos_ns"), batch.get("slowdown_matrix"),
                                   batch.get("allowed_mask"), batch["total_sms"], batch.get("switch_max", 14),
                                   batch.get("slowdown", "exclude_self"), batch.get("objective", "sum"),
                                   batch.get("p_idle_w", 75.0), batch.get("p_max_w", 225.0), False)
            self.n, self.W, self.single = self.args.n, self.args.W, False
            _check(lib().eclip_session_create(profiles.handle, C.byref(self.args.c), C.byref(o), C.byref(self._h)))

    def pass1(self) -> np.ndarray:
        m = np.zeros(self.n, np.float32)
        _check(lib().eclip_session_pass1(self._h, _ptr(m, C.c_float)))
        return m

    def pass2_min(self, global_min: np.ndarray) -> np.ndarray:
        g = _np(global_min, np.float32)
        k = np.zeros((self.n, 4), np.uint64)
        _check(lib().eclip_session_pass2_min(self._h, _ptr(g, C.c_float), _ptr(k, C.c_uint64)))
        return k

    def pass2_first(self, global_exact_min: np.ndarray) -> np.ndarray:
        """-> [n, 4] uint64: the lowest qualifying level tuple of this shard, packed
        (sum_w l_w << 16 (15 - w)); all-ones = none."""
        g = _np(global_exact_min, np.uint64)
        f = np.zeros((self.n, 4), np.uint64)
        _check(lib().eclip_session_pass2_first(self._h, _ptr(g, C.c_uint64), _ptr(f, C.c_uint64)))
        return f

    def finish(self, global_first: np.ndarray, gmax: int = 0):
        g = _np(global_first, np.uint64)
        if self.single:
            r, bufs = _result_buffers(self.W, self.args.G)
            _check(lib().eclip_session_finish_problem(self._h, _ptr(g, C.c_uint64), C.byref(r)))
            return _to_plan(r, bufs, self.args.G)
        out = alloc_batch_out(self.n, self.W, gmax)
        b = _batch_out_struct(out)
        _check(lib().eclip_session_finish(self._h, _ptr(g, C.c_uint64), C.byref(b)))
        return out

    def stats(self) -> dict:
        """counters of the last pass 1: evaluated = QoS-feasible candidates scored in FP32;
        units_processed = pass-1 units (rows) not pruned by their bound (0 when pruning is off);
        kernel_ms = CUDA-event time of the dominant pass-1 kernel's last launch"""
        v = (C.c_uint64 * 5)()
        _check(lib().eclip_session_counters(self._h, v, 5))
        return {"evaluated_candidates": int(v[0]), "units_processed": int(v[1]), "kernel_ms": int(v[2]) * 1e-6,
                "units_with_swept_entries": int(v[3]), "entries_swept": int(v[4])}

    def close(self):
        if self._h is not None and self._h.value:
            lib().eclip_session_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------------------------------
# batched co-location simulator (include/eclip.h eclip_simulate)
class _SimBatch(C.Structure):
    _fields_ = [("n_scenarios", C.c_int32), ("n_workers", C.c_int32), ("max_kernels", C.c_int32),
                ("n_sizes", C.c_int32), ("n_groups", C.c_int32), ("n_kernels", C.c_void_p), ("beta_ns", C.c_void_p),
                ("table", C.c_void_p), ("mask", C.c_void_p), ("group_sm", C.c_void_p), ("total_sms", C.c_int32),
                ("n_requests", C.c_int32), ("shared_default", C.c_int32), ("mode", C.c_int32),
                ("barrier_ns", C.c_double), ("ioctl_lo_ns", C.c_double), ("ioctl_mode_ns", C.c_double),
                ("ioctl_hi_ns", C.c_double), ("oversub", C.c_double), ("p_idle_w", C.c_double),
                ("p_max_w", C.c_double), ("seed", C.c_uint64)]


class _SimOut(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("throughput_rps", "p95_ns", "mean_ns", "makespan_ns", "energy_j",
                                          "req_per_j", "barriers", "events")]


def simulate(n_kernels, beta_ns, table, mask, group_sm, *, total_sms: int, n_requests: int,
             shared_default: bool = True, ioctl: bool = False, barrier_ns: float = 0.0,
             ioctl_ns=(10000.0, 30000.0, 55400.0), oversub: float = 1.0, p_idle_w: float = 75.0,
             p_max_w: float = 225.0, seed: int = 0, device: int = 0) -> dict:
    """eclip_simulate.  n_kernels [S, W]; beta_ns [S, W, K, C]; table [S, W, K] pool indices;
    mask [W, C] group bitsets (pool C-1 = full device); group_sm [G].  Returns numpy arrays."""
    nk = _np(n_kernels, np.int32)
    be = _np(beta_ns, np.float64)
    tb = _np(table, np.int32)
    mk = _np(mask, np.uint32)
    gs = _np(group_sm, np.int32)
    S, W, K, Cn = be.shape
    assert nk.shape == (S, W) and tb.shape == (S, W, K) and mk.shape == (W, Cn)
    b = _SimBatch(S, W, K, Cn, len(gs), nk.ctypes.data, be.ctypes.data, tb.ctypes.data, mk.ctypes.data,
                  gs.ctypes.data, total_sms, n_requests, 1 if shared_default else 0, 1 if ioctl else 0,
                  barrier_ns, ioctl_ns[0], ioctl_ns[1], ioctl_ns[2], oversub, p_idle_w, p_max_w, seed)
    out = {"throughput_rps": np.zeros((S, W)), "p95_ns": np.zeros((S, W)), "mean_ns": np.zeros((S, W)),
           "makespan_ns": np.zeros(S), "energy_j": np.zeros(S), "req_per_j": np.zeros(S),
           "barriers": np.zeros(S, np.int32), "events": np.zeros(S, np.int64)}
    o = _SimOut(*[out[n].ctypes.data for n, _ in _SimOut._fields_])
    L = lib()
    L.eclip_simulate.argtypes = [C.POINTER(_SimBatch), C.POINTER(Options), C.POINTER(_SimOut)]
    _check(L.eclip_simulate(C.byref(b), C.byref(_options("auto", device)), C.byref(o)))
    return out
