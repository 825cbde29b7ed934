"""Thin Python binding of the runtime C-ABI (include/eclip_runtime.h) — argument marshalling only.

The B200 analogue of ECLIP's runtime scheduler (§IV-A):
a pre-allocated pool of SM-partitioned streams (CUDA green contexts), lookup-table redirection of
every kernel to its pool stream, and barrier (event-wait) insertion for cross-stream dependencies.
Everything runs in libeclip.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence

import numpy as np

from .eclip import EclipError, lib

RECORD, REPARTITION = 1, 2


class _Config(C.Structure):
    _fields_ = [("device", C.c_int32), ("n_workers", C.c_int32), ("group_sms", C.c_int32),
                ("shared_default", C.c_int32)]


class _Model(C.Structure):
    _fields_ = [("n_kernels", C.c_int32), ("ctas", C.POINTER(C.c_int32)), ("iters", C.POINTER(C.c_int32))]


class _RunOut(C.Structure):
    _fields_ = [("latency_ns", C.POINTER(C.c_int64)), ("t_start", C.POINTER(C.c_int64)),
                ("t_end", C.POINTER(C.c_int64)), ("stream_id", C.POINTER(C.c_int32)),
                ("barrier", C.POINTER(C.c_int32)), ("sm_used", C.POINTER(C.c_int32)),
                ("sm_mask", C.POINTER(C.c_uint32)), ("wall_ns", C.c_int64), ("repartition_ns", C.c_int64),
                ("barriers", C.c_int32)]


_bound = False


def _lib():
    global _bound
    L = lib()
    if not _bound:
        vp = C.c_void_p
        L.eclip_rt_create.argtypes = [C.POINTER(_Config), C.POINTER(vp)]
        L.eclip_rt_free.argtypes = [vp]
        L.eclip_rt_free.restype = None
        L.eclip_rt_info.argtypes = [vp] + [C.POINTER(C.c_int32)] * 5
        L.eclip_rt_layout.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(C.c_uint32), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32)]
        L.eclip_rt_set_table.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(C.c_int32)]
        L.eclip_rt_dispatch.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(vp), C.POINTER(C.c_int32)]
        L.eclip_rt_signal.argtypes = [vp, C.c_int32]
        L.eclip_rt_profile.argtypes = [vp, C.POINTER(_Model), C.c_int32, C.POINTER(C.c_double)]
        L.eclip_rt_run.argtypes = [vp, C.POINTER(_Model), C.c_int32, C.c_int32, C.POINTER(_RunOut)]
        _bound = True
    return L


def _check(rc: int):
    if rc != 0:
        raise EclipError(rc, lib().eclip_last_error().decode())


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


class SyntheticModel:
    """Kernel k = ctas[k] CTAs (one per SM at a time) x iters[k] dependent FMAs per thread."""

    def __init__(self, ctas: Sequence[int], iters: Sequence[int]):
        self.ctas, self.iters = _i32(ctas), _i32(iters)
        assert len(self.ctas) == len(self.iters)
        self.c = _Model(len(self.ctas), self.ctas.ctypes.data_as(C.POINTER(C.c_int32)),
                        self.iters.ctypes.data_as(C.POINTER(C.c_int32)))

    @property
    def n_kernels(self) -> int:
        return len(self.ctas)


class Runtime:
    """eclip_rt: the pre-allocated stream pool of one device for n_workers co-located workers."""

    def __init__(self, n_workers: int, group_sms: int = 16, device: int = 0, shared_default: bool = True):
        self._h = C.c_void_p()
        cfg = _Config(device, n_workers, group_sms, 1 if shared_default else 0)
        _check(_lib().eclip_rt_create(C.byref(cfg), C.byref(self._h)))
        self.n_workers = n_workers
        g, ns, n = C.c_int32(), C.c_int32(), C.c_int32()
        _check(_lib().eclip_rt_info(self._h, C.byref(g), None, C.byref(ns), None, C.byref(n)))
        gs = np.zeros(g.value, np.int32)
        sz = np.zeros(ns.value, np.int32)
        _check(_lib().eclip_rt_info(self._h, None, gs.ctypes.data_as(C.POINTER(C.c_int32)), None,
                                    sz.ctypes.data_as(C.POINTER(C.c_int32)), None))
        self.n_groups, self.group_sm, self.sizes, self.total_sms = g.value, gs.tolist(), sz.tolist(), n.value

    def layout(self, worker: int, size_index: int) -> Dict[str, int]:
        m, s, c = C.c_uint32(), C.c_int32(), C.c_int32()
        _check(_lib().eclip_rt_layout(self._h, worker, size_index, C.byref(m), C.byref(s), C.byref(c)))
        return {"group_mask": m.value, "stream_id": s.value, "sm_count": c.value}

    def set_table(self, worker: int, kernel_sm: Sequence[int]):
        t = _i32(kernel_sm)
        _check(_lib().eclip_rt_set_table(self._h, worker, len(t), t.ctypes.data_as(C.POINTER(C.c_int32))))

    def dispatch(self, worker: int, kernel: int):
        """-> (cudaStream_t as int, barrier flag)"""
        s, b = C.c_void_p(), C.c_int32()
        _check(_lib().eclip_rt_dispatch(self._h, worker, kernel, C.byref(s), C.byref(b)))
        return s.value, b.value

    def signal(self, worker: int):
        _check(_lib().eclip_rt_signal(self._h, worker))

    def profile(self, model: SyntheticModel, reps: int = 5) -> np.ndarray:
        """-> exec_ns [n_kernels, n_sizes] solo device time on every pool size"""
        out = np.zeros((model.n_kernels, len(self.sizes)), np.float64)
        _check(_lib().eclip_rt_profile(self._h, C.byref(model.c), reps, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def run(self, models: List[SyntheticModel], n_requests: int, record: bool = False,
            repartition: bool = False) -> dict:
        W = self.n_workers
        assert len(models) == W
        K = max(m.n_kernels for m in models)
        arr = (_Model * W)(*[m.c for m in models])
        lat = np.zeros((W, n_requests), np.int64)
        o = _RunOut()
        o.latency_ns = lat.ctypes.data_as(C.POINTER(C.c_int64))
        rec = {}
        if record:
            shp = (W, n_requests, K)
            rec = {"t_start": np.zeros(shp, np.int64), "t_end": np.zeros(shp, np.int64),
                   "stream_id": np.zeros(shp, np.int32), "barrier": np.zeros(shp, np.int32),
                   "sm_used": np.zeros(shp, np.int32), "sm_mask": np.zeros(shp + (5,), np.uint32)}
            o.t_start = rec["t_start"].ctypes.data_as(C.POINTER(C.c_int64))
            o.t_end = rec["t_end"].ctypes.data_as(C.POINTER(C.c_int64))
            o.stream_id = rec["stream_id"].ctypes.data_as(C.POINTER(C.c_int32))
            o.barrier = rec["barrier"].ctypes.data_as(C.POINTER(C.c_int32))
            o.sm_used = rec["sm_used"].ctypes.data_as(C.POINTER(C.c_int32))
            o.sm_mask = rec["sm_mask"].ctypes.data_as(C.POINTER(C.c_uint32))
        flags = (RECORD if record else 0) | (REPARTITION if repartition else 0)
        _check(_lib().eclip_rt_run(self._h, arr, n_requests, flags, C.byref(o)))
        out = {"latency_ns": lat, "wall_ns": int(o.wall_ns), "repartition_ns": int(o.repartition_ns),
               "barriers": int(o.barriers)}
        out.update(rec)
        return out

    def close(self):
        if self._h is not None and self._h.value:
            _lib().eclip_rt_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
