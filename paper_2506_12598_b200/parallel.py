"""Multi-GPU planning: shard the candidate space over ranks, one exchange per pass
(DESIGN.md §5).

One process per GPU.  Each rank runs a Session on its shard (ENUM: a contiguous range of
pass-1 items of every problem; SLICE: the T' slices congruent to its rank) and the ranks
combine three tiny per-problem values with torch.distributed (NCCL over NVLink on the B200
box, gloo in the CPU tests):
    pass 1    float32 minimum of the FP32 filter key        -> all-reduce MIN
    pass 2a   exact 256-bit minimum key                     -> all-gather + lexicographic MIN
    pass 2b   lowest qualifying level tuple (packed 256-bit) -> all-gather + lexicographic MIN
after which every rank materialises the same plan.  Two drivers: run_sharded (the split API of
include/eclip.h, values through torch.distributed — gloo in the CPU tests) and nccl_comm /
plan_nccl (the library's own NCCL communicator: the exchanges stay on the device, no host round
trip).  Batches of independent mixes need no exchange at all: shard the mixes instead (bench.py).
"""
from __future__ import annotations

from typing import Callable

import numpy as np

U64_NONE = np.uint64(0xFFFFFFFFFFFFFFFF)
I64_MAX = np.iinfo(np.int64).max


def lexmin_u256(stacked: np.ndarray) -> np.ndarray:
    """stacked [ranks, n, 4] uint64 little-endian limbs -> [n, 4] lexicographic minimum (most
    significant limb first), vectorised over the n problems"""
    out = stacked[0].copy()
    for r in range(1, stacked.shape[0]):
        c = stacked[r]
        less = np.zeros(out.shape[0], bool)
        eq = np.ones(out.shape[0], bool)
        for limb in (3, 2, 1, 0):
            less |= eq & (c[:, limb] < out[:, limb])
            eq &= c[:, limb] == out[:, limb]
        out[less] = c[less]
    return out


class TorchComm:
    """The three reductions over a torch.distributed process group."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        backend = dist.get_backend(group)
        self.device = device if device is not None else ("cuda" if backend == "nccl" else "cpu")

    def _t(self, a):
        return self.torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    def min_f32(self, a: np.ndarray) -> np.ndarray:
        t = self._t(a.astype(np.float32))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return t.cpu().numpy()

    def min_u256(self, a: np.ndarray) -> np.ndarray:
        t = self._t(a.view(np.int64))
        world = self.dist.get_world_size(self.group)
        outs = [self.torch.empty_like(t) for _ in range(world)]
        self.dist.all_gather(outs, t, group=self.group)
        stacked = np.stack([o.cpu().numpy().view(np.uint64) for o in outs])
        return lexmin_u256(stacked)

    def min_u64(self, a: np.ndarray) -> np.ndarray:
        v = np.where(a == U64_NONE, I64_MAX, a.astype(np.int64))
        t = self._t(v)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        r = t.cpu().numpy()
        return np.where(r == I64_MAX, U64_NONE, r.astype(np.uint64))


def run_sharded(session, comm, gmax: int = 0):
    """Drive one rank's session through the protocol; returns the (identical) plan."""
    m = comm.min_f32(session.pass1())
    k = comm.min_u256(session.pass2_min(m))
    f = comm.min_u256(session.pass2_first(k))
    return session.finish(f, gmax) if not getattr(session, "single", False) else session.finish(f)


def plan_distributed(profiles, problem, group=None, **kw):
    """eclip_plan of one problem sharded over every rank of `group` (torch.distributed)."""
    import torch.distributed as dist
    from .eclip import Session
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    s = Session(profiles, problem=problem, shard=rank, n_shards=world, **kw)
    try:
        return run_sharded(s, TorchComm(group))
    finally:
        s.close()


def nccl_comm(group=None, device=None):
    """The library's own communicator (eclip_comm, NCCL over NVLink / NVSwitch) for the ranks of a
    torch.distributed group: rank 0 draws the NCCL unique id, the group broadcasts it, every rank
    creates its communicator on its device.  Pass it as comm= to plan / plan_problem / plan_batch:
    the library then shards the candidate space and runs the exchanges on device buffers."""
    import torch
    import torch.distributed as dist
    from .eclip import Comm
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    dev = torch.cuda.current_device() if device is None else device
    return Comm.create(obj[0], world, rank, dev)


def plan_nccl(profiles, problem, comm, **kw):
    """eclip_plan of one problem sharded over `comm` (every rank gets the same plan)."""
    from .eclip import plan_problem
    return plan_problem(profiles, problem, comm=comm, **kw)


def pack_tuple(levels) -> np.ndarray:
    """level tuple -> [4] uint64 limbs of sum_w l_w << 16 (15 - w) (include/eclip.h)"""
    v = 0
    for w, l in enumerate(levels):
        v |= int(l) << (16 * (15 - w))
    return np.array([(v >> (64 * i)) & 0xFFFFFFFFFFFFFFFF for i in range(4)], np.uint64)


def unpack_tuple(limbs, W: int):
    v = sum(int(limbs[i]) << (64 * i) for i in range(4))
    return [(v >> (16 * (15 - w))) & 0xFFFF for w in range(W)]
