"""Multi-process (world_size 2, gloo on CPU) coverage of the sharded planning protocol of
paper_2506_12598_b200/parallel.py: the three cross-rank reductions and run_sharded.
The per-shard work is provided by an oracle-backed stand-in session (the CUDA sessions
are covered by tests/test_gpu_parity.py::test_sharded_*)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import synth
from paper_2506_12598_b200 import parallel


class OracleShardSession:
    """Same step interface as eclip.Session, computed by the oracle over a contiguous
    index shard [total*s/n, total*(s+1)/n)."""
    single = True

    def __init__(self, problem, shard, n_shards):
        self.pp = oracle.Prepared(problem)
        tot = self.pp.n_tuples
        self.lo, self.hi = tot * shard // n_shards, tot * (shard + 1) // n_shards

    def pass1(self):
        r = oracle._Result()
        oracle.lib().or_enum_min_range(C.byref(self.pp.c), self.lo, self.hi, C.byref(r))
        self._min = None if r.status else [int(r.min_key[i]) for i in range(4)]
        return np.array([np.inf if self._min is None else float(oracle._key_int(self._min))], np.float32)

    def pass2_min(self, m):
        return np.array([self._min if self._min is not None else [2**64 - 1] * 4], np.uint64)

    def pass2_first(self, k):
        none = np.full((1, 4), 2**64 - 1, np.uint64)
        if np.all(k == np.uint64(2**64 - 1)):
            return none
        r = oracle._Result()
        kk = (C.c_uint64 * 4)(*[int(x) for x in k[0]])
        oracle.lib().or_enum_first_within(C.byref(self.pp.c), self.lo, self.hi, kk, C.byref(r))
        if r.status:
            return none
        return parallel.pack_tuple([r.levels[w] for w in range(self.pp.W)])[None, :]

    def finish(self, f):
        if np.all(f == np.uint64(2**64 - 1)):
            return None
        return parallel.unpack_tuple(f[0], self.pp.W)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, seeds, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = parallel.TorchComm()
    res = []
    for s in seeds:
        p = synth.random_tiny_problem(s, max_w=3, max_g=3, max_c=3)
        res.append(parallel.run_sharded(OracleShardSession(p, rank, world), comm))
    # the raw reductions
    a = comm.min_f32(np.array([1.0 + rank, np.inf], np.float32))
    b = comm.min_u64(np.array([parallel.U64_NONE, 5 + rank], np.uint64))
    keys = np.array([[rank, 0, 0, 1 - rank], [7, 7, 7, 7]], np.uint64)
    c = comm.min_u256(keys)
    q.put((rank, res, a.tolist(), b.tolist(), c.tolist()))
    dist.destroy_process_group()


def test_two_rank_gloo_protocol_matches_oracle():
    world, seeds = 2, list(range(40))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seeds, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    outs.sort()
    assert outs[0][1] == outs[1][1]                      # identical plans on every rank
    for s, lv in zip(seeds, outs[0][1]):
        o = oracle.solve(synth.random_tiny_problem(s, max_w=3, max_g=3, max_c=3))
        if o.status == "ok":
            assert lv == o.levels, s
        else:
            assert lv is None, s
    for rank, _, a, b, c in outs:
        assert a == [1.0, float("inf")]
        assert b == [int(parallel.U64_NONE), 5]
        assert c == [[1, 0, 0, 0], [7, 7, 7, 7]]         # (hi limb last) lexicographic min


def test_pack_tuple_order_is_index_order():
    import itertools
    L = [3, 4, 2]
    tuples = list(itertools.product(*[range(x) for x in L]))
    packed = [parallel.pack_tuple(t) for t in tuples]
    assert [parallel.unpack_tuple(p, 3) for p in packed] == [list(t) for t in tuples]
    keys = [tuple(int(x) for x in p[::-1]) for p in packed]
    assert keys == sorted(keys)


def test_lexmin_u256_orders_by_high_limb():
    a = np.array([[[5, 0, 0, 1]], [[0, 0, 0, 2]], [[9, 9, 9, 0]]], np.uint64)
    assert parallel.lexmin_u256(a).tolist() == [[9, 9, 9, 0]]
