"""Runtime scheduler (include/eclip_runtime.h): the oracle's layout and barrier
rules pinned to the paper (CPU), the library exports (CPU), and on the GPU the runtime's recorded
decisions and device timelines checked against the oracle: redirection, barrier placement,
dependency safety, SM-partition discipline."""
import os
import re

import numpy as np
import pytest

import oracle.runtime as ort
import paper_2506_12598_b200 as ec
from paper_2506_12598_b200 import runtime as rt_mod

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------------------------------- CPU
def test_layout_pinned_to_paper_two_worker_example():
    """worker 1 gets 15 CU (SE1), 30 (SE1,3), 45 (SE1,2,3); worker 2 15 (SE4), 30 (SE2,4),
    45 (SE2,3,4).  The rotation layout reproduces the sizes and every pairwise overlap."""
    paper = {1: ({1}, {4}), 2: ({1, 3}, {2, 4}), 3: ({1, 2, 3}, {2, 3, 4})}
    for j, (a, b) in paper.items():
        ga, gb = ort.pool_groups(4, 2, 0, j), ort.pool_groups(4, 2, 1, j)
        assert len(ga) == len(a) == j and len(gb) == len(b) == j
        assert ort.pairwise_overlap(4, 2, j, 0, 1) == len(a & b)
    assert ort.pool_groups(4, 2, 0, 4) == [0, 1, 2, 3]   # "the 60 CU allocation is the default stream"


def test_layout_small_pools_disjoint():
    for G in (4, 8, 9):
        for W in range(1, 9):
            if W > G:
                continue
            for j in range(1, G // W + 1):   # pools of <= G/W groups never overlap
                for a in range(W):
                    for b in range(a + 1, W):
                        assert ort.pairwise_overlap(G, W, j, a, b) == 0


def test_needs_barrier_spec_examples():
    """SPEC needs_barrier examples."""
    assert not ort.needs_barrier(-1, 3, True)      # first kernel of a request
    assert not ort.needs_barrier(3, 3, True)       # same masked stream, running: FIFO suffices
    assert ort.needs_barrier(2, 3, True)           # different stream, signal pending
    assert not ort.needs_barrier(2, 3, False)      # different stream, completed


def test_dependency_checker():
    assert ort.dependency_ok([0, 10, 20], [10, 20, 30])
    assert not ort.dependency_ok([0, 9], [10, 20])


def test_runtime_symbols_exported_and_no_cpu_fallback():
    txt = open(os.path.join(ROOT, "include", "eclip_runtime.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = sorted(set(re.findall(r"\b(eclip_rt_[a-z0-9_]+)\s*\(", txt)))
    assert len(names) == 9
    L = ec.lib()
    for n in names:
        assert hasattr(L, n), n
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(ec.EclipError) as e:
            rt_mod.Runtime(2)
        assert e.value.code == ec.eclip.E_CUDA


# ---------------------------------------------------------------------------------------- GPU
def _models(rng, W, K, sizes):
    ms = []
    for w in range(W):
        ctas = rng.choice([8, 16, 32, 64, 128, 148], size=K)
        iters = rng.integers(2000, 20000, size=K)
        ms.append(rt_mod.SyntheticModel(ctas, iters))
    return ms


@pytest.mark.gpu
@pytest.mark.parametrize("W", [1, 2, 4])
def test_gpu_layout_matches_oracle(W):
    rt = rt_mod.Runtime(W, group_sms=16)
    G = rt.n_groups
    assert G >= 2 and len(rt.sizes) == G and rt.sizes[-1] == rt.total_sms
    assert rt.sizes == sorted(rt.sizes)
    for w in range(W):
        for j in range(G):
            lay = rt.layout(w, j)
            want = ort.pool_groups(G, W, w, j + 1)
            got = [g for g in range(G) if (lay["group_mask"] >> g) & 1]
            assert got == want, (w, j)
            assert lay["sm_count"] == (rt.total_sms if j == G - 1 else sum(rt.group_sm[g] for g in want))
    rt.close()


@pytest.mark.gpu
@pytest.mark.parametrize("repartition", [False, True])
def test_gpu_dispatch_redirect_barrier_dependency(repartition):
    W, K, R = 2, 12, 6
    rng = np.random.default_rng(17 + repartition)
    rt = rt_mod.Runtime(W, group_sms=16)
    models = _models(rng, W, K, rt.sizes)
    tables = []
    for w in range(W):
        t = rng.choice(rt.sizes, size=K)
        t[: K // 3] = t[0]                       # a same-stream run (no barrier possible)
        rt.set_table(w, t)
        tables.append(t)
    out = rt.run(models, R, record=True, repartition=repartition)
    assert out["latency_ns"].shape == (W, R) and (out["latency_ns"] > 0).all()
    for w in range(W):
        for r in range(R):
            ts, te = out["t_start"][w, r], out["t_end"][w, r]
            assert ort.dependency_ok(ts, te), (w, r)
            for k in range(K):
                j = ort.redirect(rt.sizes, tables[w], k)
                sid = out["stream_id"][w, r, k]
                if not repartition:
                    assert sid == rt.layout(w, j)["stream_id"]
                    if k > 0:
                        prev = out["stream_id"][w, r, k - 1]
                        if out["barrier"][w, r, k]:
                            assert prev != sid          # a barrier only across streams
                        if prev == sid:
                            assert out["barrier"][w, r, k] == 0
                    else:
                        assert out["barrier"][w, r, k] == 0   # the previous request was observed complete
                assert 1 <= out["sm_used"][w, r, k] <= rt.layout(w, j)["sm_count"]
    if repartition:
        assert out["repartition_ns"] > 0
    else:
        # partition discipline: all CTAs of one pool stream ran inside one set of sm_count SMs, and
        # pools whose groups are disjoint ran on disjoint SMs
        used = {}
        for w in range(W):
            for r in range(R):
                for k in range(K):
                    sid = int(out["stream_id"][w, r, k])
                    m = used.setdefault(sid, np.zeros(5, np.uint32))
                    m |= out["sm_mask"][w, r, k]
        info = {}
        for w in range(W):
            for j in range(len(rt.sizes)):
                lay = rt.layout(w, j)
                info[lay["stream_id"]] = lay
        popc = lambda m: int(sum(bin(int(x)).count("1") for x in m))
        for sid, m in used.items():
            assert popc(m) <= info[sid]["sm_count"], sid
        for a in used:
            for b in used:
                if a < b and info[a]["group_mask"] & info[b]["group_mask"] == 0:
                    assert popc(used[a] & used[b]) == 0, (a, b)
    rt.close()


@pytest.mark.gpu
def test_gpu_profile_knee_shape():
    """a kernel of c CTAs is ~flat on pools >= c SMs and slower on smaller pools (P:149 knee)"""
    rt = rt_mod.Runtime(1, group_sms=16)
    m = rt_mod.SyntheticModel([32, 148, 8], [20000, 20000, 20000])
    t = rt.profile(m, reps=5)
    sizes = np.array(rt.sizes)
    for k in range(3):
        assert (np.diff(t[k]) <= 0.10 * t[k, :-1]).all(), t[k]   # non-increasing within 10 %
    big = sizes >= 32
    assert t[0, big].max() <= 1.15 * t[0, big].min()
    assert t[0, sizes == 16][0] >= 1.6 * t[0, -1]                # 2 waves on 16 SMs
    assert t[1, 0] >= 4.0 * t[1, -1]                             # 148 CTAs on 16 SMs
    assert t[2].max() <= 1.15 * t[2].min()                       # 8 CTAs: flat everywhere
    rt.close()
