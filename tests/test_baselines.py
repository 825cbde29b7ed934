"""the paper's comparison planners and the lookup table.

CPU (-m "not gpu"): oracle/baselines.py pinned to SPEC's worked examples, closed
forms of the model, and the FNV-1a test vectors; the C-ABI lookup-table serializer (host
code, no GPU work) against the oracle.  GPU: eclip_baseline_plan against the oracle's exact
evaluation of the same plan, and the comparison structure of PAPER.md §V (ECLIP never worse
than a budget- and QoS-feasible baseline; Table I: ECLIP uses at most 14 switches per worker).
"""
import json
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import baselines as ob
import paper_2506_12598_b200 as ec

US = 1000  # ns per microsecond


def _mk(times_us, sizes=(15, 30, 45, 60)):
    return synth.Model("m", list(sizes), np.array(times_us, dtype=np.int64) * US)


# ------------------------------------------------------------------ oracle pins (CPU)
def test_threshold_spec_examples():
    """SPEC S:84-87."""
    allowed = [0, 1, 2, 3]
    assert ob.min_cu_threshold([20 * US] * 4, allowed, 0.05) == 0            # flat -> 15
    assert ob.min_cu_threshold([40 * US, 21 * US, 20 * US, 20 * US], allowed, 0.05) == 1   # -> 30
    assert ob.min_cu_threshold([40, 30, 25, 20], allowed, 0.0) == 3          # strictly decreasing -> 60
    # 21 <= 1.05 * 20 = 21 holds with equality: the predicate is inclusive ("<=")
    assert ob.min_cu_threshold([40, 21, 20, 20], allowed, 0.05) == 1
    assert ob.min_cu_threshold([40, 22, 20, 20], allowed, 0.05) == 2
    # allowed-size restriction: the largest allowed size is the reference point
    assert ob.min_cu_threshold([40, 21, 20, 10], [0, 1, 2], 0.05) == 1


def test_rightsize_spec_examples():
    """SPEC S:95-98, the 3-kernel case evaluated by hand."""
    allowed = [0, 1, 2, 3]
    assert ob.model_wise_rightsize([[20] * 4, [7] * 4], allowed, 3.0) == 0           # flat -> 15
    assert ob.model_wise_rightsize([[9, 9, 9, 9], [40, 30, 25, 20]], allowed, 1.0) == 3  # factor 1 -> 60
    t = [[90, 40, 30, 30], [60, 30, 20, 20], [30, 20, 10, 10]]   # column sums 180, 90, 60, 60
    assert ob.model_wise_rightsize(t, allowed, 3.0) == 0          # 180 <= 3 x 60
    assert ob.model_wise_rightsize(t, allowed, 2.9) == 1          # 180 > 174, 90 <= 174


def test_rightsize_hand_case_1_4():
    t = [[90, 40, 30, 30], [60, 30, 20, 20], [30, 20, 10, 10]]
    assert ob.model_wise_rightsize(t, [0, 1, 2, 3], 1.4) == 2     # 1.4 x 60 = 84 < 90; 60 <= 84


def test_threshold_monotone_in_tolerance():
    rng = np.random.default_rng(3)
    for _ in range(200):
        t = sorted(rng.integers(1, 10**6, size=5).tolist(), reverse=True)
        allowed = sorted(set(rng.integers(0, 5, size=3).tolist()))
        prev = None
        for tol in (0.0, 0.01, 0.05, 0.2, 1.0, 5.0):
            j = ob.min_cu_threshold(t, allowed, tol)
            assert j in allowed
            assert t[j] <= (1 + Fraction(tol).limit_denominator(10**9)) * t[max(allowed)]
            if prev is not None:
                assert j <= prev
            prev = j


def test_fnv1a64_vectors():
    """the published FNV-1a 64 test vectors"""
    assert ob.fnv1a64(b"") == 0xCBF29CE484222325
    assert ob.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert ob.fnv1a64(b"foobar") == 0x85944171F73967E8


def _prob(models, ids, N=60, mode="exclude_self", objective="sum", **kw):
    return synth.Problem("t", models, ids, N, 14, mode, objective, **kw)


def test_all_max_closed_form():
    """ALL_MAX at c = N in EXCLUDE_SELF: every other worker averages N CUs, alpha = W - 1,
    L_w = W beta_w; a single worker recovers its solo time (alpha = 0)."""
    m1 = _mk([[40, 30, 25, 20], [10, 9, 8, 7]])
    m2 = _mk([[5, 5, 5, 5]])
    for ids in ([0], [0, 1], [0, 1, 1]):
        p = _prob([m1, m2], ids)
        cols = ob.baseline_columns(p, "all_max", 0)
        ev = ob.evaluate_columns(p, cols)
        W = len(ids)
        solo = [27 * US, 5 * US]
        assert [float(x) for x in ev["L"]] == [W * solo[i] for i in ids]
        assert ev["switches"] == [0] * W
        # power at full occupancy (min(1, sum avg / N) = 1): p_max
        assert float(ev["power"]) == 225.0


def test_kernel_wise_switch_count():
    m = _mk([[40, 21, 20, 20], [40, 40, 40, 40], [90, 50, 30, 29], [50, 49, 48, 10]])
    p = _prob([m], [0])
    cols = ob.baseline_columns(p, "kernel_wise", 0.05)
    assert cols == [[1, 0, 2, 3]]
    ev = ob.evaluate_columns(p, cols)
    assert ev["switches"] == [3] and ev["group_sm"] == [[30, 15, 45, 60]]
    assert float(ev["L"][0]) == (21 + 40 + 30 + 10) * US


def test_lookup_table_spec_examples():
    """1 worker, 3 kernels at [15,15,30] -> 3 entries; round trip; hash iff change."""
    m = _mk([[1, 1, 1, 1]] * 3)
    p = _prob([m], [0])
    canon, text, h = ob.lookup_table(p, [[15, 15, 30]])
    d = json.loads(text)
    assert d["workers"] == [{"worker_id": 0, "configs": [15, 15, 30]}]
    assert d["meta"] == {"hash": f"0x{h:016x}", "mode": "exclude_self", "switch_max": 14}
    # the hash covers exactly the serialization without the hash member
    d2 = json.loads(text)
    del d2["meta"]["hash"]
    assert json.dumps(d2, separators=(",", ":")).encode() == canon
    assert ob.fnv1a64(canon) == h
    seen = {h}
    for k in range(3):
        for c in (15, 30, 45, 60):
            cfg = [15, 15, 30]
            if cfg[k] == c:
                continue
            cfg[k] = c
            _, _, h2 = ob.lookup_table(p, [cfg])
            assert h2 not in seen
            seen.add(h2)
    assert ob.lookup_table(p, [[15, 15, 30]])[2] == h


def _c_table(p, group_sm):
    pr = ec.Profiles.from_models(p.models)
    return ec.lookup_table_json(pr, p.model_ids, group_sm, total_sms=p.total_sms, switch_max=p.switch_max,
                                slowdown=p.mode, group_bounds=p.group_bounds, slowdown_matrix=p.slowdown_matrix)


@pytest.mark.parametrize("seed", range(12))
def test_lookup_table_c_abi_equals_oracle(seed):
    """host-side serializer of the library vs the oracle, byte for byte"""
    p = synth.random_tiny_problem(seed)
    rng = np.random.default_rng(seed)
    gsm = []
    for w in range(p.W):
        gb = p.group_bounds[w] if p.group_bounds is not None and p.group_bounds[w] is not None else None
        G = len(gb) - 1 if gb else p.models[p.model_ids[w]].n_kernels
        gsm.append([int(x) for x in rng.choice(p.sizes, size=G)])
    text, h = _c_table(p, gsm)
    _, otext, oh = ob.lookup_table(p, gsm)
    assert text == otext and h == oh


# ------------------------------------------------------------------ GPU parity
KINDS = [("all_max", 0.0), ("model_wise", 3.0), ("model_wise", 1.25), ("kernel_wise", 0.05), ("kernel_wise", 0.0)]


def _check(p, kind, param):
    pr = ec.Profiles.from_models(p.models)
    g = ec.baseline_plan(pr, p.model_ids, kind=kind, param=param, total_sms=p.total_sms, switch_max=p.switch_max,
                         slowdown=p.mode, objective=p.objective, allowed_mask=p.allowed_mask, qos_ns=p.qos_ns,
                         slowdown_matrix=p.slowdown_matrix, group_bounds=p.group_bounds, p_idle_w=p.p_idle_w,
                         p_max_w=p.p_max_w)
    cols = ob.baseline_columns(p, kind, param)
    ev = ob.evaluate_columns(p, cols)
    label = f"{p.name} {kind} {param}"
    assert g.engine == "baseline", label
    assert g.group_sm == ev["group_sm"], label
    assert g.model_switches == ev["switches"], label
    assert g.status == ("ok" if ev["feasible"] else "infeasible"), label
    rel = 1e-9
    for a, b in zip(g.model_latency_ns, ev["L"]):
        assert a == pytest.approx(float(b), rel=rel), label
    mk = max(ev["L"])
    assert g.makespan_ns == pytest.approx(float(mk), rel=rel), label
    assert g.power_w == pytest.approx(float(ev["power"]), rel=rel), label
    assert g.objective == pytest.approx(float(ev["key"]), rel=rel), label
    assert g.energy_j == pytest.approx(float(ev["power"] * mk) * 1e-9, rel=rel), label
    assert g.throughput_rps == pytest.approx(sum(1e9 / float(x) for x in ev["L"]), rel=rel), label
    for w in range(p.W):
        for gl, gsz in zip(g.group_latency_ns[w], g.group_sm[w]):
            assert gl > 0
    return g, ev


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(40))
def test_baseline_random_vs_oracle(seed):
    p = synth.random_tiny_problem(1000 + seed, max_w=4, max_g=6)
    for kind, param in KINDS:
        _check(p, kind, param)


@pytest.mark.gpu
def test_baseline_c2_c3_c5_vs_oracle():
    probs = [synth.make_c2(m, o) for m in ("exclude_self", "paper", "excess", "matrix") for o in ("sum", "max", "energy")]
    probs.append(synth.make_c3())
    models, ids, qos = synth.make_c5(n_mixes=16)
    probs += [synth.c5_problem(i, models, ids, qos) for i in range(16)]
    for p in probs:
        for kind, param in KINDS:
            _check(p, kind, param)


@pytest.mark.gpu
def test_eclip_never_worse_than_feasible_baselines_and_table1():
    """PAPER.md §V: the optimizer's plan is the optimum over every plan with <= R switches that
    meets QoS, so any such baseline plan is at least as costly (up to tie_tol); Table I: ECLIP
    uses at most switchMax = 14 switches per worker (sum <= 14 W), KW typically many more."""
    models, ids, qos = synth.make_c5(n_mixes=24, seed=3)
    kw_more = 0
    for i in range(24):
        p = synth.c5_problem(i, models, ids, qos)
        pr = ec.Profiles.from_models(p.models)
        opt = ec.plan_problem(pr, p)
        if opt.status == "ok":
            assert sum(opt.model_switches) <= 14 * p.W
        for kind, param in KINDS:
            g, ev = _check(p, kind, param)
            if g.status == "ok" and max(g.model_switches) <= p.switch_max:
                assert opt.status == "ok"
                assert opt.objective <= g.objective * (1 + 1e-5) + 1e-6
            if kind == "kernel_wise" and param == 0.05 and opt.status == "ok":
                kw_more += sum(g.model_switches) >= sum(opt.model_switches)
    assert kw_more >= 1


@pytest.mark.gpu
def test_baseline_invalid_args():
    p = synth.make_c2()
    pr = ec.Profiles.from_models(p.models)
    with pytest.raises(ec.EclipError):
        ec.baseline_plan(pr, p.model_ids, kind="model_wise", param=0.5, total_sms=p.total_sms)
    with pytest.raises(ec.EclipError):
        ec.baseline_plan(pr, p.model_ids, kind="kernel_wise", param=-1.0, total_sms=p.total_sms)
