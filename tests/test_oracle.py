"""Pins for the oracle (O-A literal brute force, O-B reduced exact) against what the paper
and mathematics fix: printed values, hand-worked examples, closed forms, brute force,
invariants.  CPU only."""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from oracle import brute
from synth.profiles import Model

GOLD = os.path.join(os.path.dirname(__file__), "golden", "appB_examples.json")


def _golden_problem(case, gold):
    sizes = gold["sizes"]
    models, ids = [], []
    for w, groups in enumerate(case["workers"]):
        ex = np.array([[int(round(v * 1000)) for v in gold["profiles_us"][g]] for g in groups], dtype=np.int64)
        models.append(Model(f"w{w}", sizes, ex))
        ids.append(w)
    return synth.Problem(case["name"], models, ids, gold["N"], case["R"], case["mode"], case["objective"],
                         p_idle_w=case.get("p_idle", 75.0), p_max_w=case.get("p_max", 225.0))


# ---------------------------------------------------------------- SPEC printed values
def test_estimate_exec_printed_values():
    # S:158-160
    assert brute.estimate_exec(Fraction(10), 0) == 10
    assert brute.estimate_exec(Fraction(10), 1) == 20                      # P:309 doubling
    assert brute.estimate_exec(Fraction("19.8"), Fraction(1, 2)) == Fraction("29.7")


def test_cu_overlap_printed_values():
    # S:171-173
    assert brute.cu_overlap([Fraction(60)], 0, "exclude_self", 60) == 0
    assert brute.cu_overlap([Fraction(60), Fraction(60)], 0, "exclude_self", 60) == 60
    assert brute.cu_overlap([Fraction(30), Fraction(45)], 1, "paper", 60) == 75


def test_alpha_printed_values():
    # S:181-183
    assert brute.alpha(0, 60) == 0
    assert brute.alpha(60, 60) == 1
    assert brute.alpha(75, 60) == Fraction(5, 4)


def test_switch_count_printed_and_indicator_form():
    # S:221-223 and P:302's |x_{k,c} - x_{k-1,c}|/2
    assert brute.switch_count([15, 15, 15]) == 0
    assert brute.switch_count([15, 30, 15]) == 2
    rng = np.random.default_rng(3)
    for _ in range(20):
        seq = [int(x) for x in rng.choice([15, 30, 45, 60], size=100)]
        assert brute.switch_count(seq) == brute.switch_count_indicator(seq, [15, 30, 45, 60])
    with pytest.raises(ValueError):
        brute.switch_count([])


def test_power_at_printed_values():
    # S:412-414
    assert brute.power_at(0, 60, 75, 225) == 75
    assert brute.power_at(60, 60, 75, 225) == 225
    assert brute.power_at(30, 60, 75, 225) == 150


# ---------------------------------------------------------------- App. B worked examples
@pytest.mark.parametrize("idx", range(10))
def test_worked_examples(idx):
    gold = json.load(open(GOLD))
    case = gold["cases"][idx]
    p = _golden_problem(case, gold)
    a = brute.brute_force(p)
    assert a is not None
    assert float(a["key"]) == pytest.approx(case["expect_J"] * 1000, rel=1e-12)    # us -> ns
    assert [[gold["sizes"][j] for j in s] for s in a["sigmas"]] == case["expect_sizes"]
    # O-A's own values of the plan: makespan and power (hand values in the golden)
    assert float(max(a["L"])) == pytest.approx(case["expect_makespan_us"] * 1000, rel=1e-12)
    assert float(a["power"]) == pytest.approx(case["expect_power_w"], rel=1e-12)
    for engine in ("enum",) + (("slice",) if p.mode != "matrix" else ()):
        b = oracle.solve(p, engine)
        assert b.group_sm == case["expect_sizes"], engine
        assert b.objective == pytest.approx(case["expect_J"] * 1000, rel=1e-12)
        # or_eval_f64's reported values against the hand values (units: ns, W, J, requests/s)
        assert b.makespan_ns == pytest.approx(case["expect_makespan_us"] * 1000, rel=1e-12)
        assert b.power_w == pytest.approx(case["expect_power_w"], rel=1e-12)
        assert b.energy_j == pytest.approx(case["expect_energy_j"], rel=1e-12)
        assert b.throughput_rps == pytest.approx(case["expect_throughput_rps"], rel=1e-12)


def test_doubling_anecdote_two_and_three_workers():
    """P:309 footnote: two identical kernels sharing the same CUs both take twice as long;
    generalised: W identical heavy single-group workers -> all at max, L = W beta(max)."""
    gold = json.load(open(GOLD))
    for W in (2, 3):
        case = dict(workers=[["heavy"]] * W, R=0, mode="exclude_self", objective="sum", name="dbl")
        p = _golden_problem(case, gold)
        r = oracle.solve(p)
        assert r.group_sm == [[60]] * W
        for Lw in r.latency_ns:
            assert Lw == pytest.approx(W * 20_000, rel=1e-12)


def test_single_worker_exclude_self_recovers_solo_time():
    """alpha = 0 recovers the solo profile."""
    for seed in range(5):
        p = synth.make_c1(R=seed % 3, seed=seed)
        p.model_ids = [0]
        r = oracle.solve(p)
        assert r.alpha == [0.0]
        S, B, wit, beta, n = r.tables[0]
        assert r.latency_ns[0] == float(B[r.levels[0]])
        # single worker SUM optimum = min over all budget-feasible plans of B
        assert r.latency_ns[0] == float(B.min())


# ---------------------------------------------------------------- level tables
def _brute_levels(beta, n, sizes, mask, R):
    G, Cn = beta.shape
    allowed = [j for j in range(Cn) if (mask >> j) & 1]
    best = {}
    for sig in itertools.product(allowed, repeat=G):
        if brute.switch_count(sig) > R:
            continue
        S = sum(int(n[g]) * sizes[sig[g]] for g in range(G))
        B = sum(int(beta[g, sig[g]]) for g in range(G))
        if S not in best or (B, sig) < best[S]:
            best[S] = (B, sig)
    return sorted((sig, S, B) for S, (B, sig) in best.items())


def test_levels_vs_brute_force():
    """S:237 DP optimality: level table == exhaustive enumeration for G <= 6."""
    rng = np.random.default_rng(11)
    for t in range(40):
        G = int(rng.integers(1, 7))
        Cn = int(rng.integers(1, 5))
        sizes = synth.lattice_sizes(Cn, 60) if t % 2 else sorted(int(x) for x in rng.choice(np.arange(1, 30), Cn, replace=False))
        m = synth.synthesize_model("x", "uniform", G, sizes, 1000 + t)
        n = rng.integers(1, 3, size=G).astype(np.int32)
        mask = int(rng.integers(1, 1 << Cn))
        R = int(rng.integers(0, 4))
        S, B, wit = oracle.levels(m.exec_ns, n, sizes, mask, R)
        ref = _brute_levels(m.exec_ns, n, sizes, mask, R)
        assert [tuple(int(x) for x in w) for w in wit] == [r[0] for r in ref]
        assert list(S) == [r[1] for r in ref]
        assert list(B) == [r[2] for r in ref]


def test_levels_closed_forms():
    """R = 0: one level per allowed size, B*(K c_j) = sum_g beta_gj.
    R >= G-1: min_S B*(S) = sum_g min_j beta_gj; lattice sizes -> B* non-increasing in S."""
    for seed in range(6):
        sizes = synth.lattice_sizes(8, 148)
        m = synth.synthesize_model("x", "uniform", 12, sizes, 77 + seed)
        n = np.ones(12, np.int32)
        S, B, wit = oracle.levels(m.exec_ns, n, sizes, 0xFF, 0)
        assert len(S) == 8
        for l in range(8):
            j = int(wit[l][0])
            assert all(int(x) == j for x in wit[l])
            assert S[l] == 12 * sizes[j] and B[l] == int(m.exec_ns[:, j].sum())
        S, B, wit = oracle.levels(m.exec_ns, n, sizes, 0xFF, 11)
        assert B.min() == int(m.exec_ns.min(axis=1).sum())
        order = np.argsort(S)
        assert np.all(np.diff(B[order]) <= 0)
        assert len(S) == 12 * 7 + 1       # L = G (C-1) + 1 on the lattice


def test_level_count_c4_shape():
    """L = G (C-1) + 1 = 577 for 64 groups x 10 lattice sizes."""
    p = synth.make_c4()
    pp = oracle.Prepared(p)
    assert list(pp.L) == [577] * 8


# ---------------------------------------------------------------- O-A == O-B
def test_reduction_matches_brute_force_random():
    """SURVEY §8(c) c6 'reduction': O-B (level reduction, exact) == O-A (raw brute force)
    on random tiny instances: every mode, objective, QoS on/off, masks, groups, ties."""
    n_checked = 0
    for s in range(400):
        p = synth.random_tiny_problem(s)
        try:
            a = brute.brute_force(p)
        except ValueError:
            continue
        b = oracle.solve(p)
        if a is None:
            assert b.status == "infeasible", s
            continue
        assert b.status == "ok"
        assert b.group_cols == a["sigmas"], s
        assert b.objective == pytest.approx(float(a["key"]), rel=1e-12), s
        for w in range(p.W):
            assert b.latency_ns[w] == pytest.approx(float(a["L"][w]), rel=1e-12)
        n_checked += 1
    assert n_checked > 300


def test_level_efficient_restriction_is_exact_for_sum_tau0():
    """App. A.1: with SUM and tau = 0 every exact optimum is level-efficient, so the raw
    lexicographic arg-min over ALL joint plans equals the reduced answer."""
    n = 0
    for s in range(200):
        p = synth.random_tiny_problem(s, max_w=2, max_g=3, max_c=3)
        p.objective = "sum"
        try:
            raw = brute.brute_force(p, tol=0.0, level_efficient=False)
        except ValueError:
            continue
        red = brute.brute_force(p, tol=0.0, level_efficient=True)
        if raw is None:
            assert red is None
            continue
        assert raw["sigmas"] == red["sigmas"] and raw["key"] == red["key"]
        n += 1
    assert n > 100


@pytest.mark.parametrize("mode", ["exclude_self", "paper", "excess", "matrix"])
@pytest.mark.parametrize("objective", ["sum", "max", "energy"])
def test_level_efficient_restriction_keeps_the_exact_minimum(mode, objective):
    """App. A.1 for every slowdown mode, objective and QoS setting: the exact minimum over ALL
    raw joint plans (O-A without the level reduction) equals the minimum over level-efficient
    plans, and feasibility agrees.  (In MAX/ENERGY a raw minimiser need not be level-efficient —
    a non-bottleneck worker may take a slower plan at the same CU-sum — so only the minimum and
    the key of the reduced winner are compared; in SUM with tau = 0 the winners coincide.)"""
    n = n_qos = 0
    for s in range(60):
        p = synth.random_tiny_problem(3000 + s, max_w=2, max_g=3, max_c=3)
        p.mode, p.objective = mode, objective
        if mode == "matrix" and p.slowdown_matrix is None:
            rng = np.random.default_rng(s)
            p.slowdown_matrix = rng.uniform(0.5, 1.5, size=(p.W, p.W)).astype(np.float32)
            np.fill_diagonal(p.slowdown_matrix, 0.0)
        if mode != "matrix":
            p.slowdown_matrix = None
        try:
            raw = brute.brute_force(p, tol=0.0, level_efficient=False)
        except ValueError:
            continue
        red = brute.brute_force(p, tol=0.0, level_efficient=True)
        assert (raw is None) == (red is None), s
        if raw is None:
            continue
        assert raw["min_key"] == red["min_key"], s
        assert red["key"] == red["min_key"]
        if objective == "sum":
            assert raw["sigmas"] == red["sigmas"], s
        n += 1
        n_qos += p.qos_ns is not None
    assert n >= 40 and n_qos >= 10


def test_slice_equals_enum_random():
    """T'-slicing (App. A.2) == flat enumeration, exactly, on every linear-mode instance."""
    n = 0
    for s in range(300):
        p = synth.random_tiny_problem(1000 + s, max_w=4, max_g=4, max_c=4)
        if p.mode == "matrix":
            continue
        a = oracle.solve(p, "enum")
        b = oracle.solve(p, "slice")
        assert a.status == b.status
        if a.status == "ok":
            assert a.levels == b.levels and a.key == b.key and a.min_key == b.min_key
            n += 1
    assert n > 100


def test_slice_equals_enum_c2_all_objectives():
    for obj in ("sum", "max", "energy"):
        for mode in ("exclude_self", "paper", "excess"):
            p = synth.make_c2(mode, obj)
            a = oracle.solve(p, "enum")
            b = oracle.solve(p, "slice")
            assert a.levels == b.levels and a.key == b.key, (mode, obj)


# ---------------------------------------------------------------- invariants
def _exact_obj(p, r):
    """exact objective of the oracle's winner via O-A's evaluator"""
    choice = []
    for w in range(p.W):
        S, B, wit, beta, n = r.tables[w]
        choice.append((tuple(r.group_cols[w]), int(S[r.levels[w]]), int(B[r.levels[w]])))
    return brute.evaluate(p, choice)


def test_invariants_random():
    """Budget, allowed sizes <= N, QoS met, permutation invariance of J*, relaxations never
    increase J*, determinism, J*_SUM >= sum_w min B_w."""
    for s in range(120):
        p = synth.random_tiny_problem(2000 + s, max_w=3, max_g=3, max_c=4)
        r = oracle.solve(p)
        if r.status != "ok":
            continue
        C_ = len(p.sizes)
        for w in range(p.W):
            assert r.switches[w] <= p.switch_max
            mask = p.allowed_mask[w] if p.allowed_mask else (1 << C_) - 1
            assert all((mask >> j) & 1 for j in r.group_cols[w])
            assert all(sm <= p.total_sms for sm in r.group_sm[w])
        feas, key, L, pw, al = _exact_obj(p, r)
        assert feas
        # determinism
        r2 = oracle.solve(p)
        assert r2.levels == r.levels and r2.key == r.key
        # relaxing the budget never increases J*
        import copy
        q = copy.deepcopy(p); q.switch_max += 1
        m_p = Fraction(_min_obj(p)); m_q = Fraction(_min_obj(q))
        assert m_q <= m_p
        # removing QoS never increases J*
        if p.qos_ns is not None:
            q2 = copy.deepcopy(p); q2.qos_ns = None
            assert Fraction(_min_obj(q2)) <= m_p
        # worker permutation leaves J* invariant (matrix permuted accordingly)
        perm = list(reversed(range(p.W)))
        q3 = copy.deepcopy(p)
        q3.model_ids = [p.model_ids[i] for i in perm]
        if p.allowed_mask: q3.allowed_mask = [p.allowed_mask[i] for i in perm]
        if p.qos_ns: q3.qos_ns = [p.qos_ns[i] for i in perm]
        if p.group_bounds: q3.group_bounds = [p.group_bounds[i] for i in perm]
        if p.slowdown_matrix is not None: q3.slowdown_matrix = p.slowdown_matrix[np.ix_(perm, perm)]
        assert Fraction(_min_obj(q3)) == m_p
        if p.objective == "sum":
            lb = sum(int(r.tables[w][1].min()) for w in range(p.W))
            assert key >= lb


def _min_obj(p):
    """exact minimum objective (Fraction) via O-A-style evaluation of the O-B minimiser"""
    a = brute.brute_force(p, tol=0.0)
    return a["min_key"] if a else Fraction(10**30)


def test_table1_switch_structure():
    """P:407/P:418 (Table I): ECLIP per-request switches summed over workers <= 14 x W."""
    for p in (synth.make_c2(),):
        r = oracle.solve(p)
        assert sum(r.switches) <= 14 * p.W


# ---------------------------------------------------------------- profile files
def test_profile_roundtrip_and_rounding():
    ms = synth.make_c2().models
    txt = synth.write_profile_text(ms)
    back = oracle.parse_profiles(txt)
    assert len(back) == 3
    for a, b in zip(ms, back):
        assert np.array_equal(a.exec_ns, b.exec_ns) and a.sizes == b.sizes
    assert oracle.us_to_ns("12.3456") == 12346
    assert oracle.us_to_ns("0.0005") == 0          # half to even
    assert oracle.us_to_ns("0.0015") == 2
    assert oracle.us_to_ns("19.8") == 19800


def test_profile_errors():
    """parse failure; missing config column; non-monotone row naming the kernel."""
    good = '{"model": "m", "kernels": 2, "configs": [15, 30, 45, 60]}\n0, 4, 3, 2, 1\n1, 5, 5, 5, 5\n'
    assert len(oracle.parse_profiles(good)) == 1
    with pytest.raises(oracle.ProfileError, match="non-monotone.*kernel 1"):
        oracle.parse_profiles(good.replace("1, 5, 5, 5, 5", "1, 5, 4, 4.5, 4"))
    with pytest.raises(oracle.ProfileError, match="missing config"):
        oracle.parse_profiles(good.replace("0, 4, 3, 2, 1", "0, 4, 3, 2"))
    with pytest.raises(oracle.ProfileError, match="parse failure"):
        oracle.parse_profiles("not json\n")
    with pytest.raises(oracle.ProfileError, match="non-positive"):
        oracle.parse_profiles(good.replace("0, 4, 3, 2, 1", "0, 4, 3, 2, 0"))


# ---------------------------------------------------------------- the stored C5 answers
def test_c5_golden_table_is_the_live_oracle():
    """tests/golden/c5_mixes.json (every distinct C5 mix, tools/gen_c5_golden.py) is current: the
    library it was computed on hashes the same and sampled entries equal the live oracle."""
    import golden_c5
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import gen_c5_golden
    doc = golden_c5.load()
    models, _, _ = synth.make_c5(1)
    assert doc["library_hash"] == gen_c5_golden.library_hash(models), "stale golden: rerun tools/gen_c5_golden.py"
    assert doc["n_mixes"] == 7 ** 4 == len(doc["answers"])
    rng = np.random.default_rng(5)
    solo = np.array([synth.qos_3x(models, [m])[0] for m in range(len(models))])
    for _ in range(8):
        ids = rng.integers(0, 7, size=(1, 4)).astype(np.int32)
        r = oracle.solve(synth.c5_problem(0, models, ids, solo[ids]), "slice")
        a = doc["answers"][",".join(map(str, ids[0]))]
        assert a[0] == r.status
        if r.status == "ok":
            assert a[1] == r.levels and a[2] == r.index and int(a[3], 16) == r.key
            assert float(a[4]) == r.objective
            assert a[5] == "".join("%x" % c for row in r.group_cols for c in row)



# ---------------------------------------------------------------- per-worker weights (reading R20)
def _ex1_weighted(objective, weights):
    gold = json.load(open(GOLD))
    case = dict(gold["cases"][0])        # Ex1: two 'heavy' workers, one group each, ExcludeSelf
    case["objective"] = objective
    p = _golden_problem(case, gold)
    p.weights = weights
    return p


@pytest.mark.parametrize("objective,expect_sizes,expect_J_us", [
    # weights (3, 1), hand-enumerated over the 16 plans (SURVEY App. B profile 'heavy' = 80/40/27/20 us):
    # SUM  3 L0 + L1: (60,45) = 3*20*1.75 + 27*2 = 105 + 54 = 159 < (60,60) = 160 < (60,30) = 170
    ("sum", [[60], [45]], 159.0),
    # MAX  max(3 L0, L1): (60,30) = max(3*20*1.5, 40*2) = max(90, 80) = 90 < (60,45) = 105
    ("max", [[60], [30]], 90.0)])
def test_weighted_worked_example(objective, expect_sizes, expect_J_us):
    """Hand-worked weighted Ex1: weights change the decision (unweighted optimum is (60,60))."""
    p = _ex1_weighted(objective, [3.0, 1.0])
    a = brute.brute_force(p)
    assert [[15, 30, 45, 60][j] for s in a["sigmas"] for j in s] == [x for s in expect_sizes for x in s]
    assert float(a["key"]) == pytest.approx(expect_J_us * 1000, rel=1e-12)
    for engine in ("enum", "slice"):
        b = oracle.solve(p, engine)
        assert b.group_sm == expect_sizes, engine
        assert b.objective == pytest.approx(expect_J_us * 1000, rel=1e-12), engine


def test_weight_rounding_and_validation():
    """R20: omega -> round-half-up(omega 1e6) / 1e6; exact keys use the gcd-reduced integers."""
    assert oracle.weight_ints([2.0, 1.0, 0.5], 3) == ([4, 2, 1], [2.0, 1.0, 0.5])
    assert oracle.weight_ints([0.1, 0.2, 0.7], 3)[0] == [1, 2, 7]
    assert oracle.weight_ints(None, 2) == ([1, 1], [1.0, 1.0])
    assert oracle.weight_ints([1.0000004, 1.0], 2)[0] == [1, 1]          # below the 1e-6 resolution
    assert oracle.weight_ints([2.5e-6, 1.0], 2)[0][0] == 3                # ... 2.5 rounds half up
    for bad in ([0.0, 1.0], [-1.0, 1.0], [float("nan"), 1.0], [1001.0, 1.0], [1e-7, 1.0]):
        with pytest.raises(ValueError):
            oracle.weight_ints(bad, 2)


def test_weighted_equals_brute_force_random():
    """O-B (level reduction, exact integer keys, enum and slice) == O-A (literal brute force in
    Fractions) with random per-worker weights, every mode and SUM / MAX; uniform weights give the
    unweighted answer with the identical exact key (the gcd reduction makes them all 1)."""
    rng = np.random.default_rng(20)
    n = 0
    for s in range(240):
        p = synth.random_tiny_problem(5000 + s)
        p.objective = ("sum", "max")[s % 2]
        if p.mode == "matrix" and p.slowdown_matrix is None:
            p.mode = "exclude_self"
        p.weights = [float(x) for x in rng.choice([0.25, 0.5, 1.0, 1.5, 2.0, 3.0, 0.1, 7.3], size=p.W)]
        try:
            a = brute.brute_force(p)
        except ValueError:
            continue
        b = oracle.solve(p)
        if a is None:
            assert b.status == "infeasible", s
            continue
        assert b.group_cols == a["sigmas"], s
        assert b.objective == pytest.approx(float(a["key"]), rel=1e-12), s
        if p.mode != "matrix":
            c = oracle.solve(p, "slice")
            assert (c.group_cols, c.key) == (b.group_cols, b.key), s
        u = synth.Problem(**{**p.__dict__, "weights": [2.5] * p.W})
        u0 = synth.Problem(**{**p.__dict__, "weights": None})
        ru, r0 = oracle.solve(u), oracle.solve(u0)
        assert (ru.status, ru.group_cols, ru.key) == (r0.status, r0.group_cols, r0.key), s
        assert ru.objective == pytest.approx(2.5 * r0.objective, rel=1e-12)
        n += 1
    assert n >= 150


def test_weighted_energy_rejected_unless_uniform():
    p = _ex1_weighted("energy", [2.0, 1.0])
    with pytest.raises(ValueError):
        oracle.solve(p)
    p.weights = [2.0, 2.0]
    p0 = _ex1_weighted("energy", None)
    assert oracle.solve(p).key == oracle.solve(p0).key


# ---------------------------------------------------------------- busy-SM energy integral (reading R21)
def test_busy_energy_hand_values():
    """Hand integral, N = 60, p_idle 75 W, p_max 225 W: worker 0 runs 30 SMs for 100 ns then 60 SMs
    for 50 ns; worker 1 runs 15 SMs for 120 ns.  [0,100): busy 45 -> 187.5 W x 100 = 18750;
    [100,120): 75 -> capped at 60 -> 225 x 20 = 4500; [120,150): 60 -> 225 x 30 = 6750; total 30000 W ns."""
    sm, lat = [[30, 60], [15]], [[100, 50], [120]]
    assert oracle.busy_energy_sweep(sm, lat, 60, 75.0, 225.0) == pytest.approx(30000.0, rel=1e-15)
    exact = brute.busy_energy(sm, [[Fraction(x) for x in r] for r in lat], 60, Fraction(75), Fraction(225))
    assert exact == 30000
    # S:417 "empty timeline of duration T -> p_idle T"; one kernel of 60 CUs, 10 us in a 1 ms window
    assert oracle.busy_energy_sweep([[60], [0]], [[10_000], [1_000_000]], 60, 75.0, 225.0) == pytest.approx(
        75.0 * 1e6 + 150.0 * 1e4, rel=1e-15)
    # S:418 additivity: splitting a group's interval leaves the integral unchanged
    assert oracle.busy_energy_sweep([[30, 30, 60], [15]], [[40, 60, 50], [120]], 60, 75.0, 225.0) == pytest.approx(
        30000.0, rel=1e-15)


def test_busy_energy_single_worker_closed_form_and_paper_example():
    """One worker with every size <= N: E = p_idle L + (p_max - p_idle) sum_g c_g e_g / N.  And App. B
    Ex2 (R=1, ExcludeSelf, SUM): A(60,15), B(15,60), every e = beta x 1.625, busy >= 75 > 60 throughout,
    so E = 225 W x 48.75 us = 10968.75 W us = power x makespan."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        G = int(rng.integers(1, 6))
        c = [int(x) for x in rng.choice([15, 30, 45, 60], size=G)]
        e = [float(x) for x in rng.uniform(1, 1000, size=G)]
        ref = 75.0 * sum(e) + 150.0 * sum(ci * ei for ci, ei in zip(c, e)) / 60
        assert oracle.busy_energy_sweep([c], [e], 60, 75.0, 225.0) == pytest.approx(ref, rel=1e-13)
    gold = json.load(open(GOLD))
    case = [c for c in gold["cases"] if c["name"].startswith("Ex2") and c["R"] == 1 and c["mode"] == "exclude_self"
            and c["objective"] == "sum"][0]
    b = oracle.solve(_golden_problem(case, gold))
    assert b.energy_busy_j == pytest.approx(10968.75e-6 * 1e-3 * 1000, rel=1e-12)   # W us -> J


def test_busy_energy_sweep_equals_exact_integral_random():
    """O-B's event loop (floats) == O-A's interval integral in Fractions on random plans, and
    E_busy <= power_max x makespan, >= p_idle x makespan."""
    rng = np.random.default_rng(9)
    for _ in range(200):
        W = int(rng.integers(1, 5))
        sm = [[int(x) for x in rng.choice([14, 28, 70, 140, 148], size=int(rng.integers(1, 6)))] for _ in range(W)]
        lat = [[int(x) for x in rng.integers(1, 10_000, size=len(r))] for r in sm]
        f = oracle.busy_energy_sweep(sm, [[float(x) for x in r] for r in lat], 148, 200.0, 1000.0)
        ex = brute.busy_energy(sm, [[Fraction(x) for x in r] for r in lat], 148, Fraction(200), Fraction(1000))
        assert f == pytest.approx(float(ex), rel=1e-12)
        mk = max(sum(r) for r in lat)
        assert 200.0 * mk * (1 - 1e-12) <= f <= 1000.0 * mk * (1 + 1e-12)
