"""GPU parity: the CUDA path (through the C-ABI) against the oracle, element by element.

Bar: allocation (group sizes, level ranks, candidate index, exact integer
key) bit-exact; FP64 values within 1e-5 relative (they agree to ~1e-12 by construction).
Small cases run the oracle live; BASELINE.json's full sizes compare with
tests/golden/oracle_full.json, written by tools/gen_oracle_golden.py from oracle/ only.
"""
import copy
import json
import os

import numpy as np
import pytest

import oracle
import synth
import paper_2506_12598_b200 as ec
from paper_2506_12598_b200 import parallel

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
REL = 1e-5


def _gold():
    return json.load(open(os.path.join(HERE, "golden", "oracle_full.json")))["records"]


def _same(g, o, label=""):
    assert g.status == o.status, label
    if o.status != "ok":
        return
    assert g.winner_levels == o.levels, label
    assert g.group_sm == o.group_sm, label
    assert g.winner_index == o.index, label
    assert g.exact_key == o.key, label
    assert g.model_switches == o.switches, label
    assert g.objective == pytest.approx(o.objective, rel=REL), label
    assert g.makespan_ns == pytest.approx(o.makespan_ns, rel=REL), label
    assert g.energy_j == pytest.approx(o.energy_j, rel=REL), label
    assert g.power_w == pytest.approx(o.power_w, rel=REL), label
    assert g.throughput_rps == pytest.approx(o.throughput_rps, rel=REL), label
    eb = getattr(o, "energy_busy_j", float("nan"))
    if eb == eb:   # the busy-SM energy integral of the predicted run (R21)
        assert g.energy_busy_j == pytest.approx(eb, rel=REL), label
    for a, b in zip(g.model_latency_ns, o.latency_ns):
        assert a == pytest.approx(b, rel=REL), label
    for ga, gb in zip(g.group_latency_ns, o.group_latency_ns):
        for a, b in zip(ga, gb):
            assert a == pytest.approx(b, rel=REL), label


def _gpu(p, engine="auto", **kw):
    return ec.plan_problem(ec.Profiles.from_models(p.models), p, engine=engine, **kw)


# ---------------------------------------------------------------- worked examples
def test_worked_examples_on_gpu():
    from test_oracle import _golden_problem
    gold = json.load(open(os.path.join(HERE, "golden", "appB_examples.json")))
    for case in gold["cases"]:
        p = _golden_problem(case, gold)
        for engine in ("enum", "slice"):
            g = _gpu(p, engine)
            assert g.group_sm == case["expect_sizes"], (case["name"], engine)
            assert g.objective == pytest.approx(case["expect_J"] * 1000, rel=1e-12)
            assert g.makespan_ns == pytest.approx(case["expect_makespan_us"] * 1000, rel=1e-12)
            assert g.power_w == pytest.approx(case["expect_power_w"], rel=1e-12)
            assert g.energy_j == pytest.approx(case["expect_energy_j"], rel=1e-12)
            assert g.throughput_rps == pytest.approx(case["expect_throughput_rps"], rel=1e-12)


# ---------------------------------------------------------------- K1 level tables, whole tables
def _k1_vs_oracle(pr, models, m, R, gb=None, mask=0, label=""):
    sizes = models[m].sizes
    S, B, wit = ec.level_table(pr, m, switch_max=R, group_bounds=gb, allowed_mask=mask)
    beta, n = oracle.group_tables(models[m].exec_ns, gb)
    So, Bo, Wo = oracle.levels(beta, n, sizes, mask or (1 << len(sizes)) - 1, R)
    assert np.array_equal(S, So), f"{label}: S"
    assert np.array_equal(B, Bo), f"{label}: B*"
    assert np.array_equal(wit, Wo), f"{label}: witnesses / rank order"
    return len(S)


def test_k1_level_tables_vs_oracle():
    """K1 (the GPU's level-1 DP, suffix recurrence) == O-B's memoised forward recursion, table by
    table: every attained CU-sum S, B*(S), the canonical witness and the rank order (SURVEY §8(c)
    c6b).  Random shapes (groups of several kernels, masks, irregular sizes, R sweeps),
    the C5 library at R = 14 and two C4 models (577 levels, 64 groups)."""
    rng = np.random.default_rng(17)
    for t in range(60):
        G = int(rng.integers(1, 10))
        Cn = int(rng.integers(2, 9))
        sizes = synth.lattice_sizes(Cn, 148) if t % 3 else sorted(int(x) for x in rng.choice(np.arange(1, 60), Cn, replace=False))
        K = G + int(rng.integers(0, 4))
        mdl = synth.synthesize_model("k", ["uniform", "vgg", "bert", "shufflenet"][t % 4], K, sizes, 4000 + t)
        pr = ec.Profiles.from_models([mdl])
        gb = None
        if K > G:
            cut = sorted(int(x) for x in rng.choice(np.arange(1, K), size=G - 1, replace=False)) if G > 1 else []
            gb = [0] + cut + [K]
        mask = int(rng.integers(1, 1 << Cn)) if t % 2 else 0
        R = int(rng.integers(0, 6))
        _k1_vs_oracle(pr, [mdl], 0, R, gb, mask, f"random {t}")
    models, _, _ = synth.make_c5(1)
    pr = ec.Profiles.from_models(models)
    for m in range(len(models)):
        for R in (0, 3, 14):
            _k1_vs_oracle(pr, models, m, R, label=f"C5 library {m} R={R}")
    c4 = synth.make_c4()
    pr4 = ec.Profiles.from_models(c4.models)
    for m in (0, 1):
        assert _k1_vs_oracle(pr4, c4.models, m, 14, label=f"C4 model {m}") == 577


# ---------------------------------------------------------------- random tiny instances
@pytest.mark.parametrize("chunk", range(4))
def test_random_instances_vs_oracle(chunk):
    for s in range(chunk * 100, chunk * 100 + 100):
        p = synth.random_tiny_problem(s, max_w=4, max_g=4, max_c=4)
        o = oracle.solve(p)
        _same(_gpu(p, "enum"), o, f"enum seed {s}")
        if p.mode != "matrix":
            _same(_gpu(p, "slice"), o, f"slice seed {s}")


def test_c1_sweep():
    """C1: 2 x 3 groups x {15,30,45,60}; R in {0,1,2}; every mode x objective; QoS on/off."""
    for R in (0, 1, 2):
        for mode in ("exclude_self", "paper", "excess", "matrix"):
            for obj in ("sum", "max", "energy"):
                for qos in (False, True):
                    p = synth.make_c1(R, mode, obj, qos)
                    o = oracle.solve(p)
                    _same(_gpu(p, "enum"), o, f"C1 {R} {mode} {obj} {qos}")
                    if mode != "matrix":
                        _same(_gpu(p, "slice"), o, f"C1 slice {R} {mode} {obj} {qos}")


def test_c2_all_modes_objectives():
    for mode in ("exclude_self", "paper", "excess", "matrix"):
        for obj in ("sum", "max", "energy"):
            p = synth.make_c2(mode, obj)
            o = oracle.solve(p)
            _same(_gpu(p, "enum"), o, f"C2 {mode} {obj}")
            if mode != "matrix":
                _same(_gpu(p, "slice"), o, f"C2 slice {mode} {obj}")


# ---------------------------------------------------------------- edge cases
def test_edge_single_worker_and_tiny_levels():
    p = synth.make_c1(R=0)
    p.model_ids = [1]
    _same(_gpu(p, "enum"), oracle.solve(p), "W=1")
    _same(_gpu(p, "slice"), oracle.solve(p), "W=1 slice")
    # fewer inner levels than a thread holds (L < KIN) and a 1-level worker
    p = synth.make_c1(R=0)
    p.allowed_mask = [0b0001, 0b0110]
    _same(_gpu(p, "enum"), oracle.solve(p), "masks")


def test_edge_all_infeasible_qos():
    p = synth.make_c2()
    p.qos_ns = [1.0, 1.0, 1.0]
    assert oracle.solve(p).status == "infeasible"
    for engine in ("enum", "slice"):
        assert _gpu(p, engine).status == "infeasible"


def test_edge_exact_ties_lowest_index():
    """duplicated models (P:378 Mix 1 = 2x albert) create exact ties; lowest index wins."""
    p = synth.make_c2()
    p.model_ids = [0, 0, 1]
    o = oracle.solve(p)
    for engine in ("enum", "slice"):
        _same(_gpu(p, engine), o, engine)
    for tol in (0.0, 1e-3):
        o = oracle.solve(p, tol=tol)
        _same(_gpu(p, "enum", tie_tol=tol), o, f"tol {tol}")


def test_edge_groups_and_large_levels():
    """kernel groups (c3-K) and a worker with many levels (two C4 models, ENUM)"""
    p = synth.make_c2()
    p.group_bounds = [[0, 3, 8], None, [0, 1, 2, 4, 8]]
    _same(_gpu(p, "enum"), oracle.solve(p), "groups")
    _same(_gpu(p, "slice"), oracle.solve(p), "groups slice")
    q = synth.make_c4()
    q.model_ids = [0, 1]
    q.qos_ns = q.qos_ns[:2]
    o = oracle.solve(q, "slice")
    _same(_gpu(q, "enum"), o, "C4x2 enum")
    _same(_gpu(q, "slice"), o, "C4x2 slice")


# ---------------------------------------------------------------- full sizes (golden)
def _check_gold(g, rec, label):
    assert rec["status"] == g.status, label
    assert g.winner_levels == rec["levels"], label
    assert g.group_sm == rec["group_sm"], label
    assert g.winner_index == rec["index"], label
    assert g.exact_key == int(rec["key"]), label
    assert g.objective == pytest.approx(rec["objective"], rel=REL)
    assert g.energy_j == pytest.approx(rec["energy_j"], rel=REL)
    assert g.makespan_ns == pytest.approx(rec["makespan_ns"], rel=REL)


def test_c3_full_matrix_vs_golden():
    rec = _gold()["C3"]
    p = synth.make_c3("matrix")
    assert synth.problem_hash(p) == rec["hash"], "golden file is stale: rerun tools/gen_oracle_golden.py"
    g = _gpu(p, "enum")
    assert g.candidates == 113 ** 4 and g.units_scored == 113 ** 4
    _check_gold(g, rec, "C3")


def test_c3_excl_enum_equals_slice_equals_golden():
    rec = _gold()["C3_excl"]
    p = synth.make_c3("exclude_self")
    assert synth.problem_hash(p) == rec["hash"]
    a, b = _gpu(p, "enum"), _gpu(p, "slice")
    _check_gold(a, rec, "C3 excl enum")
    _check_gold(b, rec, "C3 excl slice")


def test_c4_full_slice_vs_golden():
    rec = _gold()["C4"]
    p = synth.make_c4()
    assert synth.problem_hash(p) == rec["hash"]
    g = _gpu(p)  # AUTO must pick SLICE (1.2e22 tuples)
    assert g.engine == "slice"
    _check_gold(g, rec, "C4")


def test_s6_full_vs_golden():
    rec = _gold()["S6"]
    p = synth.make_s6()
    assert synth.problem_hash(p) == rec["hash"]
    _check_gold(_gpu(p, "slice"), rec, "S6 slice")


@pytest.mark.parametrize("seed", [0, 1, 7])
def test_c5_batch_every_mix_vs_oracle_golden(seed):
    """the bench configuration: 4096 mixes in one launch sequence, EVERY mix against the oracle's
    stored answer (tests/golden/c5_mixes.json: all 7^4 distinct mixes); seeds 0..7 are the
    batches bench.py plans on ranks 0..7"""
    import golden_c5
    models, ids, qos = synth.make_c5(4096, seed=seed)
    pr = ec.Profiles.from_models(models)
    out = ec.plan_batch(pr, ids, total_sms=148, switch_max=14, qos_ns=qos, p_idle_w=200.0, p_max_w=1000.0, gmax=16)
    assert golden_c5.check_batch(ids, out, sizes=models[0].sizes) == 4096
    # every mix: QoS met, budget met
    ok = out["status"] == 0
    assert ok.sum() > 0
    assert np.all(out["model_switches"][ok] <= 14)
    assert np.all(out["model_latency_ns"][ok] <= qos[ok] * (1 + 1e-12))
    if seed == 0:   # the older per-record golden (oracle_full.json) agrees too
        gold = _gold()
        for i in (0, 1, 2047, 4095):
            rec = gold[f"C5_{i}"]
            assert synth.problem_hash(synth.c5_problem(i, models, ids, qos)) == rec["hash"]
            if rec["status"] == "ok":
                assert int(out["winner_index"][i]) == rec["index"]


def test_c5_small_batch_each_mix_vs_oracle():
    models, ids, qos = synth.make_c5(24, seed=3)
    pr = ec.Profiles.from_models(models)
    out = ec.plan_batch(pr, ids, total_sms=148, switch_max=14, qos_ns=qos, p_idle_w=200.0, p_max_w=1000.0, gmax=16)
    for i in range(24):
        o = oracle.solve(synth.c5_problem(i, models, ids, qos), "slice")
        assert (out["status"][i] == 0) == (o.status == "ok")
        if o.status == "ok":
            assert out["winner_levels"][i].tolist() == o.levels
            assert int(out["winner_index"][i]) == o.index


def test_batch_device_path_equals_host_path():
    import torch
    models, ids, qos = synth.make_c5(64, seed=7)
    pr = ec.Profiles.from_models(models)
    host = ec.plan_batch(pr, ids, total_sms=148, qos_ns=qos, p_idle_w=200.0, p_max_w=1000.0)
    d_ids = torch.from_numpy(ids).cuda()
    d_q = torch.from_numpy(qos).cuda()
    dev = ec.plan_batch(pr, d_ids, total_sms=148, qos_ns=d_q, p_idle_w=200.0, p_max_w=1000.0)
    torch.cuda.synchronize()
    assert np.array_equal(dev["winner_index"].cpu().numpy().view(np.uint64), host["winner_index"])
    assert np.array_equal(dev["status"].cpu().numpy(), host["status"])
    assert np.allclose(dev["objective"].cpu().numpy(), host["objective"], rtol=0, atol=0)


# ---------------------------------------------------------------- sharding
class _NumpyComm:
    """combines the per-shard values in-process (the reductions of parallel.TorchComm)"""

    def __init__(self, sessions):
        self.s = sessions


def _run_shards(make, n_shards):
    ss = [make(k) for k in range(n_shards)]
    m = np.minimum.reduce([s.pass1() for s in ss])
    k = parallel.lexmin_u256(np.stack([s.pass2_min(m) for s in ss]))
    f = parallel.lexmin_u256(np.stack([s.pass2_first(k) for s in ss]))
    return [s.finish(f) for s in ss]


@pytest.mark.parametrize("n_shards", [2, 3, 8])
def test_sharded_single_problem_vs_oracle(n_shards):
    """every shard materialises the oracle's plan (live oracle for C2, stored answers at full size)"""
    gold = _gold()
    cases = [(synth.make_c2(), "enum", oracle.solve(synth.make_c2())),
             (synth.make_c2("paper", "energy"), "slice", oracle.solve(synth.make_c2("paper", "energy"))),
             (synth.make_c3("matrix"), "enum", gold["C3"]), (synth.make_c4(), "slice", gold["C4"])]
    for p, eng, o in cases:
        pr = ec.Profiles.from_models(p.models)
        outs = _run_shards(lambda k: ec.Session(pr, problem=p, shard=k, n_shards=n_shards, engine=eng), n_shards)
        for g in outs:
            if isinstance(o, dict):
                _check_gold(g, o, f"{p.name} {eng} x{n_shards}")
            else:
                _same(g, o, f"{p.name} {eng} x{n_shards}")


def test_sharded_batch_vs_oracle():
    import golden_c5
    models, ids, qos = synth.make_c5(64, seed=11)
    pr = ec.Profiles.from_models(models)
    b = dict(model_ids=ids, qos_ns=qos, total_sms=148, p_idle_w=200.0, p_max_w=1000.0)
    outs = _run_shards(lambda k: ec.Session(pr, batch=b, shard=k, n_shards=3), 3)
    for o in outs:
        assert golden_c5.check_batch(ids, o) == 64


# ---------------------------------------------------------------- more shapes
def _many_workers_problem(W, seed, mode="exclude_self", objective="sum", qos=True, R=1):
    sizes = synth.lattice_sizes(3, 60)
    models = [synth.synthesize_model(f"m{i}", "uniform", 2, sizes, 900 + 17 * seed + i) for i in range(3)]
    rng = np.random.default_rng(seed)
    ids = [int(x) for x in rng.integers(0, 3, size=W)]
    q = synth.qos_3x(models, ids, factor=float(W) * 0.9) if qos else None
    M = None
    if mode == "matrix":
        M = rng.uniform(0.5, 1.5, size=(W, W)).astype(np.float32)
        np.fill_diagonal(M, 0.0)
    return synth.Problem(f"W{W}", models, ids, 60, R, mode, objective, qos_ns=q, slowdown_matrix=M)


@pytest.mark.parametrize("W", [5, 6, 7, 8])
def test_many_workers_fast_and_generic_kernels(W):
    """the W-templated pass-1 kernels (W = 5..8) on small level tables, every mode / objective"""
    for seed in range(3):
        for mode in ("exclude_self", "paper", "excess", "matrix"):
            for obj in ("sum", "max", "energy"):
                for qos in (False, True):
                    p = _many_workers_problem(W, seed, mode, obj, qos)
                    o = oracle.solve(p)
                    _same(_gpu(p, "enum"), o, f"W{W} {seed} {mode} {obj} {qos}")


def test_matrix_with_qos_full_size_sampled():
    """MATRIX + QoS (maybe/surely-feasible filter) on C3 shapes, oracle live"""
    p = synth.make_c3("matrix")
    p.qos_ns = synth.qos_3x(p.models, p.model_ids, factor=3.5)   # binding (the optimum changes vs no QoS)
    o = oracle.solve(p)
    assert o.status == "ok"
    _same(_gpu(p, "enum"), o, "C3 matrix qos")


def test_batch_paper_mode_and_masks():
    """batched path with PAPER_AS_WRITTEN (fast kernel's D_i term) and per-model masks"""
    models, ids, qos = synth.make_c5(12, seed=21)
    pr = ec.Profiles.from_models(models)
    masks = [0xFF, 0xFE, 0x7F, 0xFF, 0x3C, 0xFF, 0xF0]
    out = ec.plan_batch(pr, ids, total_sms=148, slowdown="paper", qos_ns=qos * 2.0, allowed_mask=masks,
                        p_idle_w=200.0, p_max_w=1000.0, gmax=16)
    for i in range(12):
        p = synth.c5_problem(i, models, ids, qos * 2.0)
        p.mode = "paper"
        p.allowed_mask = [masks[m] for m in ids[i]]
        o = oracle.solve(p, "slice")
        assert (int(out["status"][i]) == 0) == (o.status == "ok"), i
        if o.status == "ok":
            assert out["winner_levels"][i].tolist() == o.levels, i
            assert out["objective"][i] == pytest.approx(o.objective, rel=REL)


# ---------------------------------------------------------------- row-bound pruning
@pytest.mark.parametrize("mode,qf", [("exclude_self", 1.0), ("exclude_self", None), ("paper", 2.0)])
def test_pruned_equals_exhaustive_batch(mode, qf):
    """pruning is exact: the same winners, keys and values as classifying every candidate"""
    models, ids, qos = synth.make_c5(256, seed=31)
    pr = ec.Profiles.from_models(models)
    kw = dict(total_sms=148, slowdown=mode, qos_ns=None if qf is None else qos * qf, p_idle_w=200.0,
              p_max_w=1000.0, gmax=16)
    a = ec.plan_batch(pr, ids, prune=True, **kw)
    b = ec.plan_batch(pr, ids, prune=False, **kw)
    for k in ("status", "winner_index", "winner_levels", "objective", "group_sm", "model_latency_ns"):
        assert np.array_equal(a[k], b[k]), k
    # and the pruned pass 1 really skipped rows
    batch = dict(model_ids=ids, total_sms=148, slowdown=mode, p_idle_w=200.0, p_max_w=1000.0)
    if qf is not None:
        batch["qos_ns"] = qos * qf
    s = ec.Session(pr, batch=batch, engine="enum")
    s.pass1()
    rows = sum(int(np.prod([pr_levels(pr, m) for m in row[:2]])) for row in ids)
    done = s.stats()["units_processed"]
    s.close()
    assert 0 < done < rows


@pytest.mark.parametrize("W,qf,seed", [(3, 0.8, 51), (4, 0.7, 52), (4, 1.3, 53), (5, 1.0, 54), (4, 2.5, 55)])
def test_pruned_equals_exhaustive_stress(W, qf, seed):
    """the row / chunk / entry bounds (hull-restricted) and the incumbent re-check are exact across
    worker counts and QoS tightness (partially feasible rows, non-monotone QoS ranges, empty ranges)"""
    models, ids, qos = synth.make_c5(192, seed=seed, W=W)
    pr = ec.Profiles.from_models(models)
    kw = dict(total_sms=148, qos_ns=qos * qf, p_idle_w=200.0, p_max_w=1000.0, gmax=16)
    a = ec.plan_batch(pr, ids, prune=True, **kw)
    b = ec.plan_batch(pr, ids, prune=False, **kw)
    for k in ("status", "winner_index", "winner_levels", "objective", "group_sm", "model_latency_ns"):
        assert np.array_equal(a[k], b[k]), k


def pr_levels(pr, m, _cache={}):
    key = (id(pr), m)
    if key not in _cache:
        _cache[key] = ec.plan(pr, [m], total_sms=148, switch_max=14).candidates
    return _cache[key]


def test_pruned_sampled_mixes_vs_oracle_without_qos():
    """no QoS: pruning is the only thing that skips work; sampled mixes vs the oracle"""
    models, ids, _ = synth.make_c5(32, seed=41)
    pr = ec.Profiles.from_models(models)
    out = ec.plan_batch(pr, ids, total_sms=148, p_idle_w=200.0, p_max_w=1000.0, gmax=16)
    for i in range(0, 32, 4):
        p = synth.c5_problem(i, models, ids, np.full_like(ids, np.inf, dtype=np.float64))
        p.qos_ns = None
        o = oracle.solve(p, "slice")
        assert o.status == "ok" and int(out["status"][i]) == 0
        assert out["winner_levels"][i].tolist() == o.levels, i
        assert int(out["winner_index"][i]) == o.index, i


@pytest.mark.gpu
def test_overflow_fallbacks_with_tiny_list_capacities():
    """The fallbacks behind the pruned pass 1's fixed-capacity lists: with a processed-unit list and a
    pass-2 band list of capacity 1 (a test build, -DPL_CAP_N=1 -DBAND_CAP_N=1), k_reduce_min and pass 2
    scan every unit and see only the units pass 1 wrote (written-unit bitmap, the rest read +inf).
    Selected parity tests rerun against that build in a subprocess (the library is loaded once per
    process)."""
    import os
    import subprocess
    import sys
    from paper_2506_12598_b200 import build as bld
    lib = os.path.join(os.path.dirname(bld.__file__), "libeclip_tinycap.so")
    if not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(bld.LIB):
        bld.build_variant("tinycap", ["PL_CAP_N=1", "BAND_CAP_N=1"])
    env = dict(os.environ, ECLIP_LIB=lib)
    sel = "pruned_equals_exhaustive or exact_ties or c5_small_batch or c5_batch_every or sharded"
    r = subprocess.run([sys.executable, "-m", "pytest", __file__, "-q", "-m", "gpu", "-k", sel, "-p", "no:cacheprovider"],
                       env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


# ---------------------------------------------------------------- persistent planner
def test_planner_every_mix_vs_oracle_golden_host_and_device():
    """eclip_planner_*: level tables built once, then batch after batch (different sizes, host and
    device buffers, several seeds) — every mix against the oracle's stored answers, and equal to
    the one-shot eclip_plan_batch"""
    import torch
    import golden_c5
    models, _, _ = synth.make_c5(1)
    pr = ec.Profiles.from_models(models)
    pl = ec.Planner(pr, n_models=4, max_problems=4096, total_sms=148, p_idle_w=200.0, p_max_w=1000.0, timing=True)
    for seed, n in ((0, 4096), (1, 1000), (2, 1), (3, 4096), (4, 4096)):
        _, ids, qos = synth.make_c5(n, seed=seed)
        if seed % 2:
            out = pl.plan(ids, qos, gmax=16)
            got = out
        else:
            d_out = ec.alloc_batch_out(n, 4, 16, device="cuda")
            pl.plan(torch.from_numpy(ids).cuda(), torch.from_numpy(qos).cuda(), out=d_out)
            torch.cuda.synchronize()
            got = d_out
        assert golden_c5.check_batch(ids, got, sizes=models[0].sizes) == n
        ph = pl.phase_ms()
        assert all(v >= 0.0 for v in ph.values()) and ph["pass1"] > 0.0
        if seed == 3:
            ref = ec.plan_batch(pr, ids, total_sms=148, qos_ns=qos, p_idle_w=200.0, p_max_w=1000.0, gmax=16)
            for k in ("status", "winner_index", "winner_levels", "objective", "group_sm", "model_latency_ns", "power_w"):
                assert np.array_equal(np.asarray(got[k]), np.asarray(ref[k])), k
    with pytest.raises(ec.EclipError):
        pl.plan(np.zeros((4097, 4), np.int32), np.ones((4097, 4)))        # more mixes than max_problems
    with pytest.raises(ec.EclipError):
        pl.plan(np.zeros((4, 4), np.int32), None)                         # the planner has QoS
    pl.close()


def test_planner_pinned_outputs_written_by_the_kernel():
    """Host batches whose output arrays are all page-locked: k_materialize writes them directly (mapped
    memory, no staging copies); every mix against the oracle's stored answers and equal, field by field, to
    the same batch planned into unpinned host arrays (staging + copies) and into device arrays"""
    import torch
    import golden_c5
    models, ids, qos = synth.make_c5(1000, seed=5)
    pr = ec.Profiles.from_models(models)
    pl = ec.Planner(pr, n_models=4, max_problems=1000, total_sms=148, p_idle_w=200.0, p_max_w=1000.0)
    pinned = ec.alloc_batch_out(1000, 4, 16, pinned=True)
    plain = ec.alloc_batch_out(1000, 4, 16)
    dev = ec.alloc_batch_out(1000, 4, 16, device="cuda")
    for _ in range(2):   # (the second call reuses the planner's buffers)
        pl.plan(torch.from_numpy(ids).pin_memory().numpy(), torch.from_numpy(qos).pin_memory().numpy(), out=pinned)
        pl.plan(ids, qos, out=plain)
        pl.plan(torch.from_numpy(ids).cuda(), torch.from_numpy(qos).cuda(), out=dev)
        torch.cuda.synchronize()
        assert golden_c5.check_batch(ids, pinned, sizes=models[0].sizes) == 1000
        for k, v in pinned.items():
            if k.startswith("_"):
                continue
            assert np.array_equal(np.asarray(v), np.asarray(plain[k])), k
            assert np.array_equal(np.asarray(v), dev[k].cpu().numpy().view(np.asarray(v).dtype)), k
    pl.close()


def test_planner_other_settings_vs_oracle():
    """planners without QoS, in PAPER mode with masks, and MATRIX (generic kernels) against the oracle"""
    masks = [0xFF, 0xFE, 0x7F, 0xFF, 0x3C, 0xFF, 0xF0]
    rng = np.random.default_rng(3)
    for mode, use_q, mk in (("exclude_self", False, None), ("paper", True, masks), ("matrix", True, None)):
        W = 3 if mode == "matrix" else 4       # the oracle enumerates MATRIX problems: keep them at 1.4e6 tuples
        models, ids, qos = synth.make_c5(12, seed=23, W=W)
        pr = ec.Profiles.from_models(models)
        M = rng.uniform(0.5, 1.5, size=(12, W, W)).astype(np.float32)
        pl = ec.Planner(pr, n_models=W, max_problems=16, total_sms=148, slowdown=mode, qos=use_q, allowed_mask=mk,
                        p_idle_w=200.0, p_max_w=1000.0)
        q = qos * 1.5 if use_q else None
        for rep in range(2):
            out = pl.plan(ids, q, slowdown_matrix=M if mode == "matrix" else None, gmax=16)
            for i in range(0, 12, 3):
                p = synth.c5_problem(i, models, ids, qos * 1.5)
                p.mode = mode
                if not use_q:
                    p.qos_ns = None
                if mk is not None:
                    p.allowed_mask = [mk[m] for m in ids[i]]
                if mode == "matrix":
                    p.slowdown_matrix = M[i].copy()
                    np.fill_diagonal(p.slowdown_matrix, 0.0)
                o = oracle.solve(p, "enum" if mode == "matrix" else "slice")
                assert (int(out["status"][i]) == 0) == (o.status == "ok"), (mode, i)
                if o.status == "ok":
                    assert out["winner_levels"][i].tolist() == o.levels, (mode, i)
                    assert out["objective"][i] == pytest.approx(o.objective, rel=REL)
        pl.close()


# ---------------------------------------------------------------- heterogeneous kernel counts (wide)
def _hetero_problem(Ks, C, R, mode="exclude_self", objective="sum", qos=None, seed=0, fams=None):
    sizes = synth.lattice_sizes(C, 148)
    fams = fams or ["resnet", "bert", "vgg", "densenet", "shufflenet"]
    models = [synth.synthesize_model(f"k{K}", fams[i % len(fams)], K, sizes, 7000 + 31 * seed + i)
              for i, K in enumerate(Ks)]
    ids = list(range(len(Ks)))
    q = synth.qos_3x(models, ids, factor=qos) if qos else None
    return synth.Problem(f"hetero{Ks}", models, ids, 148, R, mode, objective, qos_ns=q,
                         p_idle_w=200.0, p_max_w=1000.0)


def test_heterogeneous_kernel_counts_vs_oracle():
    """PAPER.md P:299 decides per kernel and P:313 divides each worker's CU sum by its own kernel
    count; co-located models have different, often co-prime, kernel counts, so
    Lambda = lcm K_w and Lambda N (W+1) exceed 2^24: the wide launch."""
    cases = [((200, 199, 97), 2, 14, "exclude_self", "sum", 3.0),
             ((200, 199, 97), 2, 14, "exclude_self", "sum", None),
             ((200, 199, 97), 2, 3, "paper", "sum", 6.0),
             ((131, 64, 97), 3, 2, "exclude_self", "max", 3.0),
             ((131, 64, 97), 3, 2, "excess", "energy", None),
             ((61, 53, 47, 43), 2, 1, "exclude_self", "sum", 3.5),
             ((61, 53, 47, 43), 2, 1, "paper", "energy", 8.0)]
    for Ks, C, R, mode, obj, q in cases:
        p = _hetero_problem(Ks, C, R, mode, obj, q)
        o = oracle.solve(p, "enum")
        g = _gpu(p, "enum")
        _same(g, o, f"{Ks} C={C} R={R} {mode} {obj} q={q}")
        g = _gpu(p)   # AUTO: ENUM (SLICE does not apply to these T' ranges)
        assert g.engine == "enum"
        _same(g, o, f"auto {Ks}")
    with pytest.raises(ec.EclipError) as e:
        _gpu(_hetero_problem((200, 199, 97), 2, 14), "slice")
    assert e.value.code == ec.eclip.E_TOO_LARGE


def test_heterogeneous_batch_and_lcm_boundary():
    """a batch over a library with co-prime kernel counts (wide batch) vs the oracle; the exact-range
    boundary: Lambda = lcm K_w <= 2^40 plans (4 workers, K ~ 1010), 2^40 < Lambda returns E_TOO_LARGE"""
    sizes = synth.lattice_sizes(2, 148)
    Ks = (101, 103, 64, 27, 50)
    models = [synth.synthesize_model(f"b{K}", "resnet", K, sizes, 7300 + K) for K in Ks]
    pr = ec.Profiles.from_models(models)
    rng = np.random.default_rng(9)
    ids = rng.integers(0, len(Ks), size=(10, 3)).astype(np.int32)
    solo = np.array([synth.qos_3x(models, [m])[0] for m in range(len(Ks))])
    out = ec.plan_batch(pr, ids, total_sms=148, switch_max=4, qos_ns=solo[ids], p_idle_w=200.0, p_max_w=1000.0,
                        gmax=128)
    for i in range(10):
        p = synth.Problem("b", models, [int(x) for x in ids[i]], 148, 4, qos_ns=[float(x) for x in solo[ids[i]]],
                          p_idle_w=200.0, p_max_w=1000.0)
        o = oracle.solve(p, "enum")
        assert (int(out["status"][i]) == 0) == (o.status == "ok"), i
        if o.status == "ok":
            assert out["winner_levels"][i].tolist() == o.levels, i
            assert int(out["winner_index"][i]) == o.index, i
            assert out["objective"][i] == pytest.approx(o.objective, rel=REL)
    # Lambda = 1009 * 1013 * 1019 * 1021 = 1.06e12 <= 2^40: plans (R = 0: one level per size)
    big = [synth.synthesize_model(f"p{K}", "uniform", K, sizes, 7400 + K) for K in (1009, 1013, 1019, 1021, 1031)]
    p = synth.Problem("lcm", big, [0, 1, 2, 3], 148, 0, p_idle_w=200.0, p_max_w=1000.0)
    _same(_gpu(p, "enum"), oracle.solve(p, "enum"), "lcm 1.06e12")
    p.model_ids = [0, 1, 2, 3, 4]         # Lambda = 1.1e15 > 2^40
    with pytest.raises(ec.EclipError) as e:
        _gpu(p, "enum")
    assert e.value.code == ec.eclip.E_TOO_LARGE


# ---------------------------------------------------------------- in-library multi-GPU exchange
def _threads(fn, n):
    import threading
    res, errs = [None] * n, []

    def run(r):
        try:
            res[r] = fn(r)
        except Exception as e:   # noqa: BLE001
            errs.append(e)
    ts = [threading.Thread(target=run, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errs, errs
    return res


def test_comm_nccl_world_one_vs_oracle():
    """eclip_comm over NCCL at world size 1 (one B200): the in-library sharded path (device-side
    exchanges) gives the oracle's plans for ENUM and SLICE problems and a batch"""
    import golden_c5
    c = ec.Comm.create(ec.Comm.unique_id(), 1, 0, 0)
    assert c.info() == dict(rank=0, size=1, device=0)
    gold = _gold()
    p = synth.make_c2()
    pr = ec.Profiles.from_models(p.models)
    _same(ec.plan_problem(pr, p, engine="enum", comm=c), oracle.solve(p), "C2 nccl enum")
    _same(ec.plan_problem(pr, p, engine="slice", comm=c), oracle.solve(p), "C2 nccl slice")
    p4 = synth.make_c4()
    _check_gold(ec.plan_problem(ec.Profiles.from_models(p4.models), p4, comm=c), gold["C4"], "C4 nccl")
    models, ids, qos = synth.make_c5(256, seed=2)
    out = ec.plan_batch(ec.Profiles.from_models(models), ids, total_sms=148, qos_ns=qos, p_idle_w=200.0,
                        p_max_w=1000.0, comm=c, gmax=16)
    assert golden_c5.check_batch(ids, out, sizes=models[0].sizes) == 256
    c.close()


@pytest.mark.parametrize("n_ranks", [2, 3])
def test_comm_local_group_sharded_vs_oracle(n_ranks):
    """the sharded protocol with the exchanges inside the library: n ranks on one GPU (a local group
    of communicators, one host thread per rank), each planning its shard; every rank returns the
    oracle's plan (ENUM, SLICE, MATRIX+QoS with its surely-feasible minimum, a wide problem, a batch)"""
    import golden_c5
    gold = _gold()
    pc3 = synth.make_c3("matrix")
    pc3.qos_ns = synth.qos_3x(pc3.models, pc3.model_ids, factor=3.5)
    cases = [(synth.make_c2(), "enum", oracle.solve(synth.make_c2())),
             (synth.make_c2("excess", "max"), "slice", oracle.solve(synth.make_c2("excess", "max"))),
             (pc3, "enum", oracle.solve(pc3)),
             (synth.make_c4(), "slice", gold["C4"]),
             (_hetero_problem((200, 199, 97), 2, 14, qos=3.0), "enum", None)]
    for p, eng, o in cases:
        if o is None:
            o = oracle.solve(p, "enum")
        pr = ec.Profiles.from_models(p.models)
        comms = ec.Comm.local_group(n_ranks, 0)
        outs = _threads(lambda r: ec.plan_problem(pr, p, engine=eng, comm=comms[r]), n_ranks)
        for g in outs:
            if isinstance(o, dict):
                _check_gold(g, o, f"{p.name} local x{n_ranks}")
            else:
                _same(g, o, f"{p.name} {eng} local x{n_ranks}")
        for c in comms:
            c.close()
    models, ids, qos = synth.make_c5(128, seed=5)
    pr = ec.Profiles.from_models(models)
    comms = ec.Comm.local_group(n_ranks, 0)
    outs = _threads(lambda r: ec.plan_batch(pr, ids, total_sms=148, qos_ns=qos, p_idle_w=200.0, p_max_w=1000.0,
                                            comm=comms[r], gmax=16), n_ranks)
    for out in outs:
        assert golden_c5.check_batch(ids, out, sizes=models[0].sizes) == 128


# ---------------------------------------------------------------- per-worker weights (R20)
def _weighted(p, rng):
    p.weights = [float(x) for x in rng.choice([0.25, 0.5, 1.0, 1.5, 2.0, 3.0, 0.1, 7.3], size=p.W)]
    return p


def test_weighted_worked_example_on_gpu():
    from test_oracle import _ex1_weighted
    for obj, sizes in (("sum", [[60], [45]]), ("max", [[60], [30]])):
        p = _ex1_weighted(obj, [3.0, 1.0])
        o = oracle.solve(p)
        assert o.group_sm == sizes
        for engine in ("enum", "slice"):
            _same(_gpu(p, engine), o, f"{obj} {engine}")


def test_weighted_random_instances_vs_oracle():
    rng = np.random.default_rng(77)
    n = 0
    for s in range(300):
        p = _weighted(synth.random_tiny_problem(9000 + s, max_w=4, max_g=4, max_c=4), rng)
        if p.objective == "energy":
            p.objective = ("sum", "max")[s % 2]
        o = oracle.solve(p)
        _same(_gpu(p, "enum"), o, f"enum seed {s}")
        if p.mode != "matrix":
            _same(_gpu(p, "slice"), o, f"slice seed {s}")
        n += o.status == "ok"
    assert n > 150


def test_weighted_c2_c3_and_qos():
    rng = np.random.default_rng(5)
    for mode in ("exclude_self", "paper", "excess", "matrix"):
        for obj in ("sum", "max"):
            p = _weighted(synth.make_c2(mode, obj), rng)
            o = oracle.solve(p)
            _same(_gpu(p, "enum"), o, f"C2 {mode} {obj}")
            if mode != "matrix":
                _same(_gpu(p, "slice"), o, f"C2 slice {mode} {obj}")
    for qf in (None, 3.0):   # C1 with QoS bounds, weighted
        for mode in ("exclude_self", "paper", "excess"):
            p = _weighted(synth.make_c1(2, mode, "sum", qos=qf is not None), rng)
            o = oracle.solve(p)
            _same(_gpu(p, "enum"), o, f"C1 {mode}")
            _same(_gpu(p, "slice"), o, f"C1 slice {mode}")
    # a full-size weighted problem (C3 profiles, EXCLUDE_SELF, 1.6e8 candidates): ENUM == SLICE == oracle SLICE
    p = synth.make_c3("exclude_self")
    p.weights = [1.0, 2.0, 0.5, 1.5]
    o = oracle.solve(p, "slice")
    _same(_gpu(p, "enum"), o, "C3 weighted enum")
    _same(_gpu(p, "slice"), o, "C3 weighted slice")


def test_weighted_batch_and_planner_vs_oracle():
    """C5-shaped batch with per-mix weights: host batch, device batch and the persistent planner."""
    import torch
    models, ids, qos = synth.make_c5(48, seed=3)
    rng = np.random.default_rng(8)
    wts = rng.choice([0.5, 1.0, 2.0, 3.0], size=ids.shape).astype(np.float64)
    wts[::5] = 1.0   # some mixes with equal weights
    pr = ec.Profiles.from_models(models)
    kw = dict(total_sms=148, switch_max=14, p_idle_w=200.0, p_max_w=1000.0)
    host = ec.plan_batch(pr, ids, qos_ns=qos, weights=wts, gmax=16, **kw)
    dev = ec.plan_batch(pr, torch.from_numpy(ids).cuda(), qos_ns=torch.from_numpy(qos).cuda(),
                        weights=torch.from_numpy(wts).cuda(), gmax=16, **kw)
    pl = ec.Planner(pr, n_models=4, max_problems=48, weights=True, **kw)
    plo = pl.plan(ids, qos, weights=wts, gmax=16)
    torch.cuda.synchronize()
    for i in range(48):
        p = synth.c5_problem(i, models, ids, qos)
        p.weights = [float(x) for x in wts[i]]
        o = oracle.solve(p, "slice")
        for name, out in (("host", host), ("device", dev), ("planner", plo)):
            st = int(out["status"][i])
            assert (st == 0) == (o.status == "ok"), (name, i)
            if o.status != "ok":
                continue
            assert [int(x) for x in out["winner_levels"][i].tolist()] == o.levels, (name, i)
            assert float(out["objective"][i]) == pytest.approx(o.objective, rel=REL), (name, i)
            assert float(out["energy_busy_j"][i]) == pytest.approx(o.energy_busy_j, rel=REL), (name, i)


def test_weights_invalid_and_energy():
    p = synth.make_c1(1)
    for bad in ([0.0, 1.0], [-1.0, 1.0], [float("nan"), 1.0], [2000.0, 1.0]):
        p.weights = bad
        with pytest.raises(ec.EclipError) as e:
            _gpu(p)
        assert e.value.code == ec.eclip.E_INVALID_ARG
    p = synth.make_c1(1, objective="energy")
    p.weights = [2.0, 1.0]
    with pytest.raises(ec.EclipError):
        _gpu(p)
    p.weights = [2.0, 2.0]   # equal weights: the unweighted energy plan
    q = synth.make_c1(1, objective="energy")
    _same(_gpu(p), oracle.solve(q))
