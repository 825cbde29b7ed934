"""The paper's end-to-end experiment (§V) on one B200 with the runtime of
SURVEY §8(f) f2: synthetic knee-shaped models are profiled on every pre-allocated SM pool
(the offline profiling of P:265/P:308), the planner (eclip_plan) picks a per-kernel pool under the
switch budget, and co-located workers run closed-loop under the paper's scenarios:

  baseline      every kernel on the shared full-device stream ("default stream that uses all
                60 CUs")
  model_wise    one pool per model (eclip_baseline_plan MODEL_WISE, factor 3)
  kw_prealloc   every kernel at its minimum-SM threshold on the pre-allocated pool
  kw_ioctl      the same plan, repartitioning on every switch (a fresh green context: the IOCTL
                path of Obs. 1)
  eclip         the optimizer's plan on the pre-allocated pool

Reported per scenario: throughput (requests/s, sum over workers), p95 latency per worker,
energy (NVML total-energy counter over the run) and requests/J, barriers and repartition time;
and the planner's predicted per-worker latency next to the measured mean.

    python tools/runtime_experiment.py [--requests 40] [--out gpurun_out/runtime.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2506_12598_b200 as ec  # noqa: E402
from paper_2506_12598_b200 import runtime as rtm  # noqa: E402

FAMILIES = {   # (knee CTA choices, iterations range): shapes after P:265 / P:375 / P:443
    "vgg_like": ([148, 128, 112], (30000, 60000)),
    "resnet_like": ([32, 48, 64, 96], (10000, 30000)),
    "bert_like": ([148, 128, 8, 16], (8000, 25000)),
    "shufflenet_like": ([8, 16, 24], (8000, 20000)),
}


def make_models(rng, names, K):
    out = []
    for n in names:
        knees, (lo, hi) = FAMILIES[n]
        out.append(rtm.SyntheticModel(rng.choice(knees, size=K), rng.integers(lo, hi, size=K)))
    return out


def energy_mj(h):
    import pynvml
    return pynvml.nvmlDeviceGetTotalEnergyConsumption(h)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=40)
    ap.add_argument("--kernels", type=int, default=16)
    ap.add_argument("--group-sms", type=int, default=16)
    ap.add_argument("--own-default", action="store_true", help="one full-device stream per worker")
    ap.add_argument("--out", default="gpurun_out/runtime.json")
    a = ap.parse_args()
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    names = ["vgg_like", "resnet_like", "bert_like", "shufflenet_like"]
    W = len(names)
    rng = np.random.default_rng(2506_12598)
    models = make_models(rng, names, a.kernels)
    rt = rtm.Runtime(W, group_sms=a.group_sms, shared_default=not a.own_default)
    sizes = rt.sizes
    N = rt.total_sms
    # offline profiling on worker 0's pools; measurement noise is removed by a running minimum over the
    # ascending pool sizes (a larger pool is never slower; SPEC S:43 requires non-increasing profiles)
    t0 = time.perf_counter()
    prof = [rt.profile(m, reps=5) for m in models]
    prof_s = time.perf_counter() - t0
    exec_ns = [np.minimum.accumulate(np.rint(p).astype(np.int64), axis=1) for p in prof]
    pr = ec.Profiles.from_arrays(sizes, exec_ns)
    kw = dict(total_sms=N, switch_max=14, p_idle_w=200.0, p_max_w=1000.0)
    plan = ec.plan(pr, list(range(W)), **kw)
    tables = {"eclip": plan.group_sm}
    for key, kind, param in (("baseline", "all_max", 0.0), ("model_wise", "model_wise", 3.0),
                             ("kw_prealloc", "kernel_wise", 0.05)):
        tables[key] = ec.baseline_plan(pr, list(range(W)), kind=kind, param=param, **kw).group_sm
    tables["kw_ioctl"] = tables["kw_prealloc"]
    res = {"device": pynvml.nvmlDeviceGetName(h), "sizes": sizes, "total_sms": N, "group_sm": rt.group_sm,
           "models": names, "kernels": a.kernels, "shared_default": not a.own_default,
           "eclip_tables": [list(map(int, t)) for t in tables["eclip"]], "requests": a.requests, "profile_s": prof_s,
           "profiles_us": [(e / 1e3).round(2).tolist() for e in exec_ns],
           "predicted_latency_us": {"eclip": [x / 1e3 for x in plan.model_latency_ns]}, "scenarios": {}}
    # warm-up run
    for w in range(W):
        rt.set_table(w, tables["baseline"][w])
    rt.run(models, 3)
    for name in ("baseline", "model_wise", "kw_prealloc", "kw_ioctl", "eclip"):
        for w in range(W):
            rt.set_table(w, tables[name][w])
        e0 = energy_mj(h)
        out = rt.run(models, a.requests, repartition=(name == "kw_ioctl"))
        e1 = energy_mj(h)
        lat = out["latency_ns"] / 1e3
        busy_s = out["latency_ns"].sum(axis=1) / 1e9
        rps = (a.requests / busy_s)
        joules = (e1 - e0) / 1e3
        res["scenarios"][name] = {
            "throughput_rps": float(rps.sum()), "rps_per_worker": rps.round(2).tolist(),
            "p95_us": [float(np.sort(x)[int(np.ceil(0.95 * len(x))) - 1]) for x in lat],
            "mean_us": lat.mean(axis=1).round(2).tolist(), "wall_s": out["wall_ns"] / 1e9,
            "energy_j": joules, "req_per_j": (W * a.requests) / joules if joules > 0 else None,
            "barriers": out["barriers"], "repartition_ms": out["repartition_ns"] / 1e6,
            "switches": [int(np.sum(np.diff(np.asarray(t)) != 0)) for t in tables[name]],
        }
    base = res["scenarios"]["baseline"]
    for name, s in res["scenarios"].items():
        s["norm_throughput"] = s["throughput_rps"] / base["throughput_rps"]
        if s["req_per_j"] and base["req_per_j"]:
            s["norm_energy_eff"] = s["req_per_j"] / base["req_per_j"]
    rt.close()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)
    for name, s in res["scenarios"].items():
        print(f"{name:12s} rps {s['throughput_rps']:9.1f} ({s.get('norm_throughput', 0):.3f}x)  "
              f"req/J {s['req_per_j'] or 0:7.2f} ({s.get('norm_energy_eff', 0):.3f}x)  p95 {s['p95_us']}  "
              f"barriers {s['barriers']}  repart {s['repartition_ms']:.1f} ms  switches {s['switches']}")
    print("predicted (eclip)", res["predicted_latency_us"]["eclip"], "measured", res["scenarios"]["eclip"]["mean_us"])


if __name__ == "__main__":
    main()
