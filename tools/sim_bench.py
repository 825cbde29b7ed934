"""Batched co-location simulation of the planner's plans on one B200:
the C5 batch (4096 mixes x 4 models x 16 groups, 8 pool sizes {18..144} of N = 148) is planned
(eclip_plan_batch), then every mix is simulated twice -- with its ECLIP plan on the pre-allocated
pool (rotation layout over 8 groups of 18 SMs + a 4-SM remainder, barrier 2 us) and with the
all-max baseline (every kernel on the shared default stream) -- n_requests closed-loop
requests per worker.  Reports simulated scenarios/s and kernel events/s (eclip_simulate wall time,
inputs on the host) and the distribution of ECLIP / baseline throughput and requests/J.

    python tools/sim_bench.py [--mixes 4096] [--requests 20] [--out gpurun_out/sim.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2506_12598_b200 as ec  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mixes", type=int, default=4096)
    ap.add_argument("--requests", type=int, default=20)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/sim.json")
    a = ap.parse_args()
    models, ids, qos = synth.make_c5(a.mixes)
    pr = ec.Profiles.from_models(models)
    out = ec.plan_batch(pr, ids, total_sms=148, qos_ns=qos, p_idle_w=200.0, p_max_w=1000.0, gmax=16)
    W, Cn = 4, len(models[0].sizes)
    K = 16
    gsm = [18] * 8 + [4]
    G = len(gsm)
    masks = np.zeros((W, Cn), np.uint32)
    for w in range(W):
        for j in range(Cn - 1):
            masks[w, j] = sum(1 << ((w * 8 // W + t) % 8) for t in range(j + 1))
        masks[w, Cn - 1] = (1 << G) - 1
    S = a.mixes
    ok = np.asarray(out["status"]) == 0
    ex = np.stack([m.exec_ns for m in models])             # [7, K, C]
    beta = np.concatenate([ex[ids], ex[ids]]).astype(np.float64)   # [2S, W, K, C]
    gs = np.asarray(out["group_sm"])                       # [S, W, 16] pool sizes (SMs)
    sizes = np.asarray(models[0].sizes)
    tab_e = np.searchsorted(sizes, np.where(ok[:, None, None], gs, sizes[-1]))
    table = np.concatenate([tab_e, np.full((S, W, K), Cn - 1)]).astype(np.int32)
    nk = np.full((2 * S, W), K, np.int32)
    kw = dict(total_sms=148, n_requests=a.requests, barrier_ns=2000.0, p_idle_w=200.0, p_max_w=1000.0)
    ec.simulate(nk[:8], beta[:8], table[:8], masks, gsm, **kw)   # warm-up
    ts = []
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = ec.simulate(nk, beta, table, masks, gsm, **kw)
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    ev = int(r["events"].sum())
    thr = r["throughput_rps"].sum(axis=1)
    nt = thr[:S] / thr[S:]
    ne = r["req_per_j"][:S] / r["req_per_j"][S:]
    q = lambda x: {"p10": float(np.percentile(x, 10)), "median": float(np.median(x)), "p90": float(np.percentile(x, 90)),
                   "mean": float(np.mean(x))}
    res = {"scenarios": 2 * S, "requests_per_worker": a.requests, "kernel_events": ev, "wall_s": t,
           "scenarios_per_s": 2 * S / t, "events_per_s": ev / t,
           "note": "wall time of eclip_simulate (host inputs, H2D + kernel + D2H); one GPU thread per scenario",
           "feasible_mixes": int(ok.sum()),
           "eclip_over_baseline_throughput": q(nt[ok]), "eclip_over_baseline_req_per_j": q(ne[ok])}
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
