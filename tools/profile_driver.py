"""Workloads for ncu (one GPU): `python tools/profile_driver.py c5|c4|c3 [--mixes N]`.
Runs one warm-up and one measured call of the named workload through the public API (C5: the
persistent planner, so the level tables are built once before the per-step kernels)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2506_12598_b200 as ec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("what", choices=["c5", "c4", "c3", "s6"])
ap.add_argument("--mixes", type=int, default=4096)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--noqos", action="store_true")
ap.add_argument("--exhaustive", action="store_true", help="C5 without branch and bound (no_prune)")
a = ap.parse_args()
if a.what == "c5":
    models, ids, qos = synth.make_c5(a.mixes)
    pr = ec.Profiles.from_models(models)
    d_ids, d_q = torch.from_numpy(ids).cuda(), (None if a.noqos else torch.from_numpy(qos).cuda())
    out = ec.alloc_batch_out(a.mixes, 4, 16, device="cuda")
    pl = ec.Planner(pr, n_models=4, max_problems=a.mixes, total_sms=148, qos=not a.noqos, p_idle_w=200.0,
                    p_max_w=1000.0, prune=not a.exhaustive)
    for _ in range(a.reps):
        pl.plan(d_ids, d_q, out=out)
    torch.cuda.synchronize()
else:
    p = {"c4": synth.make_c4, "c3": lambda: synth.make_c3("matrix"), "s6": synth.make_s6}[a.what]()
    pr = ec.Profiles.from_models(p.models)
    for _ in range(a.reps):
        r = ec.plan_problem(pr, p)
    print(r.engine, r.objective)
