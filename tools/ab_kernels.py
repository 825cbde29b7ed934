"""A/B timing of the planner's main configurations with whichever libeclip ECLIP_LIB selects:
C5 pruned step + pass-1 kernel, exhaustive passes with / without QoS (kernel ms, FMA-pipe fraction),
and single-problem time-to-plan (C2, C3, C4, S6).   python tools/ab_kernels.py [--mixes N]"""
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

ap = argparse.ArgumentParser()
ap.add_argument("--mixes", type=int, default=4096)
a = ap.parse_args()
res = {"lib": os.environ.get("ECLIP_LIB", "default")}
models, ids, qos = synth.make_c5(a.mixes)
pr = ec.Profiles.from_models(models)
d_ids, d_q = torch.from_numpy(ids).cuda(), torch.from_numpy(qos).cuda()
out = ec.alloc_batch_out(a.mixes, 4, 16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
kw = dict(n_models=4, max_problems=a.mixes, total_sms=148, p_idle_w=200.0, p_max_w=1000.0, timing=True)
peak = 148 * 128 * 1965e6
for name, q, prune in (("pruned", True, True), ("exh_qos", True, False), ("exh_noqos", False, False)):
    pl = ec.Planner(pr, qos=q, prune=prune, **kw)
    ks, st, ev = [], [], []
    for rep in range(6 if prune else 3):
        flush.fill_(1)
        pl.plan(d_ids, d_q if q else None, out=out)
        torch.cuda.synchronize()
        if rep >= 1:
            c = pl.counters()
            ks.append(c["kernel_ms"]); ev.append(c["evaluated_candidates"]); st.append(sum(pl.phase_ms().values()))
    k = float(np.median(ks)); e = int(np.median(ev))
    res[name] = {"kernel_ms": k, "step_ms": float(np.median(st)), "evaluated": e,
                 "fma_frac": 2 * e / (k * 1e-3) / peak, "counters": c, "phases": pl.phase_ms()}
    del pl
for name, p in (("C2", synth.make_c2()), ("C3", synth.make_c3("matrix")), ("C4", synth.make_c4()), ("S6", synth.make_s6())):
    prp = ec.Profiles.from_models(p.models)
    ts = []
    for rep in range(4):
        t0 = time.perf_counter()
        r = ec.plan_problem(prp, p)
        ts.append((time.perf_counter() - t0) * 1e3)
    res[name] = {"ms": float(np.median(ts[1:])), "objective": r.objective, "levels": r.winner_levels}
print(json.dumps(res))
