"""Device timeline of bench steps (CUPTI via torch.profiler; one GPU):
    python tools/timeline.py [--mixes N] [--steps K] [--out gpurun_out/timeline.json]
Prints every kernel of each profiled plan_batch step with its start offset from the step's
first kernel, duration and the idle gap before it, and the host wall time of the call."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2506_12598_b200 as ec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mixes", type=int, default=4096)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--out", default="gpurun_out/timeline.json")
ap.add_argument("--problem", default="", help="c2|c3|c4|s6: one eclip_plan call per step instead of the C5 batch")
a = ap.parse_args()
models, ids, qos = synth.make_c5(a.mixes)
pr = ec.Profiles.from_models(models)
st = torch.cuda.current_stream()
d_ids, d_q = torch.from_numpy(ids).cuda(), torch.from_numpy(qos).cuda()
out = ec.alloc_batch_out(a.mixes, 4, 16, device="cuda")
pl = ec.Planner(pr, n_models=4, max_problems=a.mixes, total_sms=148, p_idle_w=200.0, p_max_w=1000.0,
                stream=st.cuda_stream)
if a.problem:   # single problems: the one-shot eclip_plan (session set-up, K1, search, materialisation)
    prob = {"c2": synth.make_c2, "c3": lambda: synth.make_c3("matrix"), "c4": synth.make_c4, "s6": synth.make_s6}[a.problem]()
    prp = ec.Profiles.from_models(prob.models)

    class _One:
        def plan(self, *args, **kw):
            ec.plan_problem(prp, prob, stream=st.cuda_stream)
    pl = _One()
for _ in range(3):
    pl.plan(d_ids, d_q, out=out)
torch.cuda.synchronize()
walls = []
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(a.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.profiler.record_function("step"):
            pl.plan(d_ids, d_q, out=out)
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t0) * 1e3)
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
prof.export_chrome_trace(a.out)
ev = json.load(open(a.out))["traceEvents"]
kern = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
steps = sorted([e for e in ev if e.get("name") == "step" and e.get("cat") == "user_annotation"], key=lambda e: e["ts"])
for i, s in enumerate(steps):
    ks = [k for k in kern if s["ts"] <= k["ts"] <= s["ts"] + s["dur"] + 50000]
    if i + 1 < len(steps):
        ks = [k for k in ks if k["ts"] < steps[i + 1]["ts"]]
    print(f"--- step {i}: host wall {walls[i]:.3f} ms; host step span {s['dur'] / 1e3:.3f} ms")
    prev = s["ts"]
    busy = 0.0
    for k in ks:
        gap = k["ts"] - prev
        print(f"  +{(k['ts'] - s['ts']) / 1e3:8.3f} ms  gap {gap:8.1f} us  dur {k['dur']:8.1f} us  {k['name'][:70]}")
        prev = k["ts"] + k["dur"]
        busy += k["dur"]
    if ks:
        span = ks[-1]["ts"] + ks[-1]["dur"] - s["ts"]
        print(f"  device busy {busy / 1e3:.3f} ms of {span / 1e3:.3f} ms from step start")
