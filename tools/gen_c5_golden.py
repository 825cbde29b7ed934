"""Write tests/golden/c5_mixes.json: the ORACLE's answer for EVERY distinct C5 request mix.

A C5 mix is W = 4 draws with replacement from the 7-model library (synth.make_c5), and its
QoS bounds are a function of the drawn models, so a C5 batch of any seed holds at most
7^4 = 2401 distinct (ordered) problems.  This script solves each of them with the oracle's
exact T'-slice method (oracle.solve(..., "slice"), plain single-threaded C per problem; the
problems are spread over a process pool) and stores, per ordered model tuple:
status, winning level ranks, mixed-radix index, exact integer key (hex), FP64 objective and
the chosen size column of every group.  bench.py and the GPU tests check every planned mix
of a batch against it.  Calls only oracle/ and synth/ — never the CUDA path.

    python tools/gen_c5_golden.py            (~1-2 min on 8 cores)
"""
import hashlib
import itertools
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "c5_mixes.json")
W = 4


def library_hash(models) -> str:
    h = hashlib.sha256()
    for m in models:
        h.update(np.ascontiguousarray(m.exec_ns).tobytes())
        h.update(str(m.sizes).encode())
    return h.hexdigest()[:16]


def _solve(tup):
    models, _, _ = synth.make_c5(1)
    ids = np.array([tup], np.int32)
    solo = np.array([synth.qos_3x(models, [m])[0] for m in range(len(models))])
    qos = solo[ids]
    r = oracle.solve(synth.c5_problem(0, models, ids, qos), "slice")
    if r.status != "ok":
        return tup, ["infeasible"]
    cols = "".join("%x" % c for row in r.group_cols for c in row)
    return tup, ["ok", r.levels, r.index, "%x" % r.key, repr(r.objective), cols]


def main():
    models, _, _ = synth.make_c5(1)
    tuples = list(itertools.product(range(len(models)), repeat=W))
    t = time.time()
    with mp.Pool(os.cpu_count()) as pool:
        res = dict(pool.map(_solve, tuples, chunksize=8))
    answers = {",".join(map(str, k)): res[k] for k in tuples}
    n_ok = sum(1 for v in answers.values() if v[0] == "ok")
    doc = dict(source="tools/gen_c5_golden.py (oracle/ only: oracle.solve(problem, 'slice') per distinct mix)",
               workload="synth.make_c5: W=4 draws from the 7-model library, 16 groups x 8 sizes, N=148, R=14, "
                        "EXCLUDE_SELF, SUM, Q_w = 3x isolated latency at the largest size, p 200/1000 W, tau 1e-5",
               library_hash=library_hash(models), n_models=len(models), W=W,
               fields=["status", "levels", "index", "exact_key_hex", "objective_ns", "group_cols_hex (worker-major)"],
               n_mixes=len(answers), n_feasible=n_ok, oracle_seconds=round(time.time() - t, 1), answers=answers)
    with open(OUT, "w") as f:
        json.dump(doc, f, separators=(",", ":"))
        f.write("\n")
    print(f"{len(answers)} mixes ({n_ok} feasible) in {time.time() - t:.1f} s -> {OUT}")


if __name__ == "__main__":
    main()
