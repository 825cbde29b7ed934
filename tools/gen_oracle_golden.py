"""Write tests/golden/oracle_full.json: the ORACLE's answers at BASELINE.json's full sizes
(C3 with the slowdown matrix, C3 under EXCLUDE_SELF, C4 via the oracle's T'-slice method,
sampled C5 mixes, S6).  Calls only oracle/ and synth/ — never the CUDA path.  Each record
stores a hash of its seeded inputs so a stale file is detected by the tests.

    python tools/gen_oracle_golden.py          (~5-10 min single-threaded)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "oracle_full.json")
C5_SAMPLES = [0, 1, 2047, 4095]


problem_hash = synth.problem_hash
c5_problem = synth.c5_problem


def record(p, engine):
    t = time.time()
    r = oracle.solve(p, engine)
    return dict(name=p.name, hash=problem_hash(p), engine=engine, status=r.status, levels=r.levels, index=r.index,
                key=str(r.key), min_key=str(r.min_key), group_sm=r.group_sm, switches=r.switches,
                latency_ns=r.latency_ns, objective=r.objective, makespan_ns=r.makespan_ns, power_w=r.power_w,
                energy_j=r.energy_j, throughput_rps=r.throughput_rps, oracle_seconds=round(time.time() - t, 2))


def main():
    recs = {}
    recs["C3"] = record(synth.make_c3("matrix"), "enum")
    recs["C3_excl"] = record(synth.make_c3("exclude_self"), "slice")
    recs["C4"] = record(synth.make_c4(), "slice")
    recs["S6"] = record(synth.make_s6(), "slice")
    models, ids, qos = synth.make_c5(4096)
    for i in C5_SAMPLES:
        recs[f"C5_{i}"] = record(c5_problem(i, models, ids, qos), "slice")
    for k, v in recs.items():
        print(k, v["status"], v["levels"], v["oracle_seconds"], "s")
    json.dump(dict(source="tools/gen_oracle_golden.py (oracle/ only)", records=recs), open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main()
