"""The oracle's answer for every distinct C5 mix (tests/golden/c5_mixes.json, written by
tools/gen_c5_golden.py from oracle/ only) and a checker for a planned C5 batch.

Used by the GPU tests and by bench.py to re-check every timed run's winners.  Reads the
stored answers only: no planning arithmetic here."""
from __future__ import annotations

import json
import os

import numpy as np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c5_mixes.json")
_doc = None


def load():
    global _doc
    if _doc is None:
        with open(PATH) as f:
            _doc = json.load(f)
    return _doc


def check_batch(ids, out, sizes=None, rel: float = 1e-5) -> int:
    """Compare a plan_batch result (numpy arrays or torch tensors) with the oracle's stored
    answers, mix by mix: status, winning level ranks, mixed-radix index and objective; with
    `sizes` (the library's size list) also every group's pool size.  Raises AssertionError on
    the first mismatch; returns the number of mixes checked."""
    doc = load()
    ans = doc["answers"]
    get = lambda k: (out[k].cpu().numpy() if hasattr(out[k], "cpu") else np.asarray(out[k]))
    st, lv = get("status"), get("winner_levels")
    idx = get("winner_index").view(np.uint64) if get("winner_index").dtype != np.uint64 else get("winner_index")
    obj = get("objective")
    gsm = get("group_sm") if (sizes is not None and "group_sm" in out and out["group_sm"] is not None) else None
    ids = np.asarray(ids.cpu().numpy() if hasattr(ids, "cpu") else ids)
    W = doc["W"]
    for i in range(ids.shape[0]):
        a = ans[",".join(str(int(x)) for x in ids[i])]
        if a[0] != "ok":
            assert int(st[i]) == 1, f"mix {i}: oracle INFEASIBLE, planner status {int(st[i])}"
            continue
        assert int(st[i]) == 0, f"mix {i}: oracle feasible, planner status {int(st[i])}"
        assert lv[i].tolist() == a[1], f"mix {i}: levels {lv[i].tolist()} != oracle {a[1]}"
        assert int(idx[i]) == a[2], f"mix {i}: index {int(idx[i])} != oracle {a[2]}"
        o = float(a[4])
        assert abs(float(obj[i]) - o) <= rel * abs(o), f"mix {i}: objective {float(obj[i])} != oracle {o}"
        if gsm is not None:
            cols = [int(c, 16) for c in a[5]]
            G = len(cols) // W
            want = [[sizes[cols[w * G + g]] for g in range(G)] for w in range(W)]
            assert gsm[i, :, :G].tolist() == want, f"mix {i}: group sizes differ from the oracle's"
    return int(ids.shape[0])
