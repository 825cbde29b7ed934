"""ORACLE for the batched co-location simulator — TEST INFRASTRUCTURE ONLY
(see oracle/__init__).  Plain Python floats (IEEE binary64, no fused operations), one scenario at a
time, in the order SPEC's simulator module states it ("run"; metrics S:362-430):

  * W workers, each running n_requests requests of its model back to back (closed loop: the
    paper tests the "maximum supported RPS"; R19); a request's kernels run in
    order (kernel k depends on kernel k-1 of the same request).
  * Redirection: kernel k runs on the pool of table[k]; pools are sets of SM groups
    (the SE analogue, masks[w][j] bitsets, R17/R18); the full size is the default stream,
    shared by every worker when shared_default -- a FIFO across workers in dispatch
    order (a worker dispatches its whole request when it starts it).
  * Barriers: in PREALLOC mode a kernel whose predecessor ran on another
    stream waits barrier_ns after the predecessor completes (with a fast host the predecessor is
    always still pending at dispatch time).  In IOCTL mode a kernel whose pool size differs from
    its predecessor's waits a repartition cost drawn from triangular(min, mode, max)
    with a counter-based generator (SplitMix64, below) instead.
  * Effective duration: beta(c) x oversub at rate 1 / (1 + alpha(t)), alpha(t) =
    sum over co-running kernels of |mask_k & mask_j| (SMs) / N, recomputed at every start /
    completion (piecewise-constant rate scaling).
  * Energy: integral of p_idle + (p_max - p_idle) busy(t) / N, busy = SMs in the union
    of running masks, over [0, makespan]; p95 = nearest rank; throughput = completed
    requests / the worker's finish time.
"""
from __future__ import annotations

import math
from typing import List, Sequence

M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """SplitMix64 finaliser (Steele, Lea, Flood 2014): the shared counter-based generator."""
    x = (x + 0x9E3779B97F4A7C15) & M64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def uniform(seed: int, s: int, w: int, r: int, k: int) -> float:
    key = (seed + ((((s * 8 + w) << 20) + r) << 8) + k) & M64
    return (splitmix64(key) >> 11) * (1.0 / 9007199254740992.0)


def triangular(u: float, lo: float, mode: float, hi: float) -> float:
    """inverse CDF of triangular(lo, mode, hi)"""
    if hi <= lo:
        return lo
    fc = (mode - lo) / (hi - lo)
    if u < fc:
        return lo + math.sqrt(u * (hi - lo) * (mode - lo))
    return hi - math.sqrt((1.0 - u) * (hi - lo) * (hi - mode))


def sms_of(mask: int, group_sm: Sequence[int]) -> int:
    return sum(group_sm[g] for g in range(len(group_sm)) if (mask >> g) & 1)


def _seqsum(xs: Sequence[float]) -> float:
    """left-to-right binary64 sum (Python 3.12's sum() is compensated; the definition is not)"""
    acc = 0.0
    for x in xs:
        acc += x
    return acc


def p95(values: Sequence[float]) -> float:
    v = sorted(values)
    return v[int(math.ceil(0.95 * len(v))) - 1]


def simulate(beta: Sequence[Sequence[Sequence[float]]], table: Sequence[Sequence[int]],
             masks: Sequence[Sequence[int]], group_sm: Sequence[int], N: int, n_requests: int,
             shared_default: bool = True, ioctl: bool = False, barrier_ns: float = 0.0,
             ioctl_ns=(10000.0, 30000.0, 55400.0), oversub: float = 1.0, p_idle: float = 75.0,
             p_max: float = 225.0, seed: int = 0, scenario: int = 0) -> dict:
    """One scenario.  beta[w][k][j] ns; table[w][k] pool index; masks[w][j] group bitset (the last
    pool j = C-1 is the full device / default stream)."""
    W = len(beta)
    C = len(masks[0])
    full = C - 1
    K = [len(beta[w]) for w in range(W)]

    def stream(w, j):
        if j == full:
            return -1 if shared_default else -2 - w
        return w * C + j

    req = [0] * W                    # current request
    kk = [0] * W                     # current kernel
    ready = [0.0] * W                # earliest start of the current kernel
    running = [False] * W
    rem = [0.0] * W                  # remaining solo work of the running kernel (ns)
    rstart = [0.0] * W               # start time of the current request
    disp = [0.0] * W                 # dispatch time of the current request
    finished = [None] * W
    lat = [[] for _ in range(W)]
    barriers = 0
    events = 0
    t = 0.0
    energy = 0.0                     # W*ns

    def pending_default(w):
        """first kernel index >= kk[w] of the current request on the default stream, else None"""
        if finished[w] is not None:
            return None
        for k in range(kk[w], K[w]):
            if table[w][k] == full:
                return k
        return None

    while True:
        # 1. start every startable kernel (the default stream: FIFO head only, one at a time)
        default_busy = any(running[w] and table[w][kk[w]] == full for w in range(W)) if shared_default else False
        head = None
        if shared_default:
            best = None
            for w in range(W):
                d = pending_default(w)
                if d is not None and not (running[w] and kk[w] == d):
                    key = (disp[w], w)
                    if best is None or key < best:
                        best, head = key, (w, d)
        for w in range(W):
            if finished[w] is not None or running[w] or ready[w] > t:
                continue
            j = table[w][kk[w]]
            if j == full and shared_default:
                if default_busy or head != (w, kk[w]):
                    continue
                default_busy = True
            running[w] = True
            rem[w] = beta[w][kk[w]][j] * oversub
        # 2. rates
        act = [w for w in range(W) if running[w]]
        if not act and all(f is not None for f in finished):
            break
        alpha = {}
        for a in act:
            ma = masks[a][table[a][kk[a]]]
            s = 0
            for b in act:
                if b != a:
                    s += sms_of(ma & masks[b][table[b][kk[b]]], group_sm)
            alpha[a] = s / N
        busy_mask = 0
        for a in act:
            busy_mask |= masks[a][table[a][kk[a]]]
        busy = sms_of(busy_mask, group_sm)
        # 3. next event
        tc = math.inf
        for a in act:
            tc = min(tc, t + rem[a] * (1.0 + alpha[a]))
        tr = math.inf
        for w in range(W):
            if finished[w] is None and not running[w] and ready[w] > t:
                tr = min(tr, ready[w])
        tn = min(tc, tr)
        if tn == math.inf:
            raise RuntimeError("simulator deadlock")
        dt = tn - t
        energy += (p_idle + (p_max - p_idle) * (busy / N)) * dt
        done = []
        for a in act:
            if t + rem[a] * (1.0 + alpha[a]) == tc and tc == tn:
                done.append(a)
            else:
                rem[a] = rem[a] - dt / (1.0 + alpha[a])
        t = tn
        # 4. completions
        for a in done:
            events += 1
            running[a] = False
            jprev = table[a][kk[a]]
            kk[a] += 1
            if kk[a] == K[a]:
                lat[a].append(t - rstart[a])
                req[a] += 1
                kk[a] = 0
                if req[a] == n_requests:
                    finished[a] = t
                    continue
                rstart[a] = t
                disp[a] = t
                ready[a] = t
            else:
                jn = table[a][kk[a]]
                extra = 0.0
                if ioctl:
                    if jn != jprev:
                        u = uniform(seed, scenario, a, req[a], kk[a])
                        extra = triangular(u, ioctl_ns[0], ioctl_ns[1], ioctl_ns[2])
                elif stream(a, jn) != stream(a, jprev):
                    barriers += 1
                    extra = barrier_ns
                ready[a] = t + extra
    makespan = t
    thr = [n_requests / (finished[w] * 1e-9) for w in range(W)]
    energy_j = energy * 1e-9
    return {"throughput_rps": thr, "p95_ns": [p95(lat[w]) for w in range(W)],
            "mean_ns": [_seqsum(lat[w]) / len(lat[w]) for w in range(W)], "makespan_ns": makespan,
            "energy_j": energy_j, "req_per_j": W * n_requests / energy_j, "barriers": barriers, "events": events,
            "latencies_ns": lat}
