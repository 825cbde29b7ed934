"""ORACLE for the runtime scheduler — TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Plain Python statements of what PAPER.md §IV-A fixes, used to check the GPU runtime's recorded
decisions and timelines (the runtime's timing itself has no oracle: it is measured).

  pool_groups      the SM groups (SE analogue) of worker w's pool of j groups out of G: the paper's
                   2-worker layout (worker 1 15 CU = SE1, 30 = SE1,3, 45 = SE1,2,3; worker 2
                   15 = SE4, 30 = SE2,4, 45 = SE2,3,4) generalised as a rotation (R17):
                   worker w takes groups s_w, s_w+1, ... (mod G), s_w = floor(w G / W).  The full
                   size is every group ("the 60 CU allocation is the default stream").
  pairwise_overlap groups shared by two workers' pools of the same size (the quantity the paper's
                   layout keeps small, "minimal sharing").
  redirect         kernel k -> the pool of its lookup-table size.
  needs_barrier    P:239-241: "(i) the kernel has a dependency on a previous kernel from the same
                   stream, and (ii) that previous kernel has not yet completed execution" -- and a
                   kernel redirected to the SAME pool stream needs none (FIFO order).
  dependency_ok    SPEC simulator invariant "kernel k of request r never starts before kernel k-1
                   of request r completes", on recorded device timestamps.
"""
from __future__ import annotations

from typing import List, Sequence


def pool_groups(G: int, W: int, w: int, j: int) -> List[int]:
    """groups of worker w's pool with j groups (1 <= j <= G); j == G -> all groups"""
    if j >= G:
        return list(range(G))
    start = (w * G) // W
    return sorted((start + t) % G for t in range(j))


def pairwise_overlap(G: int, W: int, j: int, a: int, b: int) -> int:
    return len(set(pool_groups(G, W, a, j)) & set(pool_groups(G, W, b, j)))


def redirect(sizes: Sequence[int], table: Sequence[int], k: int) -> int:
    """size index of kernel k's pool (table[k] is its pool size in SMs)"""
    return list(sizes).index(table[k])


def needs_barrier(prev_stream: int, stream: int, prev_pending: bool) -> bool:
    if prev_stream < 0:
        return False
    return prev_stream != stream and prev_pending


def dependency_ok(t_start: Sequence[int], t_end: Sequence[int]) -> bool:
    """every kernel of one request starts after its predecessor ended (device ns)"""
    return all(t_start[k] >= t_end[k - 1] for k in range(1, len(t_start)))
