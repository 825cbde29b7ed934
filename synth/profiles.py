"""Knee-shaped synthetic kernel profiles (SPEC.md synthesize_profile, S:70-78, S:109;
shapes after PAPER.md §IV-B P:264-265 "widely varying thresholds", §V).

Per kernel: draw a knee index k* from the family's distribution over the C sizes and a
base time t* (ns) log-uniform in the family's range, delta ~ U[0, 0.01]:
    j <  k*:  t* (1+delta) c_{k*} / c_j          (hyperbolic up to the knee)
    j >= k*:  t* (1 + delta (C-1-j)/(C-1))        (flat within 1 %, non-increasing)
rounded to integer ns.  Monotone non-increasing in the size by construction
(SPEC KernelProfile invariant S:43-44), asserted here.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

# family -> (knee sampler over C sizes, base-time range in ns).  SURVEY.md §8(d) table.
#   knee sampler gets (rng, C) and returns a knee index in [0, C).
FAMILIES = {
    # "vgg19's kernels typically require all 60 CUs": knees at the top two sizes
    "vgg": (lambda r, C: int(r.integers(C - 2, C)), (200_000, 2_000_000)),
    "resnet": (lambda r, C: int(r.integers(C // 4, max(C // 4 + 1, (3 * C) // 4))), (20_000, 300_000)),
    # bimodal: GEMM groups at the top, elementwise / softmax / LayerNorm at the bottom
    "bert": (lambda r, C: int(r.integers(C - 2, C)) if r.random() < 0.5 else int(r.integers(0, 2)),
             (5_000, 100_000)),
    "densenet": (lambda r, C: int(r.integers(0, max(1, C // 2))), (10_000, 150_000)),
    "resnext": (lambda r, C: int(r.integers(C // 2, C)), (30_000, 400_000)),
    "alexnet": (lambda r, C: C - 1, (100_000, 1_000_000)),
    "shufflenet": (lambda r, C: int(r.integers(0, max(1, C // 4))), (5_000, 50_000)),
    # uniform knees (SPEC synthesize_profile "knees uniform over configs")
    "uniform": (lambda r, C: int(r.integers(0, C)), (5_000, 200_000)),
}


@dataclass
class Model:
    """One model's profile: exec_ns[k][j] for kernel k at size column j (integer ns)."""
    name: str
    sizes: List[int]
    exec_ns: np.ndarray  # int64 [K, C]
    knees: List[int] = field(default_factory=list)

    @property
    def n_kernels(self) -> int:
        return int(self.exec_ns.shape[0])


def lattice_sizes(n_sizes: int, total: int) -> List[int]:
    """SE-granularity lattice scaled to `total` SMs: c_j = (j+1) * floor(total / C)
    (SURVEY.md §8(c) reading c3-B; MI50: 60 CUs, C=4 -> {15,30,45,60})."""
    u = total // n_sizes
    return [(j + 1) * u for j in range(n_sizes)]


def synthesize_model(name: str, family: str, n_kernels: int, sizes: Sequence[int],
                     seed: int) -> Model:
    rng = np.random.default_rng(seed)
    knee_fn, (lo, hi) = FAMILIES[family]
    C = len(sizes)
    ex = np.zeros((n_kernels, C), dtype=np.int64)
    knees = []
    for k in range(n_kernels):
        ks = knee_fn(rng, C)
        t = float(np.exp(rng.uniform(np.log(lo), np.log(hi))))
        d = float(rng.uniform(0.0, 0.01))
        for j in range(C):
            if j < ks:
                v = t * (1.0 + d) * sizes[ks] / sizes[j]
            else:
                v = t * (1.0 + d * (C - 1 - j) / max(1, C - 1))
            ex[k, j] = max(1, int(round(v)))
        knees.append(ks)
        assert all(ex[k, j] >= ex[k, j + 1] for j in range(C - 1)), "non-monotone draw"
    return Model(name, list(sizes), ex, knees)


def _us(ns: int) -> str:
    """integer ns -> exact decimal microseconds string."""
    neg = ns < 0
    ns = abs(int(ns))
    s = f"{ns // 1000}.{ns % 1000:03d}"
    return "-" + s if neg else s


def write_profile_text(models: Sequence[Model]) -> str:
    """SPEC profile format: per model a JSON header line
    {"model": name, "kernels": N, "configs": [...]} then one CSV row per kernel:
    kernel_id, t_c0, t_c1, ... in decimal microseconds.  Several models may be
    concatenated in one file ("calibration mix ... 3 ModelProfiles")."""
    out = []
    for m in models:
        cfg = ", ".join(str(c) for c in m.sizes)
        out.append(f'{{"model": "{m.name}", "kernels": {m.n_kernels}, "configs": [{cfg}]}}')
        for k in range(m.n_kernels):
            out.append(", ".join([str(k)] + [_us(int(v)) for v in m.exec_ns[k]]))
    return "\n".join(out) + "\n"
