"""BASELINE.json configs as plain seeded data (SURVEY.md §8(d) "Configs as concrete
synthetic inputs").  No method arithmetic here: only draws, model choice, and the
QoS *input* convention Q_w = 3 x isolated latency at the largest allowed size
(§II-C P:82 "typically 3x the tail latency when running in isolation").

Mode / objective are carried as strings; the oracle and the product each map them
to their own codes.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from .profiles import Model, lattice_sizes, synthesize_model

SEED_BASE = 2506_12598 * 16
MODES = ("exclude_self", "paper", "excess", "matrix")
OBJECTIVES = ("sum", "max", "energy")


@dataclass
class Problem:
    """One planning problem (one co-location mix) over a model library.

    models       : the profile library (all share `sizes`)
    model_ids    : [W] worker -> library model (repeats allowed, P:378 Mix1 = 2x albert)
    group_bounds : per worker None (one group per kernel, exact paper formulation P:299)
                   or kernel offsets [0, b1, ..., K] (contiguous kernel groups)
    allowed_mask : per worker bitmask over size columns (P:222 pool layouts); None = all
    qos_ns       : per worker latency bound Q_w (inf = none)
    """
    name: str
    models: List[Model]
    model_ids: List[int]
    total_sms: int
    switch_max: int
    mode: str = "exclude_self"
    objective: str = "sum"
    allowed_mask: Optional[List[int]] = None
    qos_ns: Optional[List[float]] = None
    slowdown_matrix: Optional[np.ndarray] = None  # float32 [W, W] (mode == "matrix")
    group_bounds: Optional[List[Optional[List[int]]]] = None
    p_idle_w: float = 75.0
    p_max_w: float = 225.0
    weights: Optional[List[float]] = None   # per-worker objective weights; None = all 1

    @property
    def W(self) -> int:
        return len(self.model_ids)

    @property
    def sizes(self) -> List[int]:
        return self.models[0].sizes


def qos_3x(models: Sequence[Model], model_ids: Sequence[int], factor: float = 3.0,
           masks: Optional[Sequence[int]] = None) -> List[float]:
    """Q_w = factor x (sum over kernels of the time at the largest allowed size)."""
    out = []
    for w, mid in enumerate(model_ids):
        m = models[mid]
        C = len(m.sizes)
        mask = (masks[w] if masks is not None else (1 << C) - 1)
        jmax = max(j for j in range(C) if (mask >> j) & 1)
        out.append(float(factor * int(m.exec_ns[:, jmax].sum())))
    return out


def _matrix(rng: np.random.Generator, W: int) -> np.ndarray:
    """c3-M: off-diagonal M ~ U[0.5, 1.5], diagonal unused (set 0), float32."""
    M = rng.uniform(0.5, 1.5, size=(W, W)).astype(np.float32)
    np.fill_diagonal(M, 0.0)
    return M


def make_c1(R: int = 1, mode: str = "exclude_self", objective: str = "sum",
            qos: bool = False, seed: int = 1) -> Problem:
    """C1: 2 models x 3 groups, sizes {15,30,45,60} of 60 CUs."""
    sizes = lattice_sizes(4, 60)
    s = SEED_BASE + 1 + 1000 * seed
    models = [synthesize_model("m0", "uniform", 3, sizes, s),
              synthesize_model("m1", "uniform", 3, sizes, s + 1)]
    ids = [0, 1]
    M = _matrix(np.random.default_rng(s + 7), 2) if mode == "matrix" else None
    return Problem("C1", models, ids, 60, R, mode, objective,
                   qos_ns=qos_3x(models, ids) if qos else None, slowdown_matrix=M)


def make_c2(mode: str = "exclude_self", objective: str = "sum") -> Problem:
    """C2: ResNet-50-, VGG-19-, BERT-base-like x 8 groups x {15,30,45,60}, N=60, R=14."""
    sizes = lattice_sizes(4, 60)
    s = SEED_BASE + 2
    models = [synthesize_model("resnet50", "resnet", 8, sizes, s),
              synthesize_model("vgg19", "vgg", 8, sizes, s + 1),
              synthesize_model("bert_base", "bert", 8, sizes, s + 2)]
    M = _matrix(np.random.default_rng(s + 7), 3) if mode == "matrix" else None
    return Problem("C2", models, [0, 1, 2], 60, 14, mode, objective, slowdown_matrix=M)


LIBRARY_FAMILIES = ("albert:bert", "densenet201:densenet", "alexnet:alexnet",
                    "resnet152:resnet", "resnext101:resnext", "shufflenet:shufflenet",
                    "vgg19:vgg")  # the paper's 7 models, as look-alike families


def library_models(n_groups: int = 16, n_sizes: int = 8, total: int = 148,
                   seed: int = 5) -> List[Model]:
    sizes = lattice_sizes(n_sizes, total)
    out = []
    for i, nf in enumerate(LIBRARY_FAMILIES):
        name, fam = nf.split(":")
        out.append(synthesize_model(name, fam, n_groups, sizes, SEED_BASE + 100 * seed + i))
    return out


def make_c3(mode: str = "matrix") -> Problem:
    """C3: 4 models x 16 groups x 8 sizes scaled to 148 SMs, slowdown matrix, SUM, R=14."""
    models = library_models(seed=3)
    rng = np.random.default_rng(SEED_BASE + 3)
    ids = [int(x) for x in rng.choice(len(models), size=4, replace=False)]
    M = _matrix(rng, 4) if mode == "matrix" else None
    return Problem("C3", models, ids, 148, 14, mode, "sum", slowdown_matrix=M,
                   p_idle_w=200.0, p_max_w=1000.0)


def make_c4(seed: int = 0) -> Problem:
    """C4: 8 models x 64 groups x 10 sizes, N=148, R=14, 3x QoS.  Composition 1 heavy
    (VGG-like) + 7 low-right-size (ShuffleNet/DenseNet-like), SURVEY.md §8(d)
    "C4 feasibility" (pairing high and low right-sizes as the paper did)."""
    sizes = lattice_sizes(10, 148)
    s = SEED_BASE + 4 + 1000 * seed
    fams = ["vgg"] + ["shufflenet", "densenet"] * 3 + ["shufflenet"]
    models = [synthesize_model(f"c4_{i}_{f}", f, 64, sizes, s + i) for i, f in enumerate(fams)]
    ids = list(range(8))
    return Problem("C4", models, ids, 148, 14, "exclude_self", "sum",
                   qos_ns=qos_3x(models, ids), p_idle_w=200.0, p_max_w=1000.0)


def make_c5(n_mixes: int = 4096, seed: int = 0, W: int = 4) -> tuple:
    """C5: batched planning, n_mixes x (W draws with replacement from the 7-model
    library) x 16 groups x 8 sizes, N=148, R=14, EXCLUDE_SELF, SUM, 3x QoS.
    Returns (library models, mix model ids [n_mixes, W] int32, qos [n_mixes, W])."""
    models = library_models(seed=5)
    rng = np.random.default_rng(SEED_BASE + 5 + 1000 * seed)
    ids = rng.integers(0, len(models), size=(n_mixes, W)).astype(np.int32)
    solo = np.array([qos_3x(models, [m])[0] for m in range(len(models))])
    qos = solo[ids]
    return models, ids, qos


def make_s6() -> Problem:
    """S6 (scaling extra): 6 x 16 x 8, N=148, R=14, no QoS."""
    models = library_models(seed=6)
    ids = [0, 1, 3, 4, 5, 2]
    return Problem("S6", models, ids, 148, 14, "exclude_self", "sum",
                   p_idle_w=200.0, p_max_w=1000.0)


def random_tiny_problem(seed: int, max_w: int = 3, max_g: int = 3, max_c: int = 4) -> Problem:
    """Random tiny instance for brute-force cross-checks (SURVEY.md §8(c) c6 "reduction")."""
    rng = np.random.default_rng(SEED_BASE + 77 + seed)
    W = int(rng.integers(1, max_w + 1))
    C = int(rng.integers(2, max_c + 1))
    if rng.random() < 0.6:
        sizes = lattice_sizes(C, 60)
        N = 60
    else:
        sizes = sorted(int(x) for x in rng.choice(np.arange(1, 41), size=C, replace=False))
        N = int(rng.integers(sizes[-1], 2 * sizes[-1] + 1))
    fams = list(("uniform", "vgg", "shufflenet", "bert", "densenet"))
    n_models = int(rng.integers(1, W + 1))
    models = []
    for i in range(n_models):
        K = int(rng.integers(1, max_g + 1))
        if rng.random() < 0.3:
            K += int(rng.integers(0, 2))
        models.append(synthesize_model(f"t{i}", fams[int(rng.integers(len(fams)))], K, sizes,
                                       SEED_BASE + 5000 + 31 * seed + i))
        if rng.random() < 0.25:  # coarse, tie-prone values
            models[-1].exec_ns = (models[-1].exec_ns // 10000 + 1) * 10000
            for k in range(K):
                for j in range(C - 1, 0, -1):
                    models[-1].exec_ns[k, j - 1] = max(models[-1].exec_ns[k, j - 1],
                                                       models[-1].exec_ns[k, j])
    ids = [int(rng.integers(0, n_models)) for _ in range(W)]
    gb = None
    if rng.random() < 0.3:
        gb = []
        for w in range(W):
            K = models[ids[w]].n_kernels
            if K >= 2 and rng.random() < 0.7:
                cut = sorted(set(int(x) for x in rng.choice(np.arange(1, K), size=int(rng.integers(1, K)), replace=False)))
                gb.append([0] + cut + [K])
            else:
                gb.append(None)
    mask = None
    if rng.random() < 0.4:
        mask = []
        for w in range(W):
            m = int(rng.integers(1, 1 << C))
            mask.append(m)
    mode = MODES[int(rng.integers(0, 4))]
    obj = OBJECTIVES[int(rng.integers(0, 3))]
    M = _matrix(rng, W) if mode == "matrix" else None
    qos = None
    if rng.random() < 0.5:
        qos = qos_3x(models, ids, factor=float(rng.choice([1.2, 1.6, 2.0, 3.0])), masks=mask)
        if rng.random() < 0.3:
            qos[int(rng.integers(0, W))] = float("inf")
    R = int(rng.integers(0, 4))
    return Problem(f"tiny{seed}", models, ids, N, R, mode, obj, allowed_mask=mask,
                   qos_ns=qos, slowdown_matrix=M, group_bounds=gb,
                   p_idle_w=float(rng.choice([75.0, 200.0])), p_max_w=float(rng.choice([225.0, 1000.0])))


def c5_problem(i: int, models, ids, qos) -> Problem:
    """Mix i of a C5 batch as a single Problem (for oracle checks of sampled mixes)."""
    return Problem(f"C5[{i}]", models, [int(x) for x in ids[i]], 148, 14, "exclude_self", "sum",
                   qos_ns=[float(x) for x in qos[i]], p_idle_w=200.0, p_max_w=1000.0)


def problem_hash(p: Problem) -> str:
    """Hash of a problem's seeded inputs (detects stale golden files)."""
    import hashlib
    import json
    h = hashlib.sha256()
    for m in p.models:
        h.update(np.ascontiguousarray(m.exec_ns).tobytes())
        h.update(str(m.sizes).encode())
    h.update(json.dumps([list(map(int, p.model_ids)), p.total_sms, p.switch_max, p.mode, p.objective,
                         p.allowed_mask, p.qos_ns, p.group_bounds, p.p_idle_w, p.p_max_w]).encode())
    if p.slowdown_matrix is not None:
        h.update(np.ascontiguousarray(p.slowdown_matrix, dtype=np.float32).tobytes())
    if p.weights is not None:
        h.update(json.dumps([float(x) for x in p.weights]).encode())
    return h.hexdigest()[:16]
