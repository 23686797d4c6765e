"""Synthetic edge streams of the BASELINE.json shapes.

Input data for tests and bench.py -- not part of the compute path.  Numpy
(seeded Generator) so the CPU oracle and the GPU see identical arrays.

dcsbm: degree-corrected planted partition.  Node weights are Pareto with
exponent gamma (capped at wmax), nodes are assigned uniformly to k blocks;
a fraction 1-mu of the m draws picks a block with probability proportional
to its weight mass and both endpoints proportional to weight inside it, the
rest pick both endpoints proportional to weight globally.  Self-loops are
dropped, duplicates kept, stream order uniformly shuffled.
"""

from __future__ import annotations

import numpy as np

CONFIGS = {
    # name: (n, m, gamma, k) -- BASELINE.json configs, SURVEY.md 8d table
    "C1": dict(n=10_000, m=100_000, gamma=None, k=100),
    "C2": dict(n=335_000, m=926_000, gamma=2.5, k=3_350),
    "C3": dict(n=685_230, m=7_600_000, gamma=2.3, k=6_852),
    "C4": dict(n=3_000_000, m=34_000_000, gamma=2.3, k=30_000),
}


def dcsbm(n: int, m: int, k: int | None = None, gamma: float | None = 2.3, mu: float = 0.1,
          seed: int = 0, wmax: float = 64.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    k = k or max(1, n // 100)
    if gamma is None:
        w = np.ones(n)
    else:
        w = np.minimum((1.0 - rng.random(n)) ** (-1.0 / (gamma - 1.0)), wmax)
    block = rng.integers(0, k, size=n)
    order = np.argsort(block, kind="stable")          # nodes grouped by block
    cw = np.cumsum(w[order])
    bounds = np.searchsorted(block[order], np.arange(k + 1), side="left")
    base = np.concatenate([[0.0], cw])[bounds[:-1]]
    mass = np.concatenate([[0.0], cw])[bounds[1:]] - base
    total = cw[-1]

    def locate(r):  # r sorted-ish targets in [0, total) -> node ids
        return order[np.minimum(np.searchsorted(cw, r, side="right"), n - 1)]

    n_intra = int(rng.binomial(m, 1.0 - mu))
    counts = rng.multinomial(n_intra, mass / mass.sum())
    blk = np.repeat(np.arange(k), counts)             # grouped -> cache-friendly search
    u = locate(base[blk] + rng.random(n_intra) * mass[blk])
    v = locate(base[blk] + rng.random(n_intra) * mass[blk])
    n_inter = m - n_intra
    ug = locate(np.sort(rng.random(n_inter)) * total)
    vg = locate(np.sort(rng.random(n_inter)) * total)[rng.permutation(n_inter)]
    e = np.stack([np.concatenate([u, ug]), np.concatenate([v, vg])], axis=1).astype(np.int32)
    e = e[rng.permutation(m)]
    return e[e[:, 0] != e[:, 1]]


def planted_partition(n: int, m: int, k: int, mu: float = 0.1, seed: int = 0) -> np.ndarray:
    """Uniform-endpoint SBM (the survey's generator shape)."""
    return dcsbm(n, m, k=k, gamma=None, mu=mu, seed=seed)


def config_graph(name: str, seed: int = 0) -> np.ndarray:
    c = CONFIGS[name]
    return dcsbm(c["n"], c["m"], k=c["k"], gamma=c["gamma"], seed=seed)


def rmat_edges(scale: int, edge_factor: int, seed: int = 0,
               abcd=(0.57, 0.19, 0.19, 0.05)) -> np.ndarray:
    """R-MAT draws (C5 shape), self-loops dropped."""
    rng = np.random.default_rng(seed)
    m = edge_factor << scale
    a, b, c, _ = abcd
    u = np.zeros(m, dtype=np.int64)
    v = np.zeros(m, dtype=np.int64)
    for _ in range(scale):
        r = rng.random(m)
        ub = (r >= a + b).astype(np.int64)
        vb = (((r >= a) & (r < a + b)) | (r >= a + b + c)).astype(np.int64)
        u = (u << 1) | ub
        v = (v << 1) | vb
    e = np.stack([u, v], axis=1).astype(np.int32)
    return e[e[:, 0] != e[:, 1]]


RMAT_ABCD = (0.57, 0.19, 0.19, 0.05)
_PHI = np.uint64(0x9E3779B97F4A7C15)


def _splitmix64(x):
    x = x + _PHI
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def rmat_counter(scale: int, start: int, count: int, seed: int = 0,
                 abcd=RMAT_ABCD) -> np.ndarray:
    """Edges [start, start + count) of the counter-based R-MAT stream that
    cvz_rmat_edges generates on the device (self-loops kept), as a (count, 2)
    int32 array -- the host twin used by the tests."""
    a, b, c, _ = abcd
    k = np.arange(start, start + count, dtype=np.uint64)
    base = np.uint64((int(seed) * 0x9E3779B97F4A7C15) % (1 << 64))
    u = np.zeros(count, dtype=np.int64)
    v = np.zeros(count, dtype=np.int64)
    with np.errstate(over="ignore"):
        for lvl in range(scale):
            z = _splitmix64(base + k * np.uint64(64) + np.uint64(lvl))
            r = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
            ub = (r >= a + b).astype(np.int64)
            vb = (((r >= a) & (r < a + b)) | (r >= a + b + c)).astype(np.int64)
            u = (u << 1) | ub
            v = (v << 1) | vb
    return np.stack([u, v], axis=1).astype(np.int32)


def rmat_dev(scale: int, start: int, count: int, seed: int = 0, abcd=RMAT_ABCD):
    """Same stream generated in HBM (cvz_rmat_edges): a (count, 2) int32 CUDA
    tensor -- no host materialisation of a 2^30-edge input."""
    from . import _native as nat
    T = nat.torch()
    out = T.empty((max(count, 1), 2), dtype=T.int32, device=nat.device())
    a, b, c, _ = abcd
    nat.call("cvz_rmat_edges", int(scale), float(a), float(b), float(c), int(seed), int(start),
             int(count), nat.ptr(out), nat.stream())
    return out[:count]
