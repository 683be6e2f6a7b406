"""fmm_inputs.py — seeded synthetic workloads shared by the oracle tests and the CUDA path.

Holds none of the method's arithmetic: only the point/charge generators of
BASELINE.json ``configs`` (recipes in DESIGN.md "Inputs", after SURVEY.md
§8(d)). numpy ``default_rng`` (PCG64), seed 0 unless stated; the target
sample uses seed 12345. The paper's own §4.1 inputs are uniform lattices
 whose sizes live only in the missing Fig 2; these synthetic
sets stand in for them.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    dist: str  # "cube" | "plummer" | "sphere"
    p: int
    ncrit: int
    theta: float
    grad: bool
    index: int  # BASELINE.json configs[index]


CONFIGS = {
    "c1": Config("c1", 1_000, "cube", 4, 32, 0.4, True, 0),
    "c2": Config("c2", 100_000, "cube", 10, 64, 0.4, True, 1),
    "c3": Config("c3", 1_000_000, "cube", 10, 64, 0.4, False, 2),
    "c4": Config("c4", 10_000_000, "plummer", 8, 64, 0.5, False, 3),
    "c5": Config("c5", 100_000_000, "sphere", 12, 128, 0.4, False, 4),
    # NEXT-3: the paper's own §4.1 geometry, a uniform 3D lattice;
    # not a BASELINE config (index -1), sized like configs[2]
    "l3": Config("l3", 1_000_000, "lattice", 10, 64, 0.4, False, -1),
}


def cube(n: int, seed: int = 0):
    """configs[0..2]: uniform in [0,1)^3, charges uniform in [-1, 1]."""
    rng = np.random.default_rng(seed)
    x = rng.random((n, 3))
    q = rng.uniform(-1.0, 1.0, n)
    return x, q


def plummer(n: int, seed: int = 0):
    """configs[3]: Plummer sphere, scale radius 1, truncated at r = 100 by inverse CDF
    on [0, M(100)] (no rejection), isotropic directions, unit positive charges."""
    rng = np.random.default_rng(seed)
    mmax = 100.0**3 / (100.0**2 + 1.0) ** 1.5
    u = rng.random(n) * mmax
    r = 1.0 / np.sqrt(u ** (-2.0 / 3.0) - 1.0)
    z = rng.uniform(-1.0, 1.0, n)
    ph = rng.uniform(0.0, 2.0 * np.pi, n)
    s = np.sqrt(1.0 - z * z)
    x = np.c_[r * s * np.cos(ph), r * s * np.sin(ph), r * z]
    q = np.ones(n)
    return np.ascontiguousarray(x), q


def sphere(n: int, seed: int = 0):
    """configs[4]: uniform on the unit sphere surface, charges standard normal."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, 3))
    x = g / np.linalg.norm(g, axis=1)[:, None]
    q = rng.standard_normal(n)
    return np.ascontiguousarray(x), q


def lattice(n: int, seed: int = 0):
    """NEXT-3: the m^3 interior nodes of [-1,1]^3 (m = round(n^(1/3)), spacing 2/(m+1); the paper's
    §4.1 inputs are "uniform lattices", sizes unstated), charges uniform in [-1, 1].
    Returns m^3 points (n itself when n is a cube)."""
    m = max(1, int(round(n ** (1.0 / 3.0))))
    c = -1.0 + (np.arange(m) + 1.0) * (2.0 / (m + 1))
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    pts = np.stack([x.ravel(), y.ravel(), z.ravel()], 1)
    q = np.random.default_rng(seed).uniform(-1.0, 1.0, pts.shape[0])
    return np.ascontiguousarray(pts), q


GENERATORS = {"cube": cube, "plummer": plummer, "sphere": sphere, "lattice": lattice}


def make(dist: str, n: int, seed: int = 0):
    return GENERATORS[dist](n, seed)


def make_config(name: str, n: int | None = None, seed: int = 0):
    cfg = CONFIGS[name]
    return make(cfg.dist, cfg.n if n is None else n, seed)


def target_sample(n: int, k: int = 10_000, seed: int = 12345):
    """Sorted seeded sample of target indices."""
    k = min(k, n)
    return np.sort(np.random.default_rng(seed).choice(n, k, replace=False))


def rank_slice(n: int, rank: int, world: int):
    """Caller-side input distribution for world > 1: rows [floor(rN/P), floor((r+1)N/P))."""
    return (rank * n) // world, ((rank + 1) * n) // world
