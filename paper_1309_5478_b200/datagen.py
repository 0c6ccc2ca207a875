"""Seeded synthetic inputs shared by the tests, the bench and the oracle runs.

This module holds NO arithmetic of the method (no distances, norms or selection): it
only draws random fp32 matrices, so that the CUDA path and the CPU oracle can be fed
identical bytes.  Recipe:

* generator: numpy ``Generator(Philox(seed))``, fp32, base seed 1309000 + config no.;
* ``uniform``  — U[0, 1) entries, the paper's "matrix ... of uniformly random floating
  point numbers";
* ``gauss``    — N(0, 1) entries;
* ``clusters`` — 64 centres ~ N(0, I_d), points = centre + 0.1 N(0, I_d), uniform
  random centre assignment (a clustered workload; the paper gives none — builder's
  choice);
* ``grid``     — integers in {-4, ..., 4}: every norm and dot product is an integer
  < 2^24, so all correct implementations agree bit-exactly (E2E-3).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

BASE_SEED = 1309000


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def points(n: int, d: int, dist: str = "uniform", seed: int = BASE_SEED) -> np.ndarray:
    """n×d fp32 row-major (vector-contiguous) points."""
    g = rng(seed)
    if dist == "uniform":
        return g.random((n, d), dtype=np.float32)
    if dist == "gauss":
        return g.standard_normal((n, d), dtype=np.float32)
    if dist == "clusters":
        centres = g.standard_normal((64, d), dtype=np.float32)
        assign = g.integers(0, 64, size=n)
        noise = g.standard_normal((n, d), dtype=np.float32)
        return (centres[assign] + np.float32(0.1) * noise).astype(np.float32)
    if dist == "grid":
        return g.integers(-4, 5, size=(n, d)).astype(np.float32)
    raise ValueError(f"unknown distribution {dist!r}")


def keys(m: int, n: int, kind: str = "uniform", seed: int = BASE_SEED + 100) -> np.ndarray:
    """m×n fp32 key matrices for select-only tests (PAPER.md:88 uniform random keys)."""
    g = rng(seed)
    if kind == "uniform":
        return g.random((m, n), dtype=np.float32)
    if kind == "dup256":  # duplicate-heavy: 256 distinct levels
        return (g.integers(0, 256, size=(m, n)).astype(np.float32) / np.float32(256))
    if kind == "descending":  # adversarial for a running threshold
        base = np.arange(n, 0, -1, dtype=np.float32)[None, :]
        return np.repeat(base, m, axis=0) + g.random((m, 1), dtype=np.float32)
    if kind == "ascending":
        base = np.arange(n, dtype=np.float32)[None, :]
        return np.repeat(base, m, axis=0)
    if kind == "equal":
        return np.full((m, n), 0.5, np.float32)
    raise ValueError(f"unknown key kind {kind!r}")


@dataclass(frozen=True)
class Config:
    name: str
    mode: str        # "graph" (k-NNG, queries = corpus) or "search"
    N: int           # corpus points
    M: int           # queries (== N for graph)
    d: int
    k: int
    dist: str
    seed: int
    sharding: str    # how BASELINE.json distributes it over GPUs


# BASELINE.json "configs", in file order (C1..C5).
CONFIGS = {
    "C1": Config("C1", "graph", 1024, 1024, 32, 8, "uniform", BASE_SEED + 1, "single"),
    "C2": Config("C2", "graph", 16384, 16384, 128, 16, "clusters", BASE_SEED + 2, "single"),
    "C3": Config("C3", "search", 65536, 65536, 256, 32, "uniform", BASE_SEED + 3, "query"),
    "C4": Config("C4", "graph", 32768, 32768, 1024, 1024, "uniform", BASE_SEED + 4, "query"),
    "C5": Config("C5", "graph", 131072, 131072, 256, 32, "gauss", BASE_SEED + 5, "corpus"),
}
# The headline metric's workload (BASELINE.json "metric"): k-NNG at N=65536, d=256, k=32.
HEADLINE = Config("H", "graph", 65536, 65536, 256, 32, "uniform", BASE_SEED + 3, "query")


def config_inputs(cfg: Config):
    """(Q, X) for a config; Q is X for graph mode."""
    X = points(cfg.N, cfg.d, cfg.dist, cfg.seed)
    if cfg.mode == "graph":
        return X, X
    Q = points(cfg.M, cfg.d, cfg.dist, cfg.seed + 1000)
    return Q, X
