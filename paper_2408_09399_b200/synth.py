"""Seeded synthetic workloads for the five BASELINE.json configs.

These stand in for the paper's UCR archive workloads: clustered
time series in the same regime (n up to tens of thousands, L 64-512) feeding the same
Pearson -> sort -> TMFG -> APSP -> DBHT path.  Every array comes from one
``np.random.default_rng(seed)`` stream, so the same (config, seed) gives the same
bytes on any host.  This is workload plumbing, not part of the accelerated path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DEFAULT_SEED = 20240817


@dataclass(frozen=True)
class SynthConfig:
    """One BASELINE.json config: n series of length L and the APSP modes run on it."""

    index: int
    n: int
    length: int
    apsp_modes: tuple
    description: str


CONFIGS = {
    1: SynthConfig(1, 500, 128, ("exact", "hub"),
                   "5 equal clusters, random-walk prototypes + N(0,0.5^2), z-normalised"),
    2: SynthConfig(2, 2000, 256, ("exact", "hub"),
                   "10 equal clusters, random-walk prototypes + N(0,1), z-normalised"),
    3: SynthConfig(3, 10000, 512, ("hub",),
                   "20 Dirichlet(1) clusters (min 10), N(0,1) x U(0.5,2) noise, z-normalised"),
    4: SynthConfig(4, 4000, 64, ("exact", "hub"),
                   "tie stress: 8 integer prototypes in {-3..3}, 30% positions redrawn, raw"),
    5: SynthConfig(5, 50000, 256, ("hub",),
                   "50 Dirichlet(1) clusters (min 10), N(0,1) noise, 5% pure noise, z-normalised"),
}


def _znorm(x: np.ndarray) -> np.ndarray:
    mu = x.mean(axis=1, keepdims=True)
    sd = x.std(axis=1, keepdims=True)  # population std (ddof=0)
    sd[sd == 0.0] = 1.0
    return (x - mu) / sd


def _dirichlet_sizes(rng, n: int, k: int, minimum: int) -> np.ndarray:
    p = rng.dirichlet(np.ones(k))
    return minimum + rng.multinomial(n - minimum * k, p)


def _walks(rng, k: int, length: int) -> np.ndarray:
    return np.cumsum(rng.standard_normal((k, length)), axis=1)


def generate(config: int, seed: int = DEFAULT_SEED, n: int | None = None):
    """Series (n, L) float64 and labels (n,) int64 for a BASELINE config.

    ``n`` optionally shrinks the config (same recipe, fewer series) for tests.
    Series are shuffled so clusters are not contiguous id ranges.
    """
    cfg = CONFIGS[config]
    n = cfg.n if n is None else int(n)
    L = cfg.length
    rng = np.random.default_rng(seed + 1000 * config)
    if config in (1, 2):
        k = 5 if config == 1 else 10
        sigma = 0.5 if config == 1 else 1.0
        sizes = np.full(k, n // k)
        sizes[: n - sizes.sum()] += 1
        protos = _walks(rng, k, L)
        labels = np.repeat(np.arange(k), sizes)
        x = protos[labels] + sigma * rng.standard_normal((n, L))
        x = _znorm(x)
    elif config == 3:
        k = 20
        sizes = _dirichlet_sizes(rng, n, k, min(10, n // k))
        protos = _walks(rng, k, L)
        labels = np.repeat(np.arange(k), sizes)
        amp = rng.uniform(0.5, 2.0, size=(n, 1))
        x = protos[labels] + amp * rng.standard_normal((n, L))
        x = _znorm(x)
    elif config == 4:
        k = 8
        sizes = np.full(k, n // k)
        sizes[: n - sizes.sum()] += 1
        protos = rng.integers(-3, 4, size=(k, L)).astype(np.float64)
        labels = np.repeat(np.arange(k), sizes)
        x = protos[labels].copy()
        redraw = rng.random((n, L)) < 0.3
        x[redraw] = rng.integers(-3, 4, size=int(redraw.sum())).astype(np.float64)
    elif config == 5:
        k = 50
        sizes = _dirichlet_sizes(rng, n, k, min(10, n // k))
        protos = _walks(rng, k, L)
        labels = np.repeat(np.arange(k), sizes)
        x = protos[labels] + rng.standard_normal((n, L))
        noisy = rng.random(n) < 0.05
        x[noisy] = rng.standard_normal((int(noisy.sum()), L))
        x = _znorm(x)
    else:
        raise ValueError(f"unknown config {config}")
    perm = rng.permutation(n)
    return np.ascontiguousarray(x[perm]), labels[perm].astype(np.int64)


def num_clusters(config: int) -> int:
    return {1: 5, 2: 10, 3: 20, 4: 8, 5: 50}[config]


# --- small similarity matrices in the style of the reference's test fixtures ---
# (the reference's conftest.py:11-26 builds the same kinds of matrices)

def uniform_matrix(n: int, seed: int) -> np.ndarray:
    """Symmetric, iid-uniform off-diagonal, unit diagonal."""
    rng = np.random.default_rng(seed)
    A = rng.random((n, n))
    S = (A + A.T) / 2.0
    np.fill_diagonal(S, 1.0)
    return S


def quantized_matrix(n: int, seed: int, levels: int = 4) -> np.ndarray:
    """Few distinct values: every row is full of exact ties."""
    rng = np.random.default_rng(seed)
    A = rng.integers(0, levels, size=(n, n)) / levels
    S = np.minimum(A, A.T).astype(np.float64)
    np.fill_diagonal(S, 1.0)
    return S
