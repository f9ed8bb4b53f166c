"""Seeded synthetic stand-ins for BASELINE.json's five configs.

The paper's real datasets (sj2, mockgalaxy, bio5, pall7)
are not available; these generators follow SURVEY.md Appendix C, which fixes
every choice BASELINE.json leaves open.  All data is float64 from
``numpy.random.default_rng(seed)`` with seed = 1000 + config index.  The
reference has no Silverman rule and no Student-t generator; both are the
builder's (Appendix C).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def silverman(points: np.ndarray) -> float:
    """h_S = mean_d std_d(ddof=1) * (4 / ((D+2) N))^(1/(D+4))."""
    n, d = points.shape
    sigma = float(np.mean(np.std(points, axis=0, ddof=1)))
    return sigma * (4.0 / ((d + 2) * n)) ** (1.0 / (d + 4))


@dataclass
class Workload:
    name: str
    dim: int
    references: np.ndarray
    weights: np.ndarray
    queries: np.ndarray | None  # None = monochromatic (queries are the references)
    bandwidths: list
    epsilon: float
    h_star: float
    notes: dict = field(default_factory=dict)

    @property
    def monochromatic(self) -> bool:
        return self.queries is None

    @property
    def m(self) -> int:
        return self.references.shape[0] if self.queries is None else self.queries.shape[0]

    @property
    def n(self) -> int:
        return self.references.shape[0]

    def query_points(self) -> np.ndarray:
        return self.references if self.queries is None else self.queries


def _gmm(rng, n, dim, k, sigma_lo, sigma_hi, anisotropic=False):
    means = rng.uniform(0.0, 1.0, (k, dim))
    if anisotropic:
        sig = rng.uniform(sigma_lo, sigma_hi, (k, dim))
    else:
        sig = np.repeat(rng.uniform(sigma_lo, sigma_hi, (k, 1)), dim, axis=1)
    lab = rng.integers(0, k, n)
    return means[lab] + sig[lab] * rng.standard_normal((n, dim))


def config(index: int, scale: float = 1.0) -> Workload:
    """Config `index` (1..5).  `scale` < 1 shrinks N (parity tests only)."""
    rng = np.random.default_rng(1000 + index)
    if index == 1:
        n = max(2, int(10_000 * scale))
        means = rng.uniform(0.0, 1.0, (4, 2))
        refs = means[rng.integers(0, 4, n)] + 0.05 * rng.standard_normal((n, 2))
        qs = means[rng.integers(0, 4, n)] + 0.05 * rng.standard_normal((n, 2))
        w = np.full(n, 1.0 / n)
        return Workload("C1", 2, refs, w, qs, [0.05], 0.01, 0.05,
                        {"mode": "bichromatic", "weights": "1/N"})
    if index == 2:
        n = max(2, int(100_000 * scale))
        refs = _gmm(rng, n, 3, 10, 0.01, 0.1)
        w = np.full(n, 1.0 / n)
        hs = silverman(refs)
        bws = [hs * 10.0 ** (-3 + 5 * j / 9) for j in range(10)]
        return Workload("C2", 3, refs, w, None, bws, 0.01, hs,
                        {"mode": "monochromatic", "weights": "1/N"})
    if index == 3:
        n = max(2, int(200_000 * scale))
        nc = int(round(0.8 * n))
        refs = np.concatenate([_gmm(rng, nc, 5, 20, 0.01, 0.1, anisotropic=True),
                               rng.uniform(0.0, 1.0, (n - nc, 5))])
        w = np.full(n, 1.0 / n)
        hs = silverman(refs)
        bws = [hs * 10.0 ** (-2 + 3 * j / 6) for j in range(7)]
        return Workload("C3", 5, refs, w, None, bws, 0.01, hs,
                        {"mode": "monochromatic", "weights": "1/N",
                         "anisotropic_sigma": "U[0.01,0.1] per (component, dim)"})
    if index == 4:
        n = max(2, int(500_000 * scale))
        s = rng.uniform(0.5, 2.0, 7)
        refs = s * rng.standard_t(3.0, (n, 7))
        w = np.ones(n)
        hs = silverman(refs)
        base = [hs * 10.0 ** (-2 + 3 * j / 9) for j in range(10)]
        bws = []
        for h in base:
            bws += [h, float(np.sqrt(2.0)) * h]
        return Workload("C4", 7, refs, w, None, bws, 0.01, hs,
                        {"mode": "monochromatic", "weights": "1 (LSCV)",
                         "lscv_bandwidths": base})
    if index == 5:
        n = max(2, int(4_000_000 * scale))
        nc = int(round(0.9 * n))
        refs = np.concatenate([_gmm(rng, nc, 3, 50, 0.01, 0.1),
                               rng.uniform(0.0, 1.0, (n - nc, 3))])
        w = rng.uniform(0.5, 1.5, n)
        w /= w.sum()
        hs = silverman(refs)
        bws = [hs * 10.0 ** (-3 + 5 * j / 15) for j in range(16)]
        return Workload("C5", 3, refs, w, None, bws, 0.001, hs,
                        {"mode": "monochromatic", "weights": "U[0.5,1.5] normalised"})
    raise ValueError("config index must be 1..5")
