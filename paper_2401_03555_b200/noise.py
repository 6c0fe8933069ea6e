"""Noise models of the drop-in surface.

Diagonal Gaussian noise is the B200 hot path (BASELINE.json north_star:
"a product of erf differences for diagonal covariance").  The
full-covariance and custom-density models (reference noise.py:41-95) take
the Monte Carlo construction path: the same
k_refine with the Monte Carlo objective, numpy's Philox streams restated
on the device (csrc/rng.h).

`interval_probability` here is the host restatement used for tests and
host-side folding; the kernels use the cephes port in csrc/ndtr.h.
"""

import math
from dataclasses import dataclass

import numpy as np

from .errors import NoiseError
from .grid import Cell

__all__ = ["DiagonalNormal", "FullNormal", "CustomNoise", "box_probability",
           "interval_probability", "DEFAULT_MC_SAMPLES"]

DEFAULT_MC_SAMPLES = 10_000


@dataclass(frozen=True)
class DiagonalNormal:
    sigma: np.ndarray

    def __post_init__(self):
        s = np.asarray(self.sigma, dtype=float)
        object.__setattr__(self, "sigma", s)
        if s.ndim != 1 or not np.all(s > 0):
            raise NoiseError("sigma must be a vector of positive reals")

    @property
    def dim(self):
        return self.sigma.shape[0]


@dataclass(frozen=True)
class FullNormal:
    inv_cov: np.ndarray
    det: float
    samples: int = DEFAULT_MC_SAMPLES

    def __post_init__(self):
        m = np.asarray(self.inv_cov, dtype=float)
        object.__setattr__(self, "inv_cov", m)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise NoiseError("inv_cov must be a square matrix")
        if not np.allclose(m, m.T, rtol=0, atol=1e-12):
            raise NoiseError("inv_cov must be symmetric to 1e-12")
        for k in range(1, m.shape[0] + 1):
            if np.linalg.det(m[:k, :k]) <= 0:
                raise NoiseError("inv_cov must be positive definite "
                                 f"(leading minor {k} non-positive)")
        if not self.det > 0:
            raise NoiseError("det must be positive")
        if self.samples < 2:
            raise NoiseError("samples must be >= 2")

    @property
    def dim(self):
        return self.inv_cov.shape[0]


@dataclass(frozen=True)
class CustomNoise:
    density_expr: object
    dim: int
    samples: int = DEFAULT_MC_SAMPLES

    def __post_init__(self):
        if self.samples < 2:
            raise NoiseError("samples must be >= 2")


def _ndtr(z):
    z = np.asarray(z, dtype=float)
    return 0.5 * np.vectorize(math.erfc)(-z / math.sqrt(2.0))


def interval_probability(sigma, mean, lo, hi):
    """P(lo <= mean + N(0, sigma^2) <= hi), broadcasting (host helper)."""
    return _ndtr((np.asarray(hi) - mean) / sigma) - \
        _ndtr((np.asarray(lo) - mean) / sigma)


def box_probability(noise: DiagonalNormal, mean, cell: Cell) -> float:
    mean = np.asarray(mean, dtype=float)
    return float(np.prod(interval_probability(noise.sigma, mean, cell.lo,
                                              cell.hi)))
