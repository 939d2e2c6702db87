"""Min-entropy oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain float64 numpy, each function following one passage of the paper:

* H_min(x) = -log2 max_x P(x)                      PAPER.md:57-61 (Sec. II.A, Eq.)
* d_U(P1, P2) = 1/2 sum_{x in U} |P1(x) - P2(x)|   PAPER.md:155   (Sec. II.C)
* Delta H_m = log2( d_U / 2^{-N-1} + 1 )            PAPER.md:147-153 (Sec. II.C, Eq.)
* H_min^modify = H_min - Delta H_m
* m = n * H_min / N - 2 log2(1/eps)                 PAPER.md:185-187 (Sec. III.B, Eq.)

Readings:
A7/A23 m = floor(n*H/N) - s with integer s = 2 log2(1/eps);  A9 the correction is
applied to H_min of the ideal model P, H_min of the histogram is reported too;
A10 the ideal model is a Gaussian discretised on bins [k-1/2, k+1/2) with the
tails absorbed by the edge bins, mu and sigma fitted from the histogram
(population sigma) unless supplied; A11 d over the full domain (U = all 2^N
bins); A12 N in Delta H_m is the ADC bit depth; A13 no finite-size
amplification; A14 H_min^modify is floored at 0.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


def histogram(samples: np.ndarray, bit_depth: int = 8) -> np.ndarray:
    """Counts of each of the 2^N sample values (the empirical P'(x) times T)."""
    samples = np.asarray(samples)
    if samples.size and int(samples.max()) >= (1 << bit_depth):
        raise ValueError("sample outside [0, 2^N)")
    return np.bincount(samples.astype(np.int64), minlength=1 << bit_depth).astype(np.uint64)


def h_min(p: np.ndarray) -> float:
    """H_min = -log2 max P."""
    p = np.asarray(p, dtype=np.float64)
    return -math.log2(float(p.max()))


def h_min_counts(counts: np.ndarray) -> float:
    """Max-probability H_min of the empirical distribution P'(x) = counts / T."""
    counts = np.asarray(counts, dtype=np.float64)
    return -math.log2(float(counts.max()) / float(counts.sum()))


def fit_gauss(counts: np.ndarray) -> tuple[float, float]:
    """Sample mean and population sigma of the histogram (reading A10)."""
    c = np.asarray(counts, dtype=np.float64)
    k = np.arange(c.size, dtype=np.float64)
    t = c.sum()
    mu = float((k * c).sum() / t)
    var = float((k * k * c).sum() / t) - mu * mu
    return mu, math.sqrt(max(var, 0.0))


def _phi(z: float) -> float:
    return 0.5 * (1.0 + math.erf(z / math.sqrt(2.0)))


def ideal_gauss(mu: float, sigma: float, bit_depth: int = 8) -> np.ndarray:
    """Discretised N(mu, sigma^2): bin k = [k-1/2, k+1/2), edge bins take the tails."""
    if not sigma > 0:
        raise ValueError("sigma must be > 0")
    K = 1 << bit_depth
    cdf = np.array([_phi((k + 0.5 - mu) / sigma) for k in range(K - 1)], dtype=np.float64)
    p = np.empty(K, dtype=np.float64)
    p[0] = cdf[0]
    p[1:K - 1] = np.diff(cdf)
    p[K - 1] = 1.0 - cdf[K - 2]
    return p


def stat_distance(p1: np.ndarray, p2: np.ndarray) -> float:
    """d_U(P1, P2) = 1/2 sum |P1 - P2| over the full domain (A11)."""
    return 0.5 * float(np.abs(np.asarray(p1, np.float64) - np.asarray(p2, np.float64)).sum())


def delta_h_m(d: float, bit_depth: int) -> float:
    """Delta H_m = log2(d / 2^{-N-1} + 1)."""
    if not 0.0 <= d <= 1.0:
        raise ValueError("d outside [0, 1]")
    return math.log2(d / 2.0 ** (-bit_depth - 1) + 1.0)


def output_length(n: int, h: float, bit_depth: int, s: int) -> int:
    """m = floor(n * H / N) - s (readings A7/A23)."""
    return int(math.floor(n * h / bit_depth)) - int(s)


@dataclasses.dataclass
class EntropyReport:
    counts: np.ndarray
    n_samples: int
    bit_depth: int
    mu: float
    sigma: float
    h_min_hist: float
    h_min_ideal: float
    stat_dist: float
    delta_h_m: float
    h_min_mod: float
    m: int


def report_from_counts(counts: np.ndarray, bit_depth: int, n: int, s: int,
                       model: tuple[float, float] | None = None) -> EntropyReport:
    """The whole Sec. II.C -> Sec. III.B chain on one histogram."""
    counts = np.asarray(counts, dtype=np.uint64)
    total = int(counts.sum())
    K = 1 << bit_depth
    c = counts[:K]
    mu, sigma = model if model is not None else fit_gauss(c)
    p_ideal = ideal_gauss(mu, sigma, bit_depth)
    p_emp = c.astype(np.float64) / float(total)
    hi = h_min(p_ideal)
    d = stat_distance(p_emp, p_ideal)
    dh = delta_h_m(d, bit_depth)
    hmod = max(0.0, hi - dh)
    return EntropyReport(c.copy(), total, bit_depth, mu, sigma, h_min_counts(c), hi, d, dh,
                         hmod, output_length(n, hmod, bit_depth, s))


def report(samples: np.ndarray, bit_depth: int, n: int, s: int,
           model: tuple[float, float] | None = None) -> EntropyReport:
    return report_from_counts(histogram(samples, bit_depth), bit_depth, n, s, model)
