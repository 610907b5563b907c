"""Synthetic cuSZ-style quantization-code fields (the bench workloads).

The reference ships no cuSZ-shaped generator (its ``synth_codes`` is a
two-sided geometric around 32768, quant.py:77-96), so the workloads follow
SURVEY.md §8(d): codes = clip(rint(N(0, sigma)) + bins/2, 0, bins-1) drawn with
``numpy.random.default_rng(seed)``; with probability ``eps`` a code is instead
drawn uniformly from [0, bins) so the whole codebook is populated.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class FieldSpec:
    name: str
    n: int
    bins: int
    sigma: float
    eps: float = 0.0
    seed: int = 0

    @property
    def decoded_bytes(self) -> int:
        return 2 * self.n


# Calibrations from SURVEY.md §8(d) (measured CR in parentheses there).
FIELDS = {
    "1m": FieldSpec("synthetic-1M", 1 << 20, 1024, 3.0),
    "hurricane": FieldSpec("hurricane-100x500x500", 100 * 500 * 500, 1024, 0.6),
    "nyx": FieldSpec("nyx-512^3", 512 ** 3, 1024, 0.2, 1e-3),
    "nyx256": FieldSpec("nyx-512^3-bins256", 512 ** 3, 256, 0.2, 1e-3),
    "nyx4096": FieldSpec("nyx-512^3-bins4096", 512 ** 3, 4096, 0.2, 1e-3),
    "hacc": FieldSpec("hacc-280953867", 280_953_867, 1024, 8.0),
    "cesm": FieldSpec("cesm-26x1800x3600", 26 * 1800 * 3600, 1024, 0.6),
    "rtm": FieldSpec("rtm-449x449x235", 449 * 449 * 235, 1024, 0.8),
    "qmcpack": FieldSpec("qmcpack-115x69x69x288", 115 * 69 * 69 * 288, 1024, 22.0),
}


def gaussian_codes(n: int, bins: int, sigma: float, eps: float = 0.0, seed: int = 0,
                   chunk: int = 1 << 24) -> np.ndarray:
    """Deterministic quantization codes of one field (chunked to bound memory)."""
    rng = np.random.default_rng(seed)
    out = np.empty(n, dtype=np.uint16)
    half = bins // 2
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        g = np.rint(rng.normal(0.0, sigma, hi - lo))
        c = np.clip(g + half, 0, bins - 1)
        if eps > 0:
            m = rng.random(hi - lo) < eps
            c[m] = rng.integers(0, bins, int(m.sum()))
        out[lo:hi] = c.astype(np.uint16)
    return out


def field_codes(spec: FieldSpec, n: int | None = None) -> np.ndarray:
    return gaussian_codes(spec.n if n is None else n, spec.bins, spec.sigma, spec.eps, spec.seed)
