"""The BASELINE.json workloads C1..C5 as seeded host generators (bands, grids, samples).

BASELINE.json names no public dataset; these seeded synthetic matrices *are* the benchmark
(SURVEY.md §8d). Spec gaps are resolved as recorded in DESIGN.md §Configs:
  * C3 coefficient scale 1/(k+1) is undefined at k = -1 -> 1/(|k|+1);
  * complex N(0,1) is (N + iN)/sqrt(2);
  * seeds: mix64(PAPER_SEED, config) with the reference splitting rule (generate.py:27-34),
    drawn with numpy PCG64 as in generate.py:102;
  * grid boxes for C3/C5 are the eigenvalue bounding boxes padded by 1.0, precomputed by
    oracle/make_golden.py (dense eigvals) and frozen here so the GPU box needs no O(n^3) step;
    C4 covers the convection-diffusion ellipse/parabola (bounds below).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import BandMatrix, ComplexGrid, make_grid

_MASK64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
PAPER_SEED = 260504550


def mix64(seed: int, index: int) -> int:
    """splitmix64 child seed (restates pseudospec/generate.py:27-34)."""
    z = (int(seed) + (int(index) + 1) * _GOLDEN) & _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return (z ^ (z >> 31)) & _MASK64


def _cn(rng, size=None):
    return (rng.standard_normal(size) + 1j * rng.standard_normal(size)) / np.sqrt(2.0)


def grcar_band(n: int, k: int = 3) -> BandMatrix:
    """Grcar matrix: subdiagonal -1, main diagonal and k superdiagonals +1."""
    band = np.zeros((k + 2, n), dtype=complex)
    band[0, 1:] = -1.0          # d = -1 : A[i, i-1]
    band[1:, :] = 1.0           # d = 0..k
    return BandMatrix(band, 1, k)


def toeplitz_c3_band(n: int = 1000, seed: int | None = None) -> BandMatrix:
    """C3: Toeplitz, c_k ~ CN(0,1)/(|k|+1) on offsets k = -2..3."""
    seed = mix64(PAPER_SEED, 3) if seed is None else seed
    rng = np.random.default_rng(np.random.PCG64(seed))
    kl, ku = 2, 3
    band = np.zeros((kl + ku + 1, n), dtype=complex)
    for d in range(-kl, ku + 1):
        band[d + kl, :] = _cn(rng) / (abs(d) + 1)
    return BandMatrix(band, kl, ku)


def convdiff_band(n: int = 2000, pe: float = 50.0) -> BandMatrix:
    """C4: centered FD of u'' + Pe u' on n interior points, h = 1/(n+1) (real entries)."""
    h = 1.0 / (n + 1)
    band = np.zeros((3, n), dtype=complex)
    band[0, :] = 1.0 / h**2 - pe / (2 * h)   # A[i, i-1]
    band[1, :] = -2.0 / h**2
    band[2, :] = 1.0 / h**2 + pe / (2 * h)   # A[i, i+1]
    return BandMatrix(band, 1, 1)


def c5_band(index: int, n: int = 4000, seed: int | None = None) -> BandMatrix:
    """C5 matrix `index` of 64: Toeplitz band CN(0,1) scaled 4.0 (upper) / 1.0 (diag) /
    0.25 (lower), plus 1e-3 CN(0,1) i.i.d. noise on every band entry."""
    seed = mix64(PAPER_SEED, 5) if seed is None else seed
    rng = np.random.default_rng(np.random.PCG64(mix64(seed, index)))
    kl = ku = 3
    band = np.zeros((kl + ku + 1, n), dtype=complex)
    for d in range(-kl, ku + 1):
        scale = 4.0 if d > 0 else (0.25 if d < 0 else 1.0)
        band[d + kl, :] = _cn(rng) * scale + 1e-3 * _cn(rng, n)
    return BandMatrix(band, kl, ku)


# Frozen grid boxes (see module docstring). C3/C5 values are written by oracle/make_golden.py.
C3_BOX = (-1.3120622297077658, 2.8202251704993175, -1.5441211819491594, 3.333362897155037)
C5_BOX = (-4.588273233499905, 6.7666325650326264, -6.490070062540546, 3.9341982302654523)
_H4 = 1.0 / 2001
C4_BOX = (-4.2 / _H4**2, 0.2 / _H4**2, -1.1e5, 1.1e5)


@dataclass(frozen=True)
class Config:
    name: str
    description: str
    grid: ComplexGrid
    batch: int = 1

    def matrix(self, index: int = 0) -> BandMatrix:
        return _MATRIX[self.name](index)


_MATRIX = {
    "C1": lambda i: grcar_band(100),
    "C2": lambda i: grcar_band(400),
    "C3": lambda i: toeplitz_c3_band(1000),
    "C4": lambda i: convdiff_band(2000),
    "C5": lambda i: c5_band(i, 4000),
}

CONFIGS = {
    "C1": Config("C1", "Grcar n=100, 50x50 over [-1,3]x[-3.5,3.5]", make_grid(-1, 3, -3.5, 3.5, 50, 50)),
    "C2": Config("C2", "Grcar n=400, 200x200 over [-1,3]x[-3.5,3.5]", make_grid(-1, 3, -3.5, 3.5, 200, 200)),
    "C3": Config("C3", "complex banded Toeplitz n=1000 (2,3), 256x256 over eig bbox + 1",
                 make_grid(*C3_BOX, 256, 256)),
    "C4": Config("C4", "convection-diffusion n=2000 Pe=50 (1,1), 512x512", make_grid(*C4_BOX, 512, 512)),
    "C5": Config("C5", "64 x complex banded n=4000 (3,3), 1024x1024 each", make_grid(*C5_BOX, 1024, 1024),
                 batch=64),
}


def sample_points(cfg: Config, count: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Seeded random subset of grid indices (row-major) and their z values."""
    rng = np.random.default_rng(np.random.PCG64(seed))
    N = cfg.grid.size
    idx = np.sort(rng.choice(N, size=min(count, N), replace=False))
    return idx, cfg.grid.points().ravel()[idx]
