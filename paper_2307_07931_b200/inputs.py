"""Seeded synthetic inputs shared by the tests, the oracle runs and the bench.

This module holds NONE of the method's arithmetic (no stencil, update or norm):
only the input fields of SURVEY.md §8(d) / DESIGN.md §4.

* ``hash_field`` -- counter-hash ρ ∈ [-1, 1): for the cell (i, j) of a domain of
  width ``n0``, ``u = splitmix64(seed XOR (i + j*n0))`` and
  ``ρ = ((u >> 11) * 2^-53) * 2 - 1`` (every step exact in fp64).  The device
  initialiser ``px_init_field(PX_FIELD_HASH, ...)`` implements the same
  counter-based generator independently, so the same cell gets the same bits
  on both sides whatever the decomposition.
* ``sine_field`` -- sin(kπx)·sin(lπy) sampled at cell centres x = (i+½)h
  (BASELINE.json configs 1, 5; wavenumber 2 gives the periodic fields of
  configs 2-4).
"""
from __future__ import annotations

import numpy as np

DEFAULT_SEED = 20230714

_M1 = np.uint64(0x9E3779B97F4A7C15)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser over uint64 (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (np.asarray(x, dtype=np.uint64) + _M1).astype(np.uint64)
        z = ((z ^ (z >> np.uint64(30))) * _M2).astype(np.uint64)
        z = ((z ^ (z >> np.uint64(27))) * _M3).astype(np.uint64)
        return z ^ (z >> np.uint64(31))


def hash_values(ix: np.ndarray, iy: np.ndarray, n0: int, seed: int = DEFAULT_SEED) -> np.ndarray:
    """ρ at global cells (ix, iy) of a domain of width n0 (coordinates in range)."""
    idx = np.asarray(ix, dtype=np.uint64) + np.asarray(iy, dtype=np.uint64) * np.uint64(n0)
    u = splitmix64(idx ^ np.uint64(seed))
    return ((u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) * 2.0 - 1.0


def hash_field(n0: int, n1: int, seed: int = DEFAULT_SEED) -> np.ndarray:
    """Full (n1, n0) interior field of the counter hash."""
    iy, ix = np.meshgrid(np.arange(n1, dtype=np.uint64), np.arange(n0, dtype=np.uint64),
                         indexing="ij")
    return hash_values(ix, iy, n0, seed)


def hash_window(n0: int, n1: int, x_lo: int, y_lo: int, wx: int, wy: int,
                seed: int = DEFAULT_SEED) -> np.ndarray:
    """(wy, wx) window of the periodic hash field starting at (x_lo, y_lo),
    coordinates wrapped modulo the domain."""
    xs = (np.arange(wx, dtype=np.int64) + x_lo) % n0
    ys = (np.arange(wy, dtype=np.int64) + y_lo) % n1
    iy, ix = np.meshgrid(ys, xs, indexing="ij")
    return hash_values(ix.astype(np.uint64), iy.astype(np.uint64), n0, seed)


def cell_centres(n: int) -> np.ndarray:
    h = 1.0 / n
    return (np.arange(n, dtype=np.float64) + 0.5) * h


def sine_field(n0: int, n1: int, k: int = 1, l: int = 1) -> np.ndarray:
    """sin(kπx) sin(lπy) at cell centres ((i+½)/n0, (j+½)/n1), shape (n1, n0)."""
    sx = np.sin(k * np.pi * cell_centres(n0))
    sy = np.sin(l * np.pi * cell_centres(n1))
    return np.outer(sy, sx)


def random_field(n0: int, n1: int, seed: int) -> np.ndarray:
    """Plain numpy-seeded uniform [-1, 1) field (for parity stress inputs)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, size=(n1, n0))


def hash_values3(ix, iy, iz, n0: int, n1: int, seed: int = DEFAULT_SEED) -> np.ndarray:
    """3D counter hash: ρ at global cells (ix, iy, iz) of an n0 x n1 x n2 domain,
    u = splitmix64(seed XOR (i + n0*(j + n1*k))) (the 2D recipe in 3D; the
    device initialiser px3_init_field implements it independently)."""
    idx = (np.asarray(ix, dtype=np.uint64) + np.uint64(n0) * (np.asarray(iy, dtype=np.uint64)
                                                              + np.uint64(n1) * np.asarray(iz, dtype=np.uint64)))
    u = splitmix64(idx ^ np.uint64(seed))
    return ((u >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) * 2.0 - 1.0


def hash_field3(n0: int, n1: int, n2: int, seed: int = DEFAULT_SEED) -> np.ndarray:
    """Full (n2, n1, n0) interior field of the 3D counter hash."""
    iz, iy, ix = np.meshgrid(np.arange(n2, dtype=np.uint64), np.arange(n1, dtype=np.uint64),
                             np.arange(n0, dtype=np.uint64), indexing="ij")
    return hash_values3(ix, iy, iz, n0, n1, seed)
