"""Seeded synthetic inputs, bit-identical to the CUDA generator ops.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  SURVEY.md §8d: element
(I, J) of an n-column matrix is ``u(seed, I*n + J)`` with

    z = seed * 0x9E3779B97F4A7C15 + g         (mod 2^64)
    z = splitmix64_finalise(z + 0x9E3779B97F4A7C15)
    u = (z >> 11) * 2^-53                      in [0, 1)

The same arithmetic is in paper_2308_15964_b200/csrc/kernels/misc.cu, so a
tile generated on the GPU equals the oracle's bit for bit, independent of the
tiling.
"""

from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def splitmix_uniform(seed: int, g) -> np.ndarray:
    g = np.asarray(g, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) * GOLDEN + g
        z = z + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_tile(seed: int, row0: int, col0: int, rows: int, cols: int, ncols_total: int) -> np.ndarray:
    I = np.arange(row0, row0 + rows, dtype=np.uint64)[:, None]
    J = np.arange(col0, col0 + cols, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        g = I * np.uint64(ncols_total) + J
    return splitmix_uniform(seed, g)


def spd_tile(seed: int, row0: int, col0: int, rows: int, cols: int, n: int) -> np.ndarray:
    """Tile of A = (R + R^T)/2 + n*I, R uniform[0,1) (SPD by diagonal dominance)."""
    I = np.arange(row0, row0 + rows, dtype=np.uint64)[:, None]
    J = np.arange(col0, col0 + cols, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        u1 = splitmix_uniform(seed, I * np.uint64(n) + J)
        u2 = splitmix_uniform(seed, J * np.uint64(n) + I)
    a = (u1 + u2) * 0.5
    d = (I == J)
    a = a + np.where(d, float(n), 0.0)
    return a


def particles(seed: int, first: int, n: int) -> np.ndarray:
    """4 x n SoA block (x, y, z in [0,1), q in [0.5, 1)) of particles first..first+n-1."""
    g = (np.arange(first, first + n, dtype=np.uint64) * np.uint64(4))[None, :] + np.arange(4, dtype=np.uint64)[:, None]
    u = splitmix_uniform(seed, g)
    u[3] = 0.5 + 0.5 * u[3]
    return u
