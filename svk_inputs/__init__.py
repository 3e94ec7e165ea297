"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic: it only knows the vector
lengths of the documented compact layout and draws seeded random numbers
(numpy PCG64 via ``default_rng``), so both sides of a parity test see
identical bits.  Problem data with physical meaning (manufactured right-hand
sides, boundary values) are computed by each side itself.

Compact layout on a level with N elements per side (both sides agree on it):
``[u_x ((2N+1)^2, x fastest), u_y ((2N+1)^2), p ((N+1)^2)]``.
"""
from __future__ import annotations

import numpy as np


def compact_len(N: int) -> int:
    """Length of a compact vector: 2 (2N+1)^2 + (N+1)^2."""
    return 2 * (2 * N + 1) ** 2 + (N + 1) ** 2


def random_vector(N: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """Standard-normal entries on every slot of a compact level-N vector."""
    rng = np.random.default_rng(seed)
    return scale * rng.standard_normal(compact_len(N))


def random_sample_indices(N: int, seed: int, count: int) -> np.ndarray:
    """Distinct, sorted sample positions in a compact level-N vector."""
    rng = np.random.default_rng(seed)
    n = compact_len(N)
    count = min(count, n)
    return np.sort(rng.choice(n, size=count, replace=False)).astype(np.int64)
