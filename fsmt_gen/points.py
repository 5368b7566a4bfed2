"""Seeded relaxed points (a, b) for parity tests and the bench (no method arithmetic).

Layout is restart-minor, matching the product's device layout: a[n_bool][R],
b[n_real][R], float32.  a ~ U(-1, 1); b ~ U(b_lo, b_hi) (the placement
coordinates live in [0, 1]; the other families use U(-1, 1)).
"""
from __future__ import annotations

import numpy as np


def random_points(n_bool: int, n_real: int, R: int, seed: int, b_lo: float = -1.0, b_hi: float = 1.0):
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1.0, 1.0, size=(n_bool, R)).astype(np.float32)
    b = rng.uniform(b_lo, b_hi, size=(n_real, R)).astype(np.float32)
    return a, b


def random_counters(n_cons: int, R: int, seed: int, max_u: int = 3):
    """Per-(constraint, restart) ERWA violation counters U (u8) for weighted parity cases."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, max_u + 1, size=(n_cons, R)).astype(np.uint8)
