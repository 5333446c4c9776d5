"""Comparison helpers following the reference's test helpers
(proj/tests/helpers.hpp:30-45)."""
import numpy as np


def rel_diff(a, b):
    """helpers.hpp:30-33: |a-b| / max(|a|, |b|, 1)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1.0)
    return np.abs(a - b) / scale


def max_rel_diff(a, b) -> float:
    return float(rel_diff(a, b).max()) if np.size(a) else 0.0


def random_upper(n: int, seed: int, lo=0.5, hi=2.0) -> np.ndarray:
    """Symmetric fp32 D with U(lo, hi) upper triangle (random_distances-like)."""
    rng = np.random.default_rng(seed)
    d = np.zeros((n, n), np.float32)
    iu = np.triu_indices(n, 1)
    v = rng.uniform(lo, hi, iu[0].size).astype(np.float32)
    d[iu] = v
    d[(iu[1], iu[0])] = v
    return d


def int_upper(n: int, seed: int, lo=1, hi=16) -> np.ndarray:
    rng = np.random.default_rng(seed)
    d = np.zeros((n, n), np.float32)
    iu = np.triu_indices(n, 1)
    v = rng.integers(lo, hi + 1, iu[0].size).astype(np.float32)
    d[iu] = v
    d[(iu[1], iu[0])] = v
    return d
