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


def rows_parallel(fn, d, rows, workers=None):
    """Run an O(n^2)-per-row oracle restatement (ctypes, releases the GIL)
    over `rows` on all host cores; returns the concatenated outputs."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    rows = np.asarray(rows, np.int64)
    workers = workers or len(os.sched_getaffinity(0))
    chunks = [c for c in np.array_split(rows, max(1, min(workers, rows.size))) if c.size]
    with ThreadPoolExecutor(len(chunks)) as ex:
        res = list(ex.map(lambda r: fn(d, r), chunks))
    return tuple(np.concatenate([x[k] for x in res]) for k in range(len(res[0])))


def boundary_rows(n, tile=128, extra=0, seed=0):
    """First / last rows of tiles 0 and 1, the middle, the last (short) tile,
    the last rows, plus `extra` random rows (SURVEY 7 hard part 6)."""
    fixed = [0, 1, tile - 1, tile, tile + 1, 2 * tile - 1, n // 2 - 1, n // 2, n // 2 + 1,
             (n - 1) // tile * tile, (n - 1) // tile * tile + 1, n - tile - 1, n - 2, n - 1]
    rng = np.random.default_rng(seed)
    rows = [r for r in fixed if 0 <= r < n] + list(rng.integers(0, n, extra))
    return np.unique(np.array(rows, np.int64))
