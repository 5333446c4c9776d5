"""Helper run in a subprocess by tests/test_gpu_tiescan.py (PALD_GPU_SYM is
read once per process): the pair kernel's full-range pass 2 against the
one-sided kernel's row bands, bit for bit, on large or degenerate inputs
that drive the tie scan through its multi-pass, bucket-overflow and
partition-overflow paths.

    python sym_vs_onesided.py KIND N [ALG]
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from helpers import random_upper  # noqa: E402
from paper_2307_16652_b200.engine import Engine  # noqa: E402


def make(kind: str, n: int) -> np.ndarray:
    if kind == "rand":
        return random_upper(n, 3)
    if kind == "grid":  # values on a 2^-18 grid: some duplicates in every column
        return (np.round(random_upper(n, 4) * 2 ** 18) / 2 ** 18).astype(np.float32)
    if kind == "mostly_one":  # one value dominates every column: partition overflow
        rng = np.random.default_rng(5)
        d = np.ones((n, n), np.float32)
        iu = np.triu_indices(n, 1)
        v = np.where(rng.random(iu[0].size) < 0.02, rng.uniform(0.5, 2.0, iu[0].size), 1.0)
        d[iu] = v.astype(np.float32)
        d[(iu[1], iu[0])] = d[iu]
        np.fill_diagonal(d, 0)
        return d
    if kind == "few_values":  # 40 distinct values: buckets of > 64 equal keys
        rng = np.random.default_rng(6)
        d = np.zeros((n, n), np.float32)
        iu = np.triu_indices(n, 1)
        d[iu] = rng.integers(1, 41, iu[0].size).astype(np.float32) / 8
        d[(iu[1], iu[0])] = d[iu]
        return d
    raise ValueError(kind)


def main():
    kind, n = sys.argv[1], int(sys.argv[2])
    alg = sys.argv[3] if len(sys.argv) > 3 else "pairwise"
    D = torch.from_numpy(make(kind, n)).cuda()
    e = Engine(n, alg)
    e.load(D)
    e.focus()
    h = (n // 2) // 128 * 128
    e.cohesion(0, h)
    e.cohesion(h, n)
    torch.cuda.synchronize()
    ref = e.C.clone()
    assert e.info()["cohesion_kernel"].startswith("pald_tile_kernel")
    e.C.zero_()
    e.cohesion()
    torch.cuda.synchronize()
    info = e.info()
    assert info["cohesion_kernel"] == "pald_sym_cohesion_kernel", info
    same = torch.equal(e.C.view(torch.int32), ref.view(torch.int32))
    print(kind, n, alg, "exact_step_share %.4f" % info["exact_step_share"], "same", same)
    sys.exit(0 if same else 1)


if __name__ == "__main__":
    main()
