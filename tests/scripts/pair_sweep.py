"""Helper for tests/test_gpu_tiescan.py: with the pair kernel forced
(PALD_GPU_SYM=2), the full-range pass 2 (pair kernel, plus the 64-wide tail
tiles where the plan uses them) must equal the one-sided kernel's row bands
bit for bit over a seeded sweep of sizes, both algorithms, random and
quantized inputs."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from helpers import random_upper  # noqa: E402
from paper_2307_16652_b200.engine import Engine  # noqa: E402


def main():
    rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
    sizes = sorted(set(int(x) for x in rng.integers(2, 3200, 10))) + [2049, 2176, 2305]
    bad = []
    for n in sizes:
        for alg in ("pairwise", "triplet"):
            d = random_upper(n, n)
            if n % 2:
                d = (np.round(d * 2 ** 14) / 2 ** 14).astype(np.float32)  # some duplicates
            D = torch.from_numpy(d).cuda()
            e = Engine(n, alg)
            e.load(D)
            e.focus()
            h = (n // 2) // 128 * 128
            e.cohesion(0, h)
            e.cohesion(h, n)
            torch.cuda.synchronize()
            ref = e.C.clone()
            e.C.zero_()
            e.cohesion()
            torch.cuda.synchronize()
            same = torch.equal(e.C.view(torch.int32), ref.view(torch.int32))
            if not same or e.info()["cohesion_kernel"] != "pald_sym_cohesion_kernel":
                bad.append((n, alg, same, e.info()["cohesion_kernel"]))
    print("sizes", sizes, "bad", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
