"""Helper run in a subprocess by tests/test_gpu_rank.py with PALD_GPU_RANK
forced (the launcher reads it once per process): the randomized case sweep of
test_gpu_parity.py (ragged sizes, uniform / integer / grid-point ties, wide
ranges; fast and exact layouts) through the pairwise kernels, strict and
InclusiveSplit, U and C bit-exact against the oracle."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle.oracle import Oracle  # noqa: E402
from paper_2307_16652_b200.engine import Engine  # noqa: E402
from test_gpu_parity import _random_case  # noqa: E402


def main():
    o = Oracle()
    seeds = [int(x) for x in sys.argv[1:]] or list(range(24))
    for seed in seeds:
        n, kind, d = _random_case(seed)
        D = torch.from_numpy(np.ascontiguousarray(d)).cuda()
        for policy in ("strict", "split"):
            e = Engine(n, "pairwise", force_exact=bool(seed % 2), policy=policy)
            e.run(D)
            torch.cuda.synchronize()
            u_ref, c_ref = o.pairwise_f32(d, policy=0 if policy == "strict" else 1)
            assert np.array_equal(e.U.cpu().numpy(), u_ref), (seed, n, kind, policy)
            assert np.array_equal(e.C.cpu().numpy().view(np.uint32), c_ref.view(np.uint32)), (seed, n, kind, policy)
    print("ok")


if __name__ == "__main__":
    main()
