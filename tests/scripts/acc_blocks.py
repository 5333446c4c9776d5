"""Accurate mode with tiny k blocks (run with PALD_GPU_ACC_BLOCK=64 by
tests/test_gpu_accurate.py): C and the double sums vs the fp64 oracle."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from helpers import int_upper, max_rel_diff, random_upper  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_2307_16652_b200.engine import Engine  # noqa: E402

orc = Oracle()
cases = [("pairwise", random_upper(1300, 1)), ("pairwise", int_upper(700, 2)), ("triplet", random_upper(900, 3))]
for alg, d in cases:
    n = d.shape[0]
    e = Engine(n, alg, accurate=True)
    e.run(torch.from_numpy(d).cuda())
    torch.cuda.synchronize()
    u64, c64 = (orc.pairwise_f64 if alg == "pairwise" else orc.triplet_f64)(d)
    assert np.array_equal(e.U.cpu().numpy(), u64), alg
    err = max_rel_diff(e.C.cpu().numpy(), c64)
    err64 = max_rel_diff(e.C64.cpu().numpy(), c64)
    assert err <= 1e-6 and err64 <= 1e-6, (alg, n, err, err64, e.info())
    print(alg, n, e.info()["cohesion_kernel"], "C err %.2e, double sums err %.2e" % (err, err64))
print("ok")
