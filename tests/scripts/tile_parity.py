"""Helper run in a subprocess by tests/test_gpu_tiles.py: parity of the
cohesion kernel at the tile width forced by PALD_GPU_COHESION_TILE, or of
the tile-pair kernel forced by PALD_GPU_SYM=2. Kinds: "rand" (no ties),
"ties" (integers 1..16: every block tied, whole tiles flagged), "fewties"
(values on a 2^-9 grid: a few duplicates per column, so flagged and
unflagged blocks mix)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from helpers import int_upper, max_rel_diff, random_upper  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402
from paper_2307_16652_b200.engine import Engine  # noqa: E402


def main():
    o = Oracle()
    sizes = [int(x) for x in sys.argv[1:]] or [2, 65, 129, 300]
    for n in sizes:
        for kind in ("rand", "ties", "fewties"):
            if kind == "rand":
                d = random_upper(n, n)
            elif kind == "ties":
                d = int_upper(n, n)
            else:
                d = (np.round(random_upper(n, n + 1) * 512) / 512).astype(np.float32)
            D = torch.from_numpy(d).cuda()
            for policy in ("strict", "split"):
                for exact in (False, True):
                    e = Engine(n, "pairwise", force_exact=exact, policy=policy)
                    e.run(D)
                    torch.cuda.synchronize()
                    u_ref, c_ref = o.pairwise_f32(d, policy=0 if policy == "strict" else 1)
                    assert np.array_equal(e.U.cpu().numpy(), u_ref), (n, kind, policy, exact)
                    assert np.array_equal(e.C.cpu().numpy().view(np.uint32), c_ref.view(np.uint32)), \
                        (n, kind, policy, exact)
            for exact in (False, True):
                e = Engine(n, "triplet", force_exact=exact)
                e.run(D)
                torch.cuda.synchronize()
                u_ref, c_ref = o.triplet_f64(d)
                assert np.array_equal(e.U.cpu().numpy(), u_ref), (n, kind, "triplet", exact)
                assert max_rel_diff(e.C.cpu().numpy(), c_ref) <= 1e-5
    print("ok")


if __name__ == "__main__":
    main()
