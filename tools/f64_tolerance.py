"""fp32 C (ours, bit-identical to the reference's fp32 pairwise C) against
fp64 accumulation on sampled rows, per BASELINE config: the numbers behind
the tolerance statements in DESIGN.md section 4.

    python tools/f64_tolerance.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import torch

    from bench import make_input
    from helpers import max_rel_diff
    from oracle.oracle import Oracle
    from paper_2307_16652_b200.engine import Engine

    o = Oracle()
    for idx, alg in ((1, "pairwise"), (3, "pairwise"), (2, "triplet"), (5, "pairwise")):
        D, cfg = make_input(idx, "cuda", 20230731)
        n = cfg.n
        e = Engine(n, alg)
        e.run(D)
        torch.cuda.synchronize()
        rows = np.array([0, n // 2, n - 1])
        d = D.cpu().numpy()
        _, c64 = (o.pairwise_rows_f64 if alg == "pairwise" else o.triplet_rows_f64)(d, rows)
        cg = e.C[rows.tolist()].cpu().numpy()
        rs = np.abs(cg.astype(np.float64).sum(1) - c64.sum(1)) / c64.sum(1)
        print(f"{cfg.name}:{alg} n={n} max rel_diff vs fp64 {max_rel_diff(cg, c64):.3e} "
              f"row-sum rel {rs.max():.3e}", flush=True)
        del e, D
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
