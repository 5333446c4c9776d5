"""Accurate-mode block size sweep (run once per PALD_GPU_ACC_BLOCK value:
the knob is read once per process): pass-2 time and max rel_diff vs the
fp64 oracle on sampled rows, for config 3 (pairwise, n = 8192) and
config 2 (triplet, n = 4096).

    PALD_GPU_ACC_BLOCK=1024 python tools/acc_sweep.py
"""
import json
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import numpy as np
    import torch

    from bench import make_input
    from helpers import boundary_rows, max_rel_diff, rows_parallel
    from oracle.oracle import Oracle
    from paper_2307_16652_b200.engine import Engine

    orc = Oracle()
    out = {"block": os.environ.get("PALD_GPU_ACC_BLOCK", "default")}
    for idx, alg in ((3, "pairwise"), (2, "triplet")):
        D, cfg = make_input(idx, "cuda", 20230731)
        n = cfg.n
        for acc in (False, True):
            if alg == "triplet" and not acc:
                continue
            e = Engine(n, alg, accurate=acc)
            for _ in range(2):
                e.run(D)
            torch.cuda.synchronize()
            s = torch.cuda.current_stream()
            ts = []
            for _ in range(3):
                e.load(D)
                e.focus()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                e.cohesion()
                b.record(s)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            rows = boundary_rows(n, extra=18, seed=1)
            d = D.cpu().numpy()
            fn = orc.pairwise_rows_f64 if alg == "pairwise" else orc.triplet_rows_f64
            _, c64 = rows_parallel(fn, d, rows)
            err = max_rel_diff(e.C[rows.tolist()].cpu().numpy(), c64)
            out[f"{cfg.name}:{alg}:{'acc' if acc else 'fp32'}"] = {"pass2_ms": statistics.median(ts), "max_rel": err}
            del e
            torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
