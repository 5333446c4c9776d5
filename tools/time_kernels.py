"""Quick kernel timing for iteration: per-pass CUDA-event times and
combos/SM-cycle on selected BASELINE configs (device-resident)."""
import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3:pairwise,2:triplet,1:pairwise")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--exact", action="store_true")
    ap.add_argument("--check", action="store_true", help="sampled-row oracle check (pairwise)")
    a = ap.parse_args()
    import numpy as np
    import torch

    from bench import make_input
    from paper_2307_16652_b200.engine import Engine

    mhz = 1965.0
    for spec in a.configs.split(","):
        idx, alg = spec.split(":")
        D, cfg = make_input(int(idx), "cuda", 20230731)
        n = cfg.n
        eng = Engine(n, alg, force_exact=a.exact)
        for _ in range(2):
            eng.run(D)
        torch.cuda.synchronize()
        s = torch.cuda.current_stream()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(a.iters)]
        for e in ev:
            e[0].record(s); eng.load(D); e[1].record(s); eng.focus(); e[2].record(s); eng.cohesion(); e[3].record(s)
        torch.cuda.synchronize()
        f = statistics.median(e[1].elapsed_time(e[2]) for e in ev) / 1e3
        c = statistics.median(e[2].elapsed_time(e[3]) for e in ev) / 1e3
        t = statistics.median(e[0].elapsed_time(e[3]) for e in ev) / 1e3
        ld_ms = statistics.median(e[0].elapsed_time(e[1]) for e in ev)
        nb = eng.tiles_per_dim
        fcombos = nb * (nb + 1) / 2 * 128 * 128 * n
        ccombos = nb * nb * 128 * 128 * n
        cyc = 148 * mhz * 1e6
        print(f"{cfg.name}:{alg} n={n} step {t*1e3:.2f} ms  load {ld_ms:.2f} ms  focus {f*1e3:.2f} ms "
              f"({fcombos/f/cyc:.1f} combos/SM-cyc)  cohesion {c*1e3:.2f} ms ({ccombos/c/cyc:.1f})  "
              f"triplets/s {n**3/t:.3e} exact={eng.exact_path}", flush=True)
        if a.check and alg == "pairwise":
            from oracle.oracle import Oracle
            d = D.cpu().numpy()
            rows = np.unique(np.r_[0, 1, 127, 128, n // 2, n - 2, n - 1])
            ur, cr = Oracle().pairwise_rows_f32(d, rows)
            U = eng.U.cpu().numpy()[rows]
            C = eng.C.cpu().numpy()[rows]
            print("   check rows", rows.tolist(), "U exact", np.array_equal(U, ur),
                  "C bit-exact", np.array_equal(C.view(np.uint32), cr.view(np.uint32)), flush=True)
        del eng, D
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
