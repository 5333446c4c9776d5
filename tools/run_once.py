"""Run the engine on one BASELINE config (for ncu / launch-list captures).

    python tools/run_once.py --config 3 --alg pairwise --iters 3
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--alg", default="pairwise")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--exact", action="store_true")
    ap.add_argument("--accurate", action="store_true")
    a = ap.parse_args()
    import torch

    from bench import make_input
    from paper_2307_16652_b200.engine import Engine

    D, cfg = make_input(a.config, "cuda", 20230731)
    eng = Engine(cfg.n, a.alg, force_exact=a.exact, accurate=a.accurate)
    for _ in range(a.iters):
        eng.run(D)
    torch.cuda.synchronize()
    print("ok", cfg.name, a.alg, "launches", eng.launches, "exact", eng.exact_path)


if __name__ == "__main__":
    main()
