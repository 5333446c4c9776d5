"""Per-pass CUDA-event times of the engine on random D at given sizes
(for cost-model checks): python tools/time_n.py 2176 pairwise"""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))


def main():
    import torch

    from helpers import random_upper
    from paper_2307_16652_b200.engine import Engine

    alg = sys.argv[2] if len(sys.argv) > 2 else "pairwise"
    for n in [int(x) for x in sys.argv[1].split(",")]:
        D = torch.from_numpy(random_upper(n, 5)).cuda()
        e = Engine(n, alg)
        e.run(D)
        s = torch.cuda.current_stream()
        ts = []
        for _ in range(5):
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record(s); e.focus(); b.record(s); e.cohesion(); c.record(s)
            torch.cuda.synchronize()
            ts.append((a.elapsed_time(b), b.elapsed_time(c)))
        f = statistics.median(t[0] for t in ts)
        c = statistics.median(t[1] for t in ts)
        print(f"n={n} {alg} focus {f:.3f} ms cohesion {c:.3f} ms kernel {e.info()['cohesion_kernel']}")


if __name__ == "__main__":
    main()
