"""One B200 at n beyond the BASELINE configs: seeded points U[0,1)^3,
D on the GPU, one full pass (load + pass 1 + pass 2) timed with CUDA
events, U/C of sampled rows checked bit-exact against the oracle's
per-row restatement (needs a host copy of D).

    python tools/large_n.py 49152 [--check]
"""
import argparse
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("n", type=int)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_2307_16652_b200.engine import Engine, points_to_distances

    rng = np.random.default_rng(20230731)
    pts = torch.from_numpy(rng.random((a.n, 3))).cuda()
    D = points_to_distances(pts)
    e = Engine(a.n, "pairwise")
    e.run(D)
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(a.iters):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(s); e.load(D); ev[1].record(s); e.focus(); ev[2].record(s); e.cohesion(); ev[3].record(s)
        torch.cuda.synchronize()
        ts.append([ev[i].elapsed_time(ev[i + 1]) for i in range(3)])
    load, foc, coh = (statistics.median(t[i] for t in ts) for i in range(3))
    step = load + foc + coh
    print(f"n={a.n} step {step / 1e3:.3f} s (load {load:.1f} ms, focus {foc / 1e3:.3f} s, cohesion "
          f"{coh / 1e3:.3f} s) {a.n ** 3 / (step / 1e3):.3e} triplets/s kernel {e.info()['cohesion_kernel']} "
          f"exact steps {100 * e.info()['exact_step_share']:.3f}% mem {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB "
          f"(torch) free {torch.cuda.mem_get_info()[0] / 2**30:.1f} GiB")
    if a.check:
        from oracle.oracle import Oracle

        d = D.cpu().numpy()
        rows = np.array([0, 1, 127, 128, a.n // 2, a.n - 2, a.n - 1])
        u_ref, c_ref = Oracle().pairwise_rows_f32(d, rows)
        ok_u = np.array_equal(e.U[rows].cpu().numpy(), u_ref)
        ok_c = np.array_equal(e.C[rows].cpu().numpy().view(np.uint32), c_ref.view(np.uint32))
        print("rows", rows.tolist(), "U exact", ok_u, "C bit-exact", ok_c)
        sys.exit(0 if ok_u and ok_c else 1)


if __name__ == "__main__":
    main()
