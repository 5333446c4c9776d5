"""Per-phase device times of one BASELINE config (engine staged calls, CUDA
events), for A/B runs of the small-n knobs in separate processes:

    PALD_GPU_RANK=2 python tools/small_n.py --config 1
"""
import argparse
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--alg", default="pairwise")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--oneshot", action="store_true", help="time pald_gpu_cohesion_f32_device instead")
    ap.add_argument("--accurate", action="store_true", help="PALD_GPU_FLAG_ACCURATE (k-block items)")
    a = ap.parse_args()
    import ctypes as C

    import torch

    from bench import make_input
    from paper_2307_16652_b200 import _lib
    from paper_2307_16652_b200.api import _raise_for
    from paper_2307_16652_b200.engine import Engine

    D, cfg = make_input(a.config, "cuda", 20230731)
    n = cfg.n
    s = torch.cuda.current_stream()
    if a.oneshot:
        lib = _lib.load()
        o = _lib.make_opts(algorithm=_lib.PAIRWISE if a.alg == "pairwise" else _lib.TRIPLET)
        U = torch.empty((n, n), dtype=torch.int32, device="cuda")
        Cm = torch.empty((n, n), dtype=torch.float32, device="cuda")
        f = lambda: _raise_for(lib.pald_gpu_cohesion_f32_device(  # noqa: E731
            D.data_ptr(), n, n, C.byref(o), U.data_ptr(), n, Cm.data_ptr(), n, s.cuda_stream))
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.iters):
            f()
        e1.record(s)
        torch.cuda.synchronize()
        print(json.dumps({"config": a.config, "alg": a.alg, "oneshot_ms": e0.elapsed_time(e1) / a.iters,
                          "env": {k: v for k, v in os.environ.items() if k.startswith("PALD_GPU")}}))
        return
    eng = Engine(n, a.alg, accurate=a.accurate)
    for _ in range(3):
        eng.run(D)
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(a.iters)]
    for e in evs:
        e[0].record(s)
        eng.load(D)
        e[1].record(s)
        eng.focus()
        e[2].record(s)
        eng.cohesion()
        e[3].record(s)
    torch.cuda.synchronize()
    med = lambda i, j: statistics.median(e[i].elapsed_time(e[j]) for e in evs)  # noqa: E731
    print(json.dumps({"config": a.config, "alg": a.alg, "n": n, "step_ms": med(0, 3), "load_ms": med(0, 1),
                      "focus_ms": med(1, 2), "cohesion_ms": med(2, 3), "accurate": a.accurate, "info": eng.info(),
                      "env": {k: v for k, v in os.environ.items() if k.startswith("PALD_GPU")}}))


if __name__ == "__main__":
    main()
