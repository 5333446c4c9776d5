"""Helper for tests/test_gpu_sharded.py: the multi-rank driver
(ShardedRunner) with the REAL GPU engine, 2-3 processes sharing one GPU,
collectives over gloo (host-mediated, so no kernel waits on another rank).
Each rank checks its U and C against a single-process run."""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from helpers import int_upper, random_upper  # noqa: E402
from paper_2307_16652_b200.distributed import ShardedRunner  # noqa: E402
from paper_2307_16652_b200.engine import Engine  # noqa: E402


def main():
    n, alg = int(sys.argv[1]), sys.argv[2]
    kind = sys.argv[3] if len(sys.argv) > 3 else "ties"
    mode = sys.argv[4] if len(sys.argv) > 4 else "collectives"
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    D = torch.from_numpy(int_upper(n, 17) if kind == "ties" else random_upper(n, 17)).cuda()
    ref = Engine(n, alg)
    ref.run(D)
    eng = Engine(n, alg)
    # mode: collectives | fused[:<pass-1 exchange>][:stream]
    parts = mode.split(":")
    fused = parts[0] == "fused"
    fx = next((p for p in parts[1:] if p in ("peer", "red", "nccl")), None)
    use_stream = "stream" in parts[1:]
    runner = ShardedRunner(eng, fused=fused, focus_exchange=fx)
    if fused:
        assert runner.fused, "peer mapping failed"
    # a non-current stream: the runner must order its barriers and
    # collectives after the work issued on it
    stream = torch.cuda.Stream() if use_stream else None
    for _ in range(2):  # repeated steps reuse the plan
        runner.step(D, stream=stream)
    torch.cuda.synchronize()
    ok_u = torch.equal(eng.U, ref.U)
    ok_c = torch.equal(eng.C.view(torch.int32), ref.C.view(torch.int32))
    flags = torch.tensor([int(ok_u), int(ok_c)], dtype=torch.int32)
    dist.all_reduce(flags, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("shares", runner.plan.focus_share, "kernel", eng.info()["cohesion_kernel"], "fused", runner.fused,
              "fused_c", runner._fused_c, "focus_exchange", runner.focus_exchange, "ok", flags.tolist())
    dist.destroy_process_group()
    sys.exit(0 if flags.tolist() == [1, 1] else 1)


if __name__ == "__main__":
    main()
