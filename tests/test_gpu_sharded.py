"""The multi-rank path with the real GPU engine (torchrun, gloo, ranks
sharing cuda:0): results bit-identical to one process. Tied integer data
takes the one-sided kernel's row bands; random data with PALD_GPU_SYM=2
the pair kernel's tile-pair shares. PALD_GPU_SPLIT=0 keeps the
single-process triplet reference on whole pairs (the shares never split)."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
SCRIPT = Path(__file__).resolve().parent / "scripts" / "sharded_gpu.py"


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,n,alg,kind,mode", [
    (2, 700, "pairwise", "ties", "collectives"), (3, 513, "triplet", "ties", "collectives"),
    (2, 300, "triplet", "ties", "collectives"), (2, 700, "pairwise", "rand", "collectives"),
    (3, 1000, "pairwise", "rand", "collectives"),
    (2, 700, "pairwise", "rand", "fused"), (3, 1000, "pairwise", "rand", "fused"),
    (2, 700, "pairwise", "ties", "fused"), (3, 513, "triplet", "rand", "fused"),
    (4, 1500, "pairwise", "rand", "fused"),
    # n > 2048: pass 1 on rank codes (built on every rank), shares of its units
    (2, 2500, "pairwise", "rand", "collectives"), (3, 2500, "pairwise", "rand", "fused"),
    (2, 2500, "triplet", "rand", "fused"),
    # per-pass transports (pass 1: peer-pull finish [default], count
    # fan-out, NCCL/gloo all-reduce) and a non-current stream
    (3, 1000, "pairwise", "rand", "fused:red"), (2, 2500, "pairwise", "rand", "fused:nccl"),
    (3, 700, "triplet", "rand", "fused:peer:stream"), (2, 700, "pairwise", "ties", "collectives:stream"),
])
def test_sharded_real_engine(world, n, alg, kind, mode):
    """mode "fused": pass-1 counts and pass-2 entries written into every
    rank's buffers through CUDA IPC mappings (the ranks' processes share
    cuda:0 here; on a node they are NVLink peers). No kernel waits on another
    rank: the ranks are ordered by host barriers between the kernels."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", str(SCRIPT), str(n), alg, kind, mode]
    env = dict(os.environ, PALD_GPU_SYM="2", PALD_GPU_SPLIT="0")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "ok [1, 1]" in out.stdout
    if mode.startswith("fused"):
        assert "fused True" in out.stdout
        if kind == "rand":
            assert "fused_c True" in out.stdout
