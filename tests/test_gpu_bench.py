"""bench.py contract on the GPU: one JSON line with the required keys, on
one rank and on two torchrun ranks (gloo test hook, ranks sharing cuda:0),
and the reference arm. Small configs keep each run to seconds."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
            "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return json.loads(lines[0])


def test_bench_single_gpu_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", "3", "--steps", "2",
                          "--warmup", "3", "--no-secondary", "--cpu-budget", "2"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    j = _last_json(out.stdout)
    for k in REQUIRED:
        assert k in j, k
    assert j["n_gpus"] == 1 and j["steps"] == 2 and j["warmup"] == 3
    assert j["roofline"]["kernel"] == "pald_sym_cohesion_kernel"
    assert 0 < j["roofline"]["frac"] < 1.5
    assert j["gpu_launches"] > 0
    assert j["e2e"]["value"] > 0 and j["e2e"]["h2d_bytes_per_step"] == 8192 * 8192 * 4
    assert j["cpu_baseline"]["kind"] == "reference" and j["cpu_baseline"]["value"] > 0


def test_bench_two_ranks_gloo():
    env = dict(os.environ, PALD_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", str(ROOT / "bench.py"), "--gpus", "2",
           "--config", "1", "--steps", "2", "--warmup", "3", "--no-secondary", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    j = _last_json(out.stdout)
    for k in REQUIRED:
        assert k in j, k
    assert j["n_gpus"] == 2
    assert j["e2e"]["value"] > 0


def test_bench_reference_arm():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "3", "--ref-step-s", "1"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    j = _last_json(out.stdout)
    assert j["impl"] == "reference" and j["value"] > 0
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["cpu_baseline"]["kind"] == "reference"
