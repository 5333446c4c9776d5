"""Both cohesion tile widths (128 and the small-n 64) and the tile-pair
kernel (pald_sym.cuh) at the same sizes, forced through
PALD_GPU_COHESION_TILE / PALD_GPU_SYM in a subprocess (the launcher reads
them once per process). PALD_GPU_RANK=2 forces the rank-coded pass 1
(pald_rank.cuh; by default only for pairwise 2048 < n <= 32768) at these
small sizes, PALD_GPU_RANK=0 covers the fp32 / integer-key pass 1 it
replaces."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
SCRIPT = Path(__file__).resolve().parent / "scripts" / "tile_parity.py"


@pytest.mark.parametrize("tile,sym,rank,sizes", [
    ("128", "0", "2", ["2", "65", "129", "300"]),
    ("64", "0", "2", ["3", "64", "257", "520"]),
    ("128", "2", "2", ["2", "127", "128", "129", "300", "520"]),
    ("128", "2", "0", ["2", "65", "129", "300"]),
    ("32", "0", "2", ["2", "33", "65", "129", "300"]),  # the tail tiles' width (pald_gpu.cu tail)
])
def test_cohesion_tile_width(tile, sym, rank, sizes):
    env = dict(os.environ, PALD_GPU_COHESION_TILE=tile, PALD_GPU_SYM=sym, PALD_GPU_RANK=rank)
    out = subprocess.run([sys.executable, str(SCRIPT), *sizes], env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    assert out.stdout.strip().endswith("ok")
