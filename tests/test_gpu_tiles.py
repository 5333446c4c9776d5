"""Both cohesion tile widths (128 and the small-n 64) at the same sizes,
forced through PALD_GPU_COHESION_TILE in a subprocess (the launcher reads
it once per process)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
SCRIPT = Path(__file__).resolve().parent / "scripts" / "tile_parity.py"


@pytest.mark.parametrize("tile,sizes", [("128", ["2", "65", "129", "300"]), ("64", ["3", "64", "257", "520"])])
def test_cohesion_tile_width(tile, sizes):
    env = dict(os.environ, PALD_GPU_COHESION_TILE=tile)
    out = subprocess.run([sys.executable, str(SCRIPT), *sizes], env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    assert out.stdout.strip().endswith("ok")
