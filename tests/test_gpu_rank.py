"""Rank-coded pass 1 (pald_rank.cuh): per-row rank codes of D, packed 16-bit
compares in the focus kernel. U must stay bit-exact (and C with it) for
every input the fp32 path handles: ties, ragged tiles, both layouts, both
policies, one- and two-segment rows (n > 16384 sorts two halves and merges
them)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from helpers import int_upper, random_upper

pytestmark = pytest.mark.gpu
SCRIPT = Path(__file__).resolve().parent / "scripts" / "rank_sweep.py"


def test_rank_path_forced_randomized_sweep():
    env = dict(os.environ, PALD_GPU_RANK="2")
    out = subprocess.run([sys.executable, str(SCRIPT)], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    assert out.stdout.strip().endswith("ok")


def _points(n, seed, dim=3):
    rng = np.random.default_rng(seed)
    p = rng.random((n, dim))
    from paper_2307_16652_b200.datagen import distances_from_points

    return distances_from_points(p)


@pytest.mark.parametrize("n,kind", [(16384, "rand"), (16385, "rand"), (20000, "int16"), (23000, "points")])
def test_rank_path_segments_sampled_rows(oracle, n, kind):
    import torch

    from paper_2307_16652_b200.engine import Engine

    if kind == "rand":
        d = random_upper(n, n)
    elif kind == "int16":
        d = int_upper(n, n)
    else:
        d = _points(n, n)
    e = Engine(n, "pairwise")
    e.run(torch.from_numpy(d).cuda())
    torch.cuda.synchronize()
    assert e.info()["rank_codes"]
    rows = np.unique(np.r_[0, 1, 127, 128, 16383, 16384 % n, n // 2, n - 1])
    ur, cr = oracle.pairwise_rows_f32(d, rows)
    assert np.array_equal(e.U[rows.tolist()].cpu().numpy(), ur)
    assert np.array_equal(e.C[rows.tolist()].cpu().numpy().view(np.uint32), cr.view(np.uint32))


def test_bins_tie_marks_equal_tie_scan():
    """The rank-code bins kernel marks the duplicate pairs of its rows for the
    pair kernel instead of tie_scan_kernel: same marked share (a few
    duplicates per column, no overflowing hash bucket) and, with the pair
    kernel forced, C equal to the one-sided kernel bit for bit."""
    script = Path(__file__).resolve().parent / "scripts" / "sym_vs_onesided.py"
    shares = {}
    for rank in ("0", "1"):
        env = dict(os.environ, PALD_GPU_SYM="2", PALD_GPU_RANK=rank)
        out = subprocess.run([sys.executable, str(script), "grid", "13001", "pairwise"], env=env,
                             capture_output=True, text=True, timeout=900)
        assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
        assert "same True" in out.stdout
        shares[rank] = float(out.stdout.split("exact_step_share")[1].split()[0])
    assert 0.0 < shares["1"] < 0.5
    assert shares["0"] == shares["1"]
