"""The tie scan behind the pair kernel (pald_sym.cuh) on inputs that take
each of its paths, with the pair kernel forced (PALD_GPU_SYM=2) and checked
bit for bit against the one-sided kernel: several hash partitions
(n > 12288), buckets of more than 64 equal-hash values and partitions over
capacity (whole tiles marked), and a ragged n. PALD_GPU_SPLIT=0 keeps the
triplet's full-range pass 2 on whole pairs (its k-split last round regroups
the sums: tests/test_gpu_parity.py::test_triplet_split_last_round)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
SCRIPT = Path(__file__).resolve().parent / "scripts" / "sym_vs_onesided.py"


@pytest.mark.parametrize("kind,n,alg", [
    ("grid", 13001, "pairwise"),       # 2 partitions, a few duplicates per column
    ("rand", 12300, "pairwise"),       # 2 partitions, ragged n
    ("few_values", 3000, "pairwise"),  # buckets > 64: whole tiles marked
    ("mostly_one", 17000, "pairwise"),  # partition over capacity: whole tiles marked
    ("grid", 5000, "triplet"),
])
def test_pair_kernel_matches_one_sided(kind, n, alg):
    env = dict(os.environ, PALD_GPU_SYM="2", PALD_GPU_SPLIT="0")
    out = subprocess.run([sys.executable, str(SCRIPT), kind, str(n), alg], env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    assert "same True" in out.stdout
    share = float(out.stdout.split("exact_step_share")[1].split()[0])
    if kind in ("few_values", "mostly_one"):
        assert share == 1.0  # whole tiles marked
    elif kind == "grid" and alg == "pairwise":
        assert 0.0 < share < 0.5  # marked k mixed with shared steps


def test_pair_kernel_size_sweep():
    """Seeded sweep of sizes (ragged, below and above one wave of pairs,
    with and without the 64-wide tail tiles), both algorithms."""
    env = dict(os.environ, PALD_GPU_SYM="2", PALD_GPU_SPLIT="0")
    script = Path(__file__).resolve().parent / "scripts" / "pair_sweep.py"
    out = subprocess.run([sys.executable, str(script), "7"], env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
