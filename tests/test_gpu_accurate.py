"""Accurate mode (PALD_GPU_FLAG_ACCURATE, include/pald_gpu.h): pass 2 keeps
each output's fp32 running sum only over k blocks of 1024 terms and adds
the block partials into a double sum (exact, order-independent), rounded to
fp32 at the end. U is unchanged (pass 1 is integer work); C is compared
with the fp64-accumulated oracle (oracle/pald_oracle.c *_f64), which the
default mode -- the reference's own single fp32 chain, bit-identical to
blocked_pairwise<float> -- drifts from by up to ~1.3e-5 at n = 32768."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from helpers import int_upper, max_rel_diff, random_upper

pytestmark = pytest.mark.gpu


def engine(D, alg, accurate, policy="strict"):
    from paper_2307_16652_b200.engine import Engine

    e = Engine(D.shape[0], alg, accurate=accurate, policy=policy)
    e.run(D)
    torch.cuda.synchronize()
    return e


def test_accurate_pairwise_pair_kernel(oracle):
    """Random D at n = 2304 (pair kernel + tail tiles): U identical to the
    default mode, C within 3e-6 of fp64 (one 1024-term fp32 chain alone
    reaches ~2e-6: config 1), the double sums likewise (both differ from the
    fp64 oracle only by the fp32 rounding of each block partial), and C = the
    double sums rounded once."""
    n = 2304
    d = random_upper(n, 11)
    D = torch.from_numpy(d).cuda()
    ref = engine(D, "pairwise", False)
    acc = engine(D, "pairwise", True)
    assert acc.info()["cohesion_kernel"] == "pald_sym_cohesion_kernel"
    U = acc.U.cpu().numpy()
    assert np.array_equal(U, ref.U.cpu().numpy())
    u64, c64 = oracle.pairwise_f64(d)
    assert np.array_equal(U, u64)
    C = acc.C.cpu().numpy()
    assert max_rel_diff(C, c64) <= 3e-6
    # the double sums: only the fp32 rounding of each <= 1024-term partial
    assert max_rel_diff(acc.C64.cpu().numpy(), c64) <= 3e-6
    # C is the double sum rounded once to fp32
    assert np.array_equal(C, acc.C64.cpu().numpy().astype(np.float32))


def test_accurate_one_sided_and_ties(oracle):
    """Integer D (every k tied: one-sided 64- / 128-wide kernels), both
    policies of the pairwise algorithm, and the exact (integer-key) path."""
    from paper_2307_16652_b200.engine import Engine

    n = 1500
    d = int_upper(n, 3)
    D = torch.from_numpy(d).cuda()
    u64, c64 = oracle.pairwise_f64(d)
    acc = engine(D, "pairwise", True)
    assert acc.info()["cohesion_kernel"].startswith("pald_tile_kernel")
    assert np.array_equal(acc.U.cpu().numpy(), u64)
    assert max_rel_diff(acc.C.cpu().numpy(), c64) <= 3e-6
    ex = Engine(n, "pairwise", force_exact=True, accurate=True)
    ex.run(D)
    torch.cuda.synchronize()
    assert ex.exact_path
    assert np.array_equal(ex.C.cpu().numpy().view(np.uint32), acc.C.cpu().numpy().view(np.uint32))
    # InclusiveSplit: same U as the default mode, C close to the default's
    sp = engine(D, "pairwise", True, policy="split")
    sd = engine(D, "pairwise", False, policy="split")
    assert np.array_equal(sp.U.cpu().numpy(), sd.U.cpu().numpy())
    assert max_rel_diff(sp.C.cpu().numpy(), sd.C.cpu().numpy()) <= 5e-6


def test_accurate_triplet(oracle):
    """Triplet pass 2 (pair kernel, no k split in accurate mode): U exact,
    C within 3e-6 of fp64, diagonal 0 in C and in the double sums."""
    n = 1700
    d = random_upper(n, 5)
    D = torch.from_numpy(d).cuda()
    acc = engine(D, "triplet", True)
    u64, c64 = oracle.triplet_f64(d)
    assert np.array_equal(acc.U.cpu().numpy(), u64)
    C = acc.C.cpu().numpy()
    assert max_rel_diff(C, c64) <= 3e-6
    assert np.all(np.diagonal(C) == 0) and np.all(np.diagonal(acc.C64.cpu().numpy()) == 0)


def test_accurate_through_c_abi(oracle):
    """The flag through the reference-facing host call."""
    import ctypes as C

    from paper_2307_16652_b200 import _lib
    from paper_2307_16652_b200.api import _raise_for

    n = 900
    d = random_upper(n, 21)
    lib = _lib.load()
    for alg, orc in ((_lib.PAIRWISE, oracle.pairwise_f64), (_lib.TRIPLET, oracle.triplet_f64)):
        o = _lib.make_opts(algorithm=alg, flags=_lib.FLAG_ACCURATE)
        u = np.empty((n, n), np.int32)
        c = np.empty((n, n), np.float32)
        _raise_for(lib.pald_gpu_cohesion_f32(d.ctypes.data, n, C.byref(o), u.ctypes.data, c.ctypes.data, None))
        u64, c64 = orc(d)
        assert np.array_equal(u, u64)
        assert max_rel_diff(c, c64) <= 3e-6


def test_accurate_small_blocks_subprocess():
    """PALD_GPU_ACC_BLOCK=64 (read once per process): every output is
    flushed every 64 terms -- many partial flushes per pair / tile on all
    pass-2 kernels (pair kernel, 64-wide tail, one-sided, triplet)."""
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, PALD_GPU_ACC_BLOCK="64")
    r = subprocess.run([sys.executable, str(root / "tests" / "scripts" / "acc_blocks.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ok" in r.stdout


def test_triplet_tie_marks_on_quantized_data(oracle):
    """Triplet with tie marks (n > 2048: rank codes; pald_sym.cuh tri_marks):
    chunks inside the row / column tiles run the fast steps for unmarked k.
    Distances on a 2^-14 grid: every row holds duplicates, so marks are
    mixed. Sampled rows (tile edges included) against the fp64 oracle: U
    exact, C within 3e-6 (accurate double sums)."""
    from helpers import boundary_rows, rows_parallel

    n = 2600
    rng = np.random.default_rng(12)
    d = np.zeros((n, n), np.float32)
    iu = np.triu_indices(n, 1)
    d[iu] = (np.floor(rng.uniform(1.0, 2.0, iu[0].size) * 2 ** 14) / 2 ** 14).astype(np.float32)
    d[(iu[1], iu[0])] = d[iu]
    e = engine(torch.from_numpy(d).cuda(), "triplet", False)
    assert e.info()["rank_codes"] and e.info()["cohesion_kernel"] == "pald_sym_cohesion_kernel"
    rows = boundary_rows(n, extra=10, seed=3)
    ur, cr = rows_parallel(oracle.triplet_rows_f64, d, rows)
    assert np.array_equal(e.U[rows.tolist()].cpu().numpy(), ur)
    assert max_rel_diff(e.C[rows.tolist()].cpu().numpy(), cr) <= 3e-6
