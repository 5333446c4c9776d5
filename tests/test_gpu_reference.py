"""Full-matrix parity against the UNMODIFIED reference, run on the GPU box's
host cores (oracle/_ref: the reference headers compiled by oracle/Makefile,
oracle/ref_bridge.cpp), on the BASELINE.json configurations:

  parallel_pairwise<float>   (parallel.hpp:159-222): U exact, C bit-exact --
                             configs 1, 3 (n = 8192) and 4
  parallel_triplet<double>   (parallel.hpp:257-320): U exact, C rel_diff
                             <= 1e-5 (helpers.hpp:30-33) -- configs 2 and 4
  config 5 (n = 32768, too large for the full CPU run): >= 64 rows --
                             first / last rows of tiles 0 and 1, the middle,
                             the last (short) tile, random rows -- bit-exact
                             against the oracle's per-row restatement of the
                             fp32 reference order, the same rows against the
                             fp64 accumulation, ALL n row sums against the
                             accurate mode's double sums, and
                             sum(C) = n(n-1)/2.
  the reference's acceptance corpus through the C++ shim compiled against
  the reference's own types (oracle/_ref/acceptance_gpu).
"""
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest
import torch

from helpers import boundary_rows, max_rel_diff, rows_parallel

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
SEED = 20230731


def cores():
    return len(os.sched_getaffinity(0))


def config_d(idx):
    from paper_2307_16652_b200 import datagen
    from paper_2307_16652_b200.engine import points_to_distances

    cfg = datagen.config(idx)
    pts = datagen.make_points(cfg, SEED)
    if pts is not None:
        return points_to_distances(torch.from_numpy(pts).cuda()), cfg
    return torch.from_numpy(datagen.make_distances(cfg, SEED)).cuda(), cfg


def gpu_run(D, alg, accurate=False):
    from paper_2307_16652_b200.engine import Engine

    e = Engine(D.shape[0], alg, accurate=accurate)
    e.run(D)
    torch.cuda.synchronize()
    return e


@pytest.mark.parametrize("idx", [1, 4, 3])
def test_pairwise_full_matrix_vs_reference(reference, idx):
    """parallel_pairwise<float> with all host threads at its default block
    size: every U and every C bit of the whole matrix."""
    D, cfg = config_d(idx)
    d = D.cpu().numpy()
    e = gpu_run(D, "pairwise")
    b = reference.default_block_config(4)[0]
    u_ref, c_ref, _ = reference.parallel_pairwise(d.astype(np.float64), b, cores(), use_float=True)
    assert np.array_equal(e.U.cpu().numpy(), u_ref)
    c = e.C.cpu().numpy()
    assert np.array_equal(c.view(np.uint32), c_ref.astype(np.float32).view(np.uint32))
    assert np.array_equal(c.astype(np.float64), c_ref)  # the widened fp32 values, exactly


@pytest.mark.parametrize("idx", [4, 2])
def test_triplet_full_matrix_vs_reference(reference, idx):
    """parallel_triplet<double>: U exact; C (diagonal 0) within 1e-5, and
    every row sum within 1e-5."""
    D, cfg = config_d(idx)
    d = D.cpu().numpy()
    e = gpu_run(D, "triplet")
    bf, bc = reference.default_block_config(8)[1:]
    u_ref, c_ref, _ = reference.parallel_triplet(d.astype(np.float64), bf, bc, cores(), use_float=False)
    assert np.array_equal(e.U.cpu().numpy(), u_ref)
    c = e.C.cpu().numpy()
    assert max_rel_diff(c, c_ref) <= 1e-5
    rs = np.abs(c.astype(np.float64).sum(1) - c_ref.sum(1)) / np.maximum(c_ref.sum(1), 1.0)
    assert float(rs.max()) <= 1e-5


@pytest.mark.slow
def test_cfg5_rows_rowsums_and_accurate_mode(oracle):
    """n = 32768 (config 5). Default mode: >= 64 rows bit-exact against the
    fp32 reference-order restatement (U and C). Accurate mode: the same rows
    within 1e-5 (in fact ~1e-7) of the fp64 accumulation, U identical. All n
    row sums of the default C within 1e-5 of the accurate double sums, and
    sum(C) = n(n-1)/2."""
    D, cfg = config_d(5)
    n = cfg.n
    d = D.cpu().numpy()
    rows = boundary_rows(n, extra=64 - 14, seed=5)
    assert rows.size >= 60
    e = gpu_run(D, "pairwise")
    U_rows = e.U[rows.tolist()].cpu().numpy()
    C_rows = e.C[rows.tolist()].cpu().numpy()
    rs_default = e.C.double().sum(1).cpu().numpy()
    total = float(rs_default.sum())
    del e
    torch.cuda.empty_cache()
    ur, cr = rows_parallel(oracle.pairwise_rows_f32, d, rows)
    assert np.array_equal(U_rows, ur)
    assert np.array_equal(C_rows.view(np.uint32), cr.view(np.uint32))
    a = gpu_run(D, "pairwise", accurate=True)
    assert np.array_equal(a.U[rows.tolist()].cpu().numpy(), ur)
    A_rows = a.C[rows.tolist()].cpu().numpy()
    A64_rows = a.C64[rows.tolist()].cpu().numpy()
    rs_acc = a.C64.sum(1).cpu().numpy()
    total_acc = float(rs_acc.sum())
    del a
    u64, c64 = rows_parallel(oracle.pairwise_rows_f64, d, rows)
    assert np.array_equal(u64, ur)
    err_acc = max_rel_diff(A_rows, c64)
    err_acc64 = max_rel_diff(A64_rows, c64)
    err_default = max_rel_diff(C_rows, c64)
    print(f"cfg5 rows vs fp64: default {err_default:.3g}, accurate {err_acc:.3g} (double sums {err_acc64:.3g})")
    assert err_acc <= 1e-5 and err_acc64 <= 1e-5
    # row sums: the fp64 oracle's own rows, then every row against the
    # accurate mode's double sums (validated on the rows above)
    assert float(np.max(np.abs(rs_acc[rows] - c64.sum(1)) / c64.sum(1))) <= 1e-6
    assert float(np.max(np.abs(rs_default - rs_acc) / rs_acc)) <= 1e-5
    # conservation, sum(C) = n(n-1)/2 (test_reference.cpp:160-181): the
    # default fp32 chains carry their rounding (2.7e-6 here), the accurate
    # double sums almost none
    half = n * (n - 1) / 2
    assert abs(total - half) / half < 1e-5
    assert abs(total_acc - half) / half < 1e-7  # measured 2.2e-8


def test_reference_acceptance_corpus_through_shim():
    """The reference's acceptance corpus through pald::gpu::* compiled with
    the reference's own types, against the reference's drivers in the same
    process; once on one device and once across a device list."""
    exe = ROOT / "oracle" / "_ref" / "acceptance_gpu"
    if not exe.exists():
        pytest.skip("oracle/_ref/acceptance_gpu not built (needs the reference headers at build time)")
    for devices in (None, "0,0"):
        env = dict(os.environ)
        if devices:
            env["PALD_GPU_DEVICES"] = devices
        r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900, env=env)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "0 failure(s)" in r.stdout, r.stdout
        print(devices, r.stdout.strip())
