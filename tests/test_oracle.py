"""Pin the CPU oracle (oracle/pald_oracle.c) before trusting it:
  * the reference's hand-traced known answers (test_reference.cpp:12-124,
    acceptance.cpp:120-146),
  * golden vectors produced by the reference itself (tests/golden/golden.npz,
    tests/golden/make_golden.py),
  * live cross-checks against the compiled reference when oracle/_ref exists.
"""
from pathlib import Path

import numpy as np
import pytest

from helpers import int_upper, max_rel_diff, random_upper

GOLDEN = np.load(Path(__file__).resolve().parent / "golden" / "golden.npz")
CASES = sorted({k.split(".")[0] for k in GOLDEN.files})


def dmat(n, upper):
    d = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    d[iu] = upper
    d[(iu[1], iu[0])] = upper
    return d


def test_focus_size_hand_traced(oracle):
    d3 = dmat(3, [1.0, 2.0, 3.0])
    assert oracle.focus_size(d3, 0, 1, 0) == 2
    assert oracle.focus_size(d3, 0, 2, 0) == 3
    assert oracle.focus_size(d3, 1, 2, 0) == 3
    t3 = dmat(3, [1.0, 1.0, 1.0])
    assert oracle.focus_size(t3, 0, 1, 1) == 3
    assert oracle.focus_size(t3, 0, 2, 1) == 3
    assert oracle.focus_size(t3, 0, 1, 0) == 2


def test_pairwise_hand_traced(oracle):
    u, c = oracle.pairwise_entrywise(dmat(3, [1.0, 2.0, 3.0]), 0)
    assert u[0, 1] == u[1, 0] == 2 and u[0, 2] == 3 and u[1, 2] == 3
    assert c[0, 0] == pytest.approx(5 / 6, abs=1e-15)
    assert c[1, 1] == pytest.approx(5 / 6, abs=1e-15)
    assert c[2, 2] == pytest.approx(2 / 3, abs=1e-15)
    assert c[0, 1] == pytest.approx(1 / 3, abs=1e-15)
    assert c[0, 2] == 0.0
    assert c.sum() == pytest.approx(3.0, abs=1e-12)
    u2, c2 = oracle.pairwise_entrywise(dmat(2, [5.0]), 0)
    assert u2[0, 1] == 2 and c2[0, 0] == 0.5 and c2[1, 1] == 0.5


def test_t3_strict_and_split(oracle):
    t3 = dmat(3, [1.0, 1.0, 1.0])
    us, cs = oracle.pairwise_entrywise(t3, 0)
    ui, ci = oracle.pairwise_entrywise(t3, 1)
    for x in range(3):
        for z in range(3):
            assert cs[x, z] == (1.0 if x == z else 0.0)
            assert ci[x, z] == pytest.approx(2 / 3 if x == z else 1 / 6, abs=1e-15)
            if x != z:
                assert us[x, z] == 2 and ui[x, z] == 3


def test_triplet_hand_traced(oracle):
    d3 = dmat(3, [1.0, 2.0, 3.0])
    u, c = oracle.triplet_entrywise(d3)
    assert u[0, 1] == 2 and u[0, 2] == 3 and u[1, 2] == 3
    assert c[0, 1] == pytest.approx(1 / 3, abs=1e-15)
    assert c[1, 0] == pytest.approx(1 / 3, abs=1e-15)
    assert c[0, 0] == 0.0
    u2, c2 = oracle.triplet_entrywise(dmat(2, [5.0]))
    assert u2[0, 1] == 2 and c2[0, 1] == 0.0
    with pytest.raises(ValueError):
        oracle.triplet_entrywise(dmat(3, [1.0, 1.0, 1.0]), validate_ties=True)
    oracle.fill_diagonal(u, c)
    assert c[0, 0] == pytest.approx(5 / 6, abs=1e-15)
    assert c[2, 2] == pytest.approx(2 / 3, abs=1e-15)


@pytest.mark.parametrize("case", CASES)
def test_oracle_matches_golden(oracle, case):
    g = lambda k: GOLDEN[f"{case}.{k}"]  # noqa: E731
    d = g("D")
    u, c = oracle.pairwise_entrywise(d, 0)
    assert np.array_equal(u, g("pw_U"))
    assert np.array_equal(c, g("pw_C"))
    us, cs = oracle.pairwise_entrywise(d, 1)
    assert np.array_equal(us, g("split_U"))
    assert np.array_equal(cs, g("split_C"))
    ut, ct = oracle.triplet_entrywise(d)
    assert np.array_equal(ut, g("tr_U"))
    assert np.array_equal(ct, g("tr_C"))
    oracle.fill_diagonal(ut, ct)
    assert np.array_equal(ct, g("fill_C"))
    # fp32 reference-order restatement == blocked_pairwise<float>, bit for bit
    u32, c32 = oracle.pairwise_f32(d.astype(np.float32))
    assert np.array_equal(u32, g("pw_U"))
    assert np.array_equal(c32.astype(np.float64), g("pwf_C"))
    us32, cs32 = oracle.pairwise_f32(d.astype(np.float32), policy=1)
    assert np.array_equal(us32, g("split_U"))
    assert np.array_equal(cs32.astype(np.float64), g("splitf_C"))
    # fp64-on-fp32 oracles: U identical to the reference's, C within tolerance
    uf, cf = oracle.pairwise_f64(d.astype(np.float32))
    assert np.array_equal(uf, g("pw_U"))
    assert max_rel_diff(cf, g("pw_C")) < 1e-6
    utf, ctf = oracle.triplet_f64(d.astype(np.float32))
    assert np.array_equal(utf, g("tr_U"))
    assert max_rel_diff(ctf, g("trf_C")) < 1e-5


def test_invariants(oracle):
    """Conservation (test_reference.cpp:160-181): sum C = n(n-1)/2, mean
    normalized depth 1/2, 2 <= u <= n -- ties included."""
    for d in (random_upper(40, 1).astype(np.float64), int_upper(40, 2).astype(np.float64)):
        n = d.shape[0]
        u, c = oracle.pairwise_entrywise(d, 0)
        assert c.sum() == pytest.approx(n * (n - 1) / 2, rel=1e-12)
        off = u[~np.eye(n, dtype=bool)]
        assert off.min() >= 2 and off.max() <= n
        oracle.normalize(c)
        assert oracle.local_depths(c).mean() == pytest.approx(0.5, abs=1e-12)
        ut, ct = oracle.triplet_entrywise(d)
        oracle.fill_diagonal(ut, ct)
        assert ct.sum() == pytest.approx(n * (n - 1) / 2, rel=1e-12)


def test_oracle_vs_live_reference(oracle, reference):
    for n, seed in ((7, 1), (31, 2), (64, 3)):
        d = reference.random_distances(n, seed)
        assert np.array_equal(oracle.pairwise_entrywise(d, 0)[0], reference.pairwise_entrywise(d, 0)[0])
        u32, c32 = oracle.pairwise_f32(d.astype(np.float32))
        ur, cr, _ = reference.parallel_pairwise(d, 7, 4, use_float=True)
        assert np.array_equal(u32, ur)
        assert np.array_equal(c32.astype(np.float64), cr)
    d = int_upper(50, 9).astype(np.float64)
    u32, c32 = oracle.pairwise_f32(d.astype(np.float32))
    ur, cr, _ = reference.blocked_pairwise(d, 13, use_float=True)
    assert np.array_equal(u32, ur) and np.array_equal(c32.astype(np.float64), cr)
    ut, _ = oracle.triplet_entrywise(d)
    utr, _, _ = reference.parallel_triplet(d, 8, 4, 3, use_float=True)
    assert np.array_equal(ut, utr)


def test_rows_oracle_matches_full(oracle):
    d = int_upper(70, 5)
    u, c = oracle.pairwise_f32(d)
    rows = [0, 13, 69]
    ur, cr = oracle.pairwise_rows_f32(d, rows)
    assert np.array_equal(ur, u[rows])
    assert np.array_equal(cr.view(np.uint32), c[rows].view(np.uint32))


def test_pairwise_rows_f64_oracle_matches_full(oracle):
    for d in (int_upper(70, 6), random_upper(61, 7)):
        u, c = oracle.pairwise_f64(d)
        rows = [0, 17, d.shape[0] - 1]
        ur, cr = oracle.pairwise_rows_f64(d, rows)
        assert np.array_equal(ur, u[rows])
        assert np.max(np.abs(cr - c[rows])) < 1e-12


def test_triplet_rows_oracle_matches_full(oracle):
    for d in (int_upper(41, 3), random_upper(37, 4)):
        u, c = oracle.triplet_f64(d)
        rows = [0, 5, d.shape[0] - 1]
        ur, cr = oracle.triplet_rows_f64(d, rows)
        assert np.array_equal(ur, u[rows])
        assert np.max(np.abs(cr - c[rows])) < 1e-12


def test_oracle_matches_reference_on_fp32_degenerate_input(oracle, reference):
    """Distances valid in double that underflow to 0 in fp32 give u = 0 and
    w = inf; the reference's masked fp32 update then adds 0*inf = NaN. The
    restatement reproduces that exactly (same NaN rows, same finite values)."""
    n = 40
    rng = np.random.default_rng(5)
    d = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    v = rng.uniform(0.5, 2.0, iu[0].size)
    v[rng.random(iu[0].size) < 0.02] = 1e-50
    d[iu] = v
    d[(iu[1], iu[0])] = v
    ur, cr, _ = reference.blocked_pairwise(d, 8, use_float=True)
    uo, co = oracle.pairwise_f32(d.astype(np.float32))
    assert np.array_equal(uo, ur)
    assert np.array_equal(co.astype(np.float64), cr, equal_nan=True)
    assert np.isnan(cr).any()
