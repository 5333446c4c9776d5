"""The Python mirror of the reference API, host-side behaviour (no GPU):
DistanceMatrix validation identical to the compiled reference's
(types.hpp:45-65), error types, normalize / local_depths semantics."""
import numpy as np
import pytest

import paper_2307_16652_b200 as pg
from helpers import random_upper


def _cases():
    good = random_upper(6, 1).astype(np.float64)
    yield "good", good
    bad = good.copy(); bad[2, 2] = 1e-9; yield "diag", bad
    bad = good.copy(); bad[1, 3] = bad[3, 1] = 0.0; yield "zero", bad
    bad = good.copy(); bad[1, 3] = bad[3, 1] = -2.0; yield "neg", bad
    bad = good.copy(); bad[1, 3] = bad[3, 1] = np.nan; yield "nan", bad
    bad = good.copy(); bad[1, 3] += 1e-12; yield "asym", bad
    ok = good.copy(); ok[0, 0] = -0.0; yield "negzero_diag", ok
    ok = good.copy(); ok[1, 2] = ok[2, 1] = np.inf; yield "inf", ok


@pytest.mark.parametrize("name,d", list(_cases()))
def test_validation_matches_reference(reference, name, d):
    ref_rc = reference.validate(d)
    try:
        pg.DistanceMatrix(d.shape[0], d)
        ours = 0
    except pg.ValidationError:
        ours = 2
    assert ours == ref_rc, name


def test_validation_messages():
    with pytest.raises(pg.ValidationError, match="n >= 2"):
        pg.DistanceMatrix(1, [0.0])
    with pytest.raises(pg.ValidationError, match="storage size"):
        pg.DistanceMatrix(3, [0.0] * 8)
    d = random_upper(4, 2).astype(np.float64)
    d[0, 0] = 1.0
    with pytest.raises(pg.ValidationError, match=r"diagonal entry \(0,0\)"):
        pg.DistanceMatrix(4, d)


def test_policy_and_block_errors_without_gpu():
    d = pg.DistanceMatrix(3, np.array([[0, 1, 2], [1, 0, 3], [2, 3, 0]], float))
    with pytest.raises(pg.ValidationError):
        pg.blocked_pairwise(d, 0)
    with pytest.raises(pg.ValidationError):
        pg.blocked_triplet(d, 0, 1)
    with pytest.raises(pg.UnsupportedPolicyError):
        pg.blocked_triplet(d, 1, 1, pg.Policy.InclusiveSplit)
    with pytest.raises(pg.ValidationError):
        pg.parallel_pairwise(d, 1, pg.ParallelPlan(0, True))
    with pytest.raises(pg.UnsupportedPolicyError):
        pg.parallel_triplet(d, 1, 1, pg.ParallelPlan(2, True), pg.Policy.InclusiveSplit)
    with pytest.raises(pg.UnsupportedPolicyError):
        pg.blocked_pairwise(d, 1, real="float64")
    assert pg.to_string(pg.Policy.Strict) == "strict" and pg.to_string(pg.Policy.InclusiveSplit) == "split"


def test_normalize_and_depths_semantics():
    """The reference's precondition errors (reference.hpp:223-241) come
    before any device work; the arithmetic runs on the GPU
    (pald_gpu_normalize_f64 / pald_gpu_row_sums_f64) and is checked bit for
    bit against the reference in tests/test_gpu_analyze.py."""
    n = 7
    vals = np.random.default_rng(0).random((n, n))
    with pytest.raises(pg.ValidationError, match="already normalized"):
        pg.normalize(pg.CohesionMatrix(n, vals.copy(), True))
    with pytest.raises(pg.ValidationError, match="normalized"):
        pg.local_depths(pg.CohesionMatrix(n, vals.copy(), False))


@pytest.mark.parametrize("case", ["diag_after_offdiag", "offdiag_before_diag", "asym_then_negative", "nan", "neg_zero"])
def test_distance_matrix_first_violation_like_reference(reference, case):
    """The reference scans row by row (types.hpp:50-62): (x, x), then (x, y)
    for y > x with positivity before symmetry. With several violations the
    first in that order is reported, with the reference's exact message."""
    n = 9
    rng = np.random.default_rng(3)
    d = rng.uniform(0.5, 2.0, (n, n))
    d = np.triu(d, 1)
    d = d + d.T
    if case == "diag_after_offdiag":
        d[5, 5] = 1.0
        d[2, 7] = d[7, 2] = -1.5
    elif case == "offdiag_before_diag":
        d[4, 4] = 0.5
        d[1, 8] = 0.25  # asymmetric at (1, 8)
    elif case == "asym_then_negative":
        d[6, 2] = 3.0  # lower entry differs: "not symmetric at (2,6)"
        d[3, 8] = d[8, 3] = 0.0
    elif case == "nan":
        d[0, 4] = d[4, 0] = np.nan
    else:
        d[3, 3] = -0.0  # accepted: -0.0 == 0.0
        d[2, 5] = d[5, 2] = -0.0
    rc = reference.validate(d)
    assert rc == 2
    want = reference.lib.ref_last_error().decode()
    with pytest.raises(pg.ValidationError) as ei:
        pg.DistanceMatrix(n, d)
    assert str(ei.value) == want
