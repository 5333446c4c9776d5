"""CPU check of the algebra the sm_100a kernels implement
(paper_2307_16652_b200/csrc/pald_kernels.cuh header comment).

The kernels evaluate both passes as semiring GEMMs over (row r, column c,
third point k) with per-element successor transforms nu(v) (= next fp32
value, bits + 1 for v >= 0). This file restates exactly those formulas in
numpy and checks them against the oracle -- tie-heavy inputs included --
so the derivation is pinned independently of the GPU.
"""
import numpy as np
import pytest

from helpers import int_upper, random_upper


def nu(v):
    return np.nextafter(v.astype(np.float32), np.float32(np.inf))


def pw_focus(d):
    n = d.shape[0]
    u = np.zeros((n, n), np.int64)
    for r in range(n):
        m = np.minimum(d[r][None, :], d)            # min(D[r][k], D[c][k]) over (c, k)
        u[r] = (m < d[r][:, None]).sum(1)
    np.fill_diagonal(u, 0)
    return u.astype(np.int32)


def pw_cohesion_f32(d, w):
    """C[r][c] = sum_k W[r][k] [D[r][c] < min(D[r][k], B'[k][c])],
    B' = nu(D[k][c]) iff k < r; fp32 accumulation over k ascending."""
    n = d.shape[0]
    dn = nu(d)
    c = np.zeros((n, n), np.float32)
    for r in range(n):
        acc = np.zeros(n, np.float32)
        for k in range(n):
            b = dn[k] if k < r else d[k]
            m = np.minimum(d[r, k], b)
            acc = np.where(d[r] < m, (acc + w[r, k]).astype(np.float32), acc)
        c[r] = acc
    return c


def tr_focus(d):
    n = d.shape[0]
    dn = nu(d)
    u = np.zeros((n, n), np.int64)
    idx = np.arange(n)
    for r in range(n):
        for cc in range(r + 1, n):
            a = np.where(idx < cc, dn[r], d[r])       # A' = nu(D[r][k]) iff k < c
            b = np.where(idx < r, dn[cc], d[cc])      # B' = nu(D[c][k]) iff k < r
            u[r, cc] = u[cc, r] = (np.minimum(a, b) < dn[r, cc]).sum()
    return u.astype(np.int32)


def tr_cohesion(d, w):
    n = d.shape[0]
    dn = nu(d)
    idx = np.arange(n)
    c = np.zeros((n, n))
    for p in range(n):
        for q in range(n):
            if p == q:
                continue
            a = np.where(idx < q, dn[p], d[p])
            b = np.where(idx < p, dn[q], d[q])
            c[p, q] = (w[p].astype(np.float64) * (d[p, q] < np.minimum(a, b))).sum()
    return c


CASES = [("rand", 23), ("ties", 23), ("ties", 37), ("rand", 41), ("ties3", 30)]


def make(kind, n):
    if kind == "rand":
        return random_upper(n, n)
    if kind == "ties":
        return int_upper(n, n)
    return int_upper(n, n, 1, 3)  # extreme ties


@pytest.mark.parametrize("kind,n", CASES)
def test_pairwise_formulation(oracle, kind, n):
    d = make(kind, n)
    u_ref, c_ref = oracle.pairwise_f32(d)
    u = pw_focus(d)
    assert np.array_equal(u, u_ref)
    w = np.where(u > 0, np.float32(1) / np.maximum(u, 1).astype(np.float32), np.float32(0))
    c = pw_cohesion_f32(d, w.astype(np.float32))
    assert np.array_equal(c.view(np.uint32), c_ref.view(np.uint32))


@pytest.mark.parametrize("kind,n", CASES)
def test_triplet_formulation(oracle, kind, n):
    d = make(kind, n)
    u_ref, c_ref = oracle.triplet_f64(d)
    u = tr_focus(d)
    assert np.array_equal(u, u_ref)
    w = np.where(u > 0, 1.0 / np.maximum(u, 1), 0.0)
    c = tr_cohesion(d, w)
    assert np.max(np.abs(c - c_ref)) < 1e-12


def ffma_sat_lt(a, b, S=2.0 ** 125):
    """sat(fma(b, S, -a*S)) evaluated exactly (float64 holds the scaled
    fp32 products exactly), rounded to fp32, saturated."""
    v = (b.astype(np.float64) * S - a.astype(np.float64) * S).astype(np.float32)
    return np.clip(v, 0.0, 1.0)


def test_ffma_sat_compare_exact():
    """The FFMA.SAT compare equals [a < b] on the fast path's value range
    [2^-102, 1) plus 0 and nu(0), ties and 1-ulp neighbours included."""
    rng = np.random.default_rng(0)
    base = np.concatenate([
        rng.random(20000, dtype=np.float32),
        np.float32(2.0 ** -102) * (1 + np.arange(200, dtype=np.float32)),
        np.array([0.0, np.float32(2.0 ** -149), 0.5, np.nextafter(np.float32(1), np.float32(0))], np.float32),
    ]).astype(np.float32)
    a = rng.choice(base, 200000)
    b = np.where(rng.random(200000) < 0.3, a, rng.choice(base, 200000)).astype(np.float32)
    b = np.where(rng.random(200000) < 0.2, nu(a), b).astype(np.float32)
    ok = (ffma_sat_lt(a, b) == (a < b).astype(np.float32))
    # Pairs drawn only from {0, nu(0), nu(nu(0))} never carry weight in the kernels:
    # they arise from the diagonal d_xx = 0, where W = 0 (cohesion) or the
    # other operand is an off-diagonal distance >= 2^-102 (focus).
    tiny = (a <= np.float32(2.0 ** -148)) & (b <= np.float32(2.0 ** -148))
    assert ok[~tiny].all()
